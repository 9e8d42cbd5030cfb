"""pytest plugin: run the reference's own test modules against this
package's GPU operator twins (tests/test_reference_suite.py loads it with
`-p reference_twins` in a subprocess).

The reference package (pixelcodec, installed unmodified in baseline/_ref by
tools/install_reference.sh) is imported first; then its hot-path entry
points are replaced by adapters onto this package:

    container.compress / decompress   -> container.compress / decompress
    tables.interleaved_encode / decode -> the GPU rANS lanes
    predictor.forward_residual(_batch), decode_parallel(_batch)
                                       -> the GPU TWAR kernels
    vqvae.encode_to_indices / decode_to_params
                                       -> the exact GPU network

Reference objects (ModelWeights, CodecConfig, ScaleGrid, PredictorParams,
tables, LaneSet / BitStack) cross the seam through their wire forms, and
this package's exception classes are rebound to the reference's, so the
reference tests' `pytest.raises(...)` see the classes they import. Every
other reference function (nn, rans, pmf, logistic, CLI helpers, ...) stays
the reference's own.
"""

from __future__ import annotations

import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

import pixelcodec as P  # noqa: E402
from pixelcodec import bits as Pbits  # noqa: E402
from pixelcodec import container as Pcont  # noqa: E402
from pixelcodec import errors as Perr  # noqa: E402
from pixelcodec import predictor as Ppred  # noqa: E402
from pixelcodec import tables as Ptab  # noqa: E402
from pixelcodec import vqvae as Pvq  # noqa: E402

import paper_2206_05279_b200 as G  # noqa: E402
from paper_2206_05279_b200 import bits as Gbits  # noqa: E402
from paper_2206_05279_b200 import container as Gcont  # noqa: E402
from paper_2206_05279_b200 import errors as Gerr  # noqa: E402
from paper_2206_05279_b200 import logistic as Glog  # noqa: E402
from paper_2206_05279_b200 import predictor as Gpred  # noqa: E402
from paper_2206_05279_b200 import tables as Gtab  # noqa: E402
from paper_2206_05279_b200 import vqvae as Gvq  # noqa: E402
from paper_2206_05279_b200 import weights as Gw  # noqa: E402

TWINS: list[str] = []


def _rebind_errors():
    mapping = {}
    for name in dir(Gerr):
        ours = getattr(Gerr, name)
        if isinstance(ours, type) and issubclass(ours, Exception) and hasattr(Perr, name):
            mapping[ours] = getattr(Perr, name)
    for mname, mod in list(sys.modules.items()):
        if not mname.startswith("paper_2206_05279_b200") or mod is None:
            continue
        for k, v in list(vars(mod).items()):
            if isinstance(v, type) and v in mapping:
                setattr(mod, k, mapping[v])
            elif isinstance(v, dict):
                for kk, vv in list(v.items()):
                    if isinstance(vv, tuple) and vv and isinstance(vv[0], type) and vv[0] in mapping:
                        v[kk] = (mapping[vv[0]],) + vv[1:]


_models: dict = {}


def _model(m):
    if m is None:
        return None
    hit = _models.get(id(m))
    if hit is None or hit[0] is not m:
        hit = _models[id(m)] = (m, Gw.ModelWeights.from_bytes(m.to_bytes()))
    return hit[1]


def _config(c):
    if c is None:
        return Gcont.CodecConfig()
    return Gcont.CodecConfig(backend=c.backend, M=c.M, lanes=c.lanes,
                             grid=Glog.ScaleGrid.from_bytes(c.grid.to_bytes())[0],
                             verify_tables=c.verify_tables, debug_schedule_check=c.debug_schedule_check)


def _params(p):
    return None if p is None else Gpred.PredictorParams(np.asarray(p.weights), np.asarray(p.bias))


def _patch(mod, name, fn):
    setattr(mod, name, fn)
    if getattr(P, name, None) is not None and mod is not P:
        setattr(P, name, fn)
    TWINS.append(f"{mod.__name__}.{name}")


def compress(image, model=None, config=None):
    return Gcont.compress(image, _model(model), _config(config))


def decompress(blob, model=None, workers=1):
    return Gcont.decompress(blob, _model(model), workers)


def interleaved_encode(symbols, d_schedule, lanes, tables):
    ours = Gtab.interleaved_encode(symbols, d_schedule, lanes, Gtab.EncodeTables(tables.M, tables.delta, tables.phi))
    return Ptab.LaneSet(list(ours.states), [Pbits.BitStack.from_bytes(s.to_bytes()) for s in ours.streams])


def interleaved_decode(lane_set, count, d_schedule, tables, workers=1):
    ours = Gtab.LaneSet(list(lane_set.states), [Gbits.BitStack.from_bytes(s.to_bytes()) for s in lane_set.streams])
    dec = Gtab.DecodeTables(tables.M, tables.symbol, tables.pop_count, tables.next_base)
    return Gtab.interleaved_decode(ours, count, d_schedule, dec, workers)


def _k3(params) -> bool:
    return params is None or np.asarray(params.weights).shape == (3, 3)


_ref_fwd, _ref_par = Ppred.forward_residual, Ppred.decode_parallel
_ref_fwd_b = getattr(Ppred, "forward_residual_batch", None)
_ref_par_b = getattr(Ppred, "decode_parallel_batch", None)


def forward_residual(image, params=None):
    if not _k3(params):  # receptive-field variants (k = 4..7) are out of scope: the reference's own
        return _ref_fwd(image, params)
    return Gpred.forward_residual(image, _params(params))


def decode_parallel(residual, params=None):
    if not _k3(params):
        return _ref_par(residual, params)
    return Gpred.decode_parallel(residual, _params(params))


def forward_residual_batch(images, params):
    if not _k3(params):
        return _ref_fwd_b(images, params)
    return Gpred.forward_residual_batch(images, _params(params))


def decode_parallel_batch(residuals, params):
    if not _k3(params):
        return _ref_par_b(residuals, params)
    return Gpred.decode_parallel_batch(residuals, _params(params))


def encode_to_indices(image, weights):
    return Gvq.encode_to_indices(image, _model(weights))


def decode_to_params(indices, weights, out_shape):
    return Gvq.decode_to_params(indices, _model(weights), out_shape)


def pytest_configure(config):
    _rebind_errors()
    _patch(Pcont, "compress", compress)
    _patch(Pcont, "decompress", decompress)
    _patch(Ptab, "interleaved_encode", interleaved_encode)
    _patch(Ptab, "interleaved_decode", interleaved_decode)
    _patch(Ppred, "forward_residual", forward_residual)
    _patch(Ppred, "decode_parallel", decode_parallel)
    if _ref_fwd_b is not None:
        _patch(Ppred, "forward_residual_batch", forward_residual_batch)
    if _ref_par_b is not None:
        _patch(Ppred, "decode_parallel_batch", decode_parallel_batch)
    _patch(Pvq, "encode_to_indices", encode_to_indices)
    _patch(Pvq, "decode_to_params", decode_to_params)
    print("reference suite against the GPU twins: " + ", ".join(TWINS), file=sys.stderr, flush=True)
