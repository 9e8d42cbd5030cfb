"""CPU tests: host-side config-time code of the product vs the reference's
golden vectors, the C-ABI surface, and header handling. No GPU needed."""

import ctypes
import hashlib
import json
import os
import re
import struct

import numpy as np
import pytest

import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import _lib, container, logistic, tables
from paper_2206_05279_b200.bits import BitStack
from paper_2206_05279_b200.errors import CorruptStreamError, FormatError, ParameterError
from paper_2206_05279_b200.synth import mulberry32, smooth_images

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")


@pytest.fixture(scope="module")
def meta():
    with open(os.path.join(GOLDEN, "meta.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("M", [10, 11, 12])
def test_tables_match_reference(golden, meta, M):
    t = golden("tables.npz")
    pmfs = logistic.residual_distributions(logistic.default_grid(), M)
    assert np.array_equal(np.stack([p.P.astype(np.int64) for p in pmfs]), t[f"P_M{M}"])
    enc, dec = tables.build_tables(pmfs, M, verify=True)
    assert np.array_equal(enc.delta, t[f"delta_M{M}"]) and np.array_equal(enc.phi, t[f"phi_M{M}"])
    assert np.array_equal(dec.symbol, t[f"symbol_M{M}"])
    assert np.array_equal(dec.pop_count, t[f"pop_M{M}"])
    assert np.array_equal(dec.next_base, t[f"next_M{M}"])
    h = hashlib.sha256()
    for a in (enc.delta, enc.phi, dec.symbol, dec.pop_count, dec.next_base):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest()[:16] == meta[f"table_digest_M{M}"]
    assert enc.footprint_bytes == 4 * 8 * 256 and dec.footprint_bytes == 8 * (1 << (M + 2))


def test_golden_delta_phi():
    # test_tables.py:17-28: P=1024 at M=12 -> delta=4096, phi=3072
    P = np.full(4, 1024)
    enc, _ = tables.build_tables([pc.QuantizedPmf(12, P)], 12)
    assert int(enc.delta[0, 0]) == 4096 and int(enc.phi[0, 0]) == 3072


def test_table_cache_by_content():
    """build_tables is memoised by the masses' bytes: equal content -> the
    same tables (per-call host time), rejections are never cached."""
    pmfs = logistic.residual_distributions(logistic.default_grid(), 12)
    a = tables.build_tables(pmfs, 12)
    copies = [pc.QuantizedPmf(12, p.P.copy()) for p in pmfs]
    b = tables.build_tables(copies, 12, verify=True)
    assert a[0] is b[0] and a[1] is b[1]
    bad = pc.QuantizedPmf(12, np.array([2047, 2049]))  # inadmissible: P > 2^(M-1) - 1
    for _ in range(2):
        with pytest.raises(pc.CodecError):
            tables.build_tables([bad], 12)
    with pytest.raises(pc.CodecError):
        tables.build_tables(pmfs, 11)  # quantized at M=12


def test_quantizer_known_answers():
    assert np.all(pc.quantize_pmf(np.ones(256), 12).P == 16)
    q = pc.quantize_pmf(np.array([3.0, 1.0]), 12)  # test_pmf.py:58-62
    assert list(q.P.astype(int)) == [2047, 2049] and not q.is_admissible
    p = logistic.discretized_logistic_pmf(128, 8, 12)
    assert int(p.P[128]) == 111  # test_logistic.py:32-38


def test_recentring_kl_frozen():
    # test_logistic.py:160-169 frozen values (mpmath oracle)
    assert abs(logistic.recentring_kl(96, 8.0) - 1.98021255006e-5) < 1e-13
    assert abs(logistic.recentring_kl(160, 8.0) - 2.25015791305e-5) < 1e-13
    assert logistic.recentring_kl(128, 4.0) == 0.0


def test_model_hashes(golden, meta):
    small = pc.ModelWeights.load(os.path.join(GOLDEN, "small.pilw"))
    assert small.hash8().hex() == meta["small_hash8"]
    assert small.to_bytes() == golden("small.pilw")
    assert pc.random_weights(pc.ModelConfig(32, 8, 8, 1), seed=42).to_bytes() == golden("small.pilw")
    assert pc.random_weights(seed=1).hash8().hex() == meta["full_seed1_hash8"]
    assert pc.default_params().hash8().hex() == meta["default_params_hash8"]


def test_bits_wire_golden(meta):
    s = BitStack()
    for b in (1, 0, 1, 1):
        s.push(b)
    assert list(s.to_bytes()) == meta["bits_golden"]
    back = BitStack.from_bytes(s.to_bytes())
    assert back.pop_bits(4) == 0b1101


def test_parse_header_on_golden_static(golden):
    z = golden("static.npz")
    offs, buf = z["offs"], z["buf"]
    for i in range(len(offs) - 1):
        blob = buf[offs[i]:offs[i + 1]].tobytes()
        h, off = container.parse_header(blob)
        L, M, dbg = (int(v) for v in z["cfg"][i])
        img = z[f"img{z['img_index'][i]}"]
        assert (h.lanes, h.M, h.height, h.width) == (L, M, img.shape[0], img.shape[1])
        assert (h.schedule_checksum is not None) == bool(dbg)
        info = container.inspect(blob)
        assert info["container_bytes"] == len(blob)


def test_parse_header_errors(golden):
    z = golden("static.npz")
    blob = z["buf"][z["offs"][0]:z["offs"][1]].tobytes()
    with pytest.raises(FormatError):
        container.parse_header(b"JUNK" + blob[4:])
    with pytest.raises(FormatError):
        container.parse_header(b"PIL")
    bad = bytearray(blob)
    bad[-6] ^= 1
    with pytest.raises(CorruptStreamError):
        container.parse_header(bytes(bad))


def test_config_validation():
    with pytest.raises(ParameterError):
        pc.CodecConfig(backend="zip")
    with pytest.raises(ParameterError):
        pc.CodecConfig(M=13)
    with pytest.raises(ParameterError):
        pc.CodecConfig(lanes=0)


def test_header_template_layout():
    cfg = pc.CodecConfig(lanes=3, M=11)
    t = container._template(0, cfg, 5, 9, pc.default_params(), None)
    assert t[:4] == b"PILC" and t[4:9] == bytes([1, 0, 11, 0, 0])
    assert struct.unpack_from("<IIHH", t, 9) == (5, 9, 3, 0)
    assert len(t) == 23 + 8 * 8 + 8


def test_library_exports_every_declared_symbol():
    """libpilc_sm100a.so loads on a CPU-only host and exports every entry
    point include/pilc.h declares (no compute calls without a GPU)."""
    with open(os.path.join(REPO, "include", "pilc.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"\b(pilc_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 18
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert set(_lib._SIGS) == declared
    assert _lib.version().startswith("pilc-sm100a")
    # host-only helpers are callable without a device
    L = _lib.load()
    assert L.pilc_model_floats(256, 32, 32, 4) > 207142
    assert L.pilc_vq_workspace_bytes(8, 32, 32, 256, 32, 32, 4) > 0


def test_model_pack_layout():
    m = pc.random_weights(pc.ModelConfig(16, 4, 8, 1), seed=3)
    L = _lib.load()
    n = L.pilc_model_floats(16, 4, 8, 1)
    canon = np.concatenate([m.tensors[k].ravel() for k in pc.weights.tensor_shapes(m.config)]).astype(np.float32)
    out = np.zeros(n, np.float32)
    _lib.call("pilc_model_pack", ctypes.c_void_p(canon.ctypes.data), 16, 4, 8, 1, ctypes.c_void_p(out.ctypes.data))
    # every weight appears exactly once (padding is zero)
    assert np.isclose(np.sort(np.abs(out[out != 0])), np.sort(np.abs(canon[canon != 0]))).all()


def test_synth_mulberry32_matches_reference_generator():
    # mulberry32(seed=0) first outputs (trainer data.ts:17-26), checked by
    # an independent scalar transcription
    def scalar(seed, k):
        out, a = [], seed
        for _ in range(k):
            a = (a + 0x6D2B79F5) & 0xFFFFFFFF
            t = ((a ^ (a >> 15)) * (1 | a)) & 0xFFFFFFFF
            t = ((t + (((t ^ (t >> 7)) * (61 | t)) & 0xFFFFFFFF)) & 0xFFFFFFFF) ^ t
            out.append(((t ^ (t >> 14)) & 0xFFFFFFFF) / 4294967296)
        return out
    assert np.allclose(mulberry32(7, 0, 50), scalar(7, 50), rtol=0, atol=0)
    imgs = smooth_images(2, 8, 12, seed=3)
    assert imgs.shape == (2, 8, 12, 3) and imgs.dtype == np.uint8


def test_offsets_validation():
    """decompress_batch / decompress_frames validate blob offsets before any
    device work (the parse kernel trusts them): one-dimensional,
    non-negative, non-decreasing."""
    from paper_2206_05279_b200.container import check_offsets
    from paper_2206_05279_b200.errors import FormatError

    assert check_offsets([0, 5, 5, 9]).dtype == np.uint64
    for bad in ([[0, 1], [1, 2]], [0, 7, 3], [-1, 4], []):
        with pytest.raises(FormatError):
            check_offsets(np.array(bad))


def test_lane_size_limit():
    """The GPU coder's lane bit positions are 32-bit: compress refuses lanes
    that could exceed 2^31 bits (and tells the caller to use more lanes)."""
    from paper_2206_05279_b200.container import _check_lane_size
    from paper_2206_05279_b200.errors import ParameterError

    _check_lane_size(3 * 4096 * 4096, 1, 12)
    with pytest.raises(ParameterError, match="more lanes"):
        _check_lane_size(3 * 8192 * 8192, 1, 12)
    _check_lane_size(3 * 8192 * 8192, 2, 12)
