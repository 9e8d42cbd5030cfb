"""VQ-VAE density network on the GPU (semantics of `pixelcodec/vqvae.py`).

encode_to_indices: image -> nearest-codebook indices at half resolution
(vqvae.py:51-76); decode_to_params: indices -> per-subpixel logistic
(mu, s) (vqvae.py:79-113). On the codec path the decoder is fused with the
logistic head and emits the recentring shift round(mu) and the grid index d
directly (csrc/vq.cu); (mu, s) planes are only materialised for the
operator-level API below.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .device import CACHE, as_device_u8, ptr, require_device, sptr
from .errors import ModelError
from .logistic import ScaleGrid, default_grid
from .pmf import QuantizedPmf, quantize_pmf
from .predictor import validate_image
from .weights import ModelWeights


def _require_network(weights: ModelWeights) -> None:
    if not weights.has_network:
        raise ModelError("model has no network tensors")


def latent_shape(H: int, W: int) -> tuple[int, int]:
    return (H + 1) // 2, (W + 1) // 2


def grid_device(grid: ScaleGrid, dev):
    """(log2 grid values, d thresholds) as float64 device tensors, cached."""
    def make():
        lg = torch.from_numpy(np.log2(grid.values).astype(np.float64)).to(dev)
        th = grid.d_thresholds().astype(np.float64)
        return lg, (torch.from_numpy(th).to(dev) if th.size else None)
    return CACHE.get(("grid", grid.to_bytes()), dev, make)


def _workspace(n: int, H: int, W: int, weights: ModelWeights, dev) -> torch.Tensor:
    nb = _lib.load().pilc_vq_workspace_bytes(n, H, W, *weights.cfg_tuple())
    if nb < 0:
        raise ModelError("unsupported model configuration")
    return torch.empty(max(nb, 256), dtype=torch.uint8, device=dev)


def encode_indices_device(img_d: torch.Tensor, weights: ModelWeights, dev, stream, z_out=None,
                          exact: bool = True) -> torch.Tensor:
    """exact=True: the exact network (the reference's float arithmetic, z
    bit-identical); exact=False: the fast encoder (fp16-split tcgen05 for the
    default C=Dc=32 model, else the exact network)."""
    N, H, W, _ = img_d.shape
    gh, gw = latent_shape(H, W)
    idx = torch.empty((N, gh, gw), dtype=torch.uint8, device=dev)
    ws = _workspace(N, H, W, weights, dev)
    _lib.call("pilc_vq_encode_exact" if exact else "pilc_vq_encode", ptr(img_d), N, H, W, ptr(weights.device_model(dev)), *weights.cfg_tuple(),
              ptr(ws), ws.numel(), ptr(idx), ptr(z_out), sptr(stream))
    return idx


def decode_head_device(idx_d: torch.Tensor, weights: ModelWeights, H: int, W: int, grid: ScaleGrid, dev, stream,
                       want_params: bool = False, exact: bool = True, out=None):
    """-> (shift u8, d u8[, mu f32, s f32]) each (N, H, W, 3).

    exact=True: the exact network (mu, s bit-identical to the reference's
    decode_to_params); exact=False: the fast decoder (tcgen05 bf16 when
    container.fast_decoder(model, H, W), else the exact network).
    out=(shift, dsel): contiguous (N, H, W, 3) uint8 tensors to fill (e.g.
    row slices of a batch-sized pair)."""
    N = idx_d.shape[0]
    if out is not None:
        shift, dsel = out
        assert shift.is_contiguous() and dsel.is_contiguous() and shift.shape == dsel.shape == (N, H, W, 3)
    else:
        shift = torch.empty((N, H, W, 3), dtype=torch.uint8, device=dev)
        dsel = torch.empty((N, H, W, 3), dtype=torch.uint8, device=dev)
    mu = s = None
    if want_params:
        mu = torch.empty((N, H, W, 3), dtype=torch.float32, device=dev)
        s = torch.empty((N, H, W, 3), dtype=torch.float32, device=dev)
    thr = grid_device(grid, dev)[1]
    ws = _workspace(N, H, W, weights, dev)
    _lib.call("pilc_vq_decode_exact" if exact else "pilc_vq_decode", ptr(idx_d), N, H, W, ptr(weights.device_model(dev)), *weights.cfg_tuple(),
              ptr(thr), grid.D, ptr(ws), ws.numel(), ptr(shift), ptr(dsel), ptr(mu), ptr(s),
              sptr(stream))
    return (shift, dsel, mu, s) if want_params else (shift, dsel)


def encode_to_indices(image, weights: ModelWeights, *, exact: bool = True) -> np.ndarray:
    """Nearest-codebook index per latent; ties take the smaller index."""
    validate_image(image)
    _require_network(weights)
    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    img_d = as_device_u8(np.asarray(image)[None], dev, stream)
    return encode_indices_device(img_d, weights, dev, stream, exact=exact)[0].cpu().numpy()


def encoder_latents(image, weights: ModelWeights, *, exact: bool = True) -> np.ndarray:
    """Pre-argmin latents z (gh, gw, Dc) float32 (testing hook)."""
    validate_image(image)
    _require_network(weights)
    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    H, W = np.asarray(image).shape[:2]
    gh, gw = latent_shape(H, W)
    z = torch.empty((1, gh, gw, weights.config.Dc), dtype=torch.float32, device=dev)
    img_d = as_device_u8(np.asarray(image)[None], dev, stream)
    encode_indices_device(img_d, weights, dev, stream, z_out=z, exact=exact)
    return z[0].cpu().numpy()


def argmin_codebook(z, weights: ModelWeights, *, tensor_cores: bool = False) -> np.ndarray:
    """Codebook argmin alone on (..., Dc) latents (vqvae.py:66-76): the
    float32-screen kernel, or (tensor_cores=True, Dc = C = 32) the encoders'
    tensor-core argmin (3xTF32 GEMM, proven radius, float64 rescore)."""
    z = np.ascontiguousarray(z, dtype=np.float32)
    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    zd = torch.from_numpy(z.reshape(-1, z.shape[-1]).copy()).to(dev)
    out = torch.empty(zd.shape[0], dtype=torch.uint8, device=dev)
    if tensor_cores:
        nb = _lib.load().pilc_vq_argmin_tc_workspace(zd.shape[0])
        ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=dev)
        _lib.call("pilc_vq_argmin_tc", ptr(zd), zd.shape[0], ptr(weights.device_model(dev)), *weights.cfg_tuple(),
                  ptr(ws), ws.numel(), ptr(out), sptr(stream))
    else:
        _lib.call("pilc_vq_argmin", ptr(zd), zd.shape[0], ptr(weights.device_model(dev)), *weights.cfg_tuple(),
                  ptr(out), sptr(stream))
    return out.cpu().numpy().reshape(z.shape[:-1])


def decode_to_params(indices, weights: ModelWeights, out_shape: tuple[int, int], *, exact: bool = True):
    """Per-pixel (mu, s) planes H x W x 3 float32, computed on the GPU by the
    exact network (bit-identical to the reference's) or, exact=False, by the
    fast decoder."""
    _require_network(weights)
    H, W = out_shape
    gh, gw = latent_shape(H, W)
    indices = np.asarray(indices)
    if indices.shape != (gh, gw):
        raise ModelError(f"index grid {indices.shape}, expected {(gh, gw)}")
    if indices.min() < 0 or indices.max() >= weights.config.K:
        raise ModelError("codebook index out of range")
    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    idx_d = torch.from_numpy(indices.astype(np.uint8)[None].copy()).to(dev)
    _, _, mu, s = decode_head_device(idx_d, weights, H, W, default_grid(), dev, stream, want_params=True,
                                     exact=exact)
    return mu[0].cpu().numpy(), s[0].cpu().numpy()


def index_histogram_pmf(weights: ModelWeights, M: int) -> QuantizedPmf:
    """Index-stream distribution: stored usage counts + 1 (vqvae.py:116-119).
    Memoised per (histogram bytes, M) on the weights object."""
    memo = weights.__dict__.setdefault("_index_pmf_memo", {})
    key = (weights.histogram.tobytes(), M)
    pmf = memo.get(key)
    if pmf is None:
        pmf = memo[key] = quantize_pmf(weights.histogram.astype(np.float64) + 1.0, M)
    return pmf
