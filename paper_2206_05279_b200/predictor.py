"""TWAR three-neighbour predictor (semantics of `pixelcodec/predictor.py`).

Parameters, hashing and validation are host-side; the residual transform and
its inverse run on the GPU (csrc/twar.cu) with the reference's float
contract: float32 accumulation left to right, bias last, no FMA, round half
away from zero in float64, mod 256 (_kernels.py:69-88).

Out of scope here (offline, sequential-only in the reference): ridge
fitting (`fit_params`) and the k=4..7 receptive-field variants.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import as_device_u8, ptr, require_device, sptr
from .errors import ParameterError, UnsupportedConfigurationError


@dataclass(frozen=True)
class PredictorParams:
    """Per-channel context weights (3, 3) and biases (3,), float32."""

    weights: np.ndarray
    bias: np.ndarray

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=np.float32)
        b = np.asarray(self.bias, dtype=np.float32)
        if w.ndim != 2 or w.shape[0] != 3 or b.shape != (3,):
            raise ParameterError("weights must be (3, k), bias (3,)")
        if not (np.all(np.isfinite(w)) and np.all(np.isfinite(b))):
            raise ParameterError("predictor parameters must be finite")
        object.__setattr__(self, "weights", w)
        object.__setattr__(self, "bias", b)

    @property
    def k(self) -> int:
        return int(self.weights.shape[1])

    def to_bytes(self) -> bytes:
        """12 float32 LE: (W_r, b_r, W_g, b_g, W_b, b_b) (predictor.py:66-74)."""
        if self.k != 3:
            raise ParameterError("only 3-context parameters serialize")
        return b"".join(struct.pack("<3f", *self.weights[c]) + struct.pack("<f", self.bias[c]) for c in range(3))

    @classmethod
    def from_bytes(cls, data: bytes) -> "PredictorParams":
        if len(data) != 48:
            raise ParameterError("expected 48 bytes of predictor parameters")
        v = struct.unpack("<12f", data)
        return cls(np.array([v[0:3], v[4:7], v[8:11]], np.float32), np.array([v[3], v[7], v[11]], np.float32))

    def hash8(self) -> bytes:
        return hashlib.sha256(self.to_bytes()).digest()[:8]

    def wire12(self) -> np.ndarray:
        """The 12 floats in wire order, as passed to the CUDA kernels."""
        if self.k != 3:
            raise UnsupportedConfigurationError(f"GPU predictor needs k=3, not k={self.k}")
        return np.frombuffer(self.to_bytes(), dtype="<f4").copy()


def default_params() -> PredictorParams:
    """Gradient predictor (predictor.py:89-92)."""
    return PredictorParams(np.array([[-1, 1, 1], [1, -1, 1], [1, -1, 1]], np.float32), np.zeros(3, np.float32))


def validate_image(image) -> np.ndarray:
    image = np.asarray(image)
    if image.dtype != np.uint8:
        raise ParameterError("image must be uint8")
    if image.ndim != 3 or image.shape[2] != 3:
        raise ParameterError("image must be H x W x 3")
    if image.shape[0] < 1 or image.shape[1] < 1:
        raise ParameterError("image dimensions must be >= 1")
    return image


def _batch(x) -> tuple:
    x = np.asarray(x) if not isinstance(x, torch.Tensor) else x
    if x.ndim == 3:
        return x[None], True
    if x.ndim != 4 or x.shape[-1] != 3:
        raise ParameterError("expected (H, W, 3) or (N, H, W, 3)")
    return x, False


def forward_residual_device(img_d: torch.Tensor, params: PredictorParams, stream) -> torch.Tensor:
    N, H, W, _ = img_d.shape
    res = torch.empty_like(img_d)
    p12 = params.wire12()
    _lib.call("pilc_twar_forward", ptr(img_d), ptr(res), N, H, W, ptr(p12), sptr(stream))
    return res


def decode_device(coded_d: torch.Tensor, params: PredictorParams, stream, shift_d=None) -> torch.Tensor:
    N, H, W, _ = coded_d.shape
    out = torch.empty_like(coded_d)
    p12 = params.wire12()
    _lib.call("pilc_twar_decode", ptr(coded_d), ptr(shift_d), ptr(out), N, H, W, ptr(p12), sptr(stream))
    return out


def _run(fn, x, params):
    xb, single = _batch(x)
    if not isinstance(xb, torch.Tensor):
        if xb.dtype != np.uint8:
            raise ParameterError("image must be uint8")
        if xb.shape[1] < 1 or xb.shape[2] < 1:
            raise ParameterError("image dimensions must be >= 1")
    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    xd = as_device_u8(xb, dev, stream)
    out = fn(xd, params or default_params(), stream)
    if isinstance(x, torch.Tensor):
        return out[0] if single else out
    o = out.cpu().numpy()
    return o[0] if single else o


def forward_residual(image, params: PredictorParams | None = None):
    """(x - x_hat + 128) mod 256 (predictor.py:292-294), on the GPU."""
    return _run(forward_residual_device, image, params)


def forward_residual_batch(images, params: PredictorParams):
    return _run(forward_residual_device, images, params)


def decode_parallel(residual, params: PredictorParams | None = None):
    """Wavefront inverse (predictor.py:309-311), on the GPU."""
    return _run(decode_device, residual, params)


# The GPU wavefront decode is bit-identical to the raster order by
# construction (cells within a wave are independent), so the sequential
# entry points share it.
decode_sequential = decode_parallel


def decode_parallel_batch(residuals, params: PredictorParams):
    return _run(decode_device, residuals, params)


decode_sequential_batch = decode_parallel_batch
