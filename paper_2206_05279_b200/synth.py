"""Synthetic benchmark images (no datasets offline).

"smooth": vectorised port of the trainer's generator
(`pkg/trainer/src/data.ts:16-59`): mulberry32 stream, three sinusoids with
per-channel tint over a random base, +-2 uniform noise, clip + round-half-up.
mulberry32's k-th output depends only on seed + k*0x6d2b79f5, so the whole
stream is computed in one numpy pass. Generalised from square to H x W.

"noise": uniform bytes from numpy's default_rng, as the reference tests use.
"""

from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x6D2B79F5)
_M32 = np.uint64(0xFFFFFFFF)


def _imul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    return (a * b) & _M32


def mulberry32(seed: int, start: int, count: int) -> np.ndarray:
    """Outputs start..start+count-1 of mulberry32(seed) as float64 in [0,1)."""
    k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    a = (np.uint64(seed & 0xFFFFFFFF) + k * _GOLDEN) & _M32
    t = _imul(a ^ (a >> np.uint64(15)), np.uint64(1) | a)
    t = ((t + _imul(t ^ (t >> np.uint64(7)), np.uint64(61) | t)) & _M32) ^ t
    return ((t ^ (t >> np.uint64(14))) & _M32).astype(np.float64) / 4294967296.0


def smooth_images(count: int, height: int, width: int | None = None, seed: int = 0) -> np.ndarray:
    """(count, H, W, 3) uint8 smooth colour fields (data.ts:28-59)."""
    W = height if width is None else width
    H = height
    per_img = 22 + H * W * 3
    out = np.empty((count, H, W, 3), dtype=np.uint8)
    u = np.arange(H, dtype=np.float64)[:, None]
    v = np.arange(W, dtype=np.float64)[None, :]
    for n in range(count):
        r = mulberry32(seed, n * per_img, per_img)
        head, noise = r[:22], r[22:].reshape(H, W, 3)
        val = np.full((H, W, 3), 60.0 + 140.0 * head[21])
        for k in range(3):
            amp, fu, fv, ph = 20 + 60 * head[7 * k], (head[7 * k + 1] - 0.5) / 4, (head[7 * k + 2] - 0.5) / 4, head[7 * k + 3] * np.pi * 2
            tint = head[7 * k + 4 : 7 * k + 7]
            wave = np.sin(2 * np.pi * (fu * u + fv * v) + ph)
            val += amp * tint[None, None, :] * wave[:, :, None]
        val += 4 * (noise - 0.5)
        out[n] = np.clip(np.floor(val + 0.5), 0, 255).astype(np.uint8)
    return out


def noise_images(count: int, height: int, width: int | None = None, seed: int = 0) -> np.ndarray:
    W = height if width is None else width
    return np.random.default_rng(seed).integers(0, 256, (count, height, W, 3), dtype=np.uint8)
