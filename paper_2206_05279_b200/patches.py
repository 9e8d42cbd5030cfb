"""High-resolution frames as independent patch containers (BASELINE config 4).

The paper evaluates high-resolution images as fixed-size crops
(`PAPER.md:431-432`). A frame is split into a grid of ph x pw patches (the
last row / column may be smaller) and each patch is a self-contained PILC
blob, so a frame compresses and decompresses as one batch of patches (two or
four shape groups) and the patches shard across CTAs and GPUs with no
exchange.
"""

from __future__ import annotations

import numpy as np

from .container import CodecConfig, compress_batch, decompress_batch


def patch_grid(H: int, W: int, ph: int = 64, pw: int = 64):
    """[(y0, y1, x0, x1)] in raster order."""
    return [(y, min(y + ph, H), x, min(x + pw, W)) for y in range(0, H, ph) for x in range(0, W, pw)]


def split_frame(frame: np.ndarray, ph: int = 64, pw: int = 64) -> list:
    H, W = frame.shape[:2]
    return [np.ascontiguousarray(frame[y0:y1, x0:x1]) for (y0, y1, x0, x1) in patch_grid(H, W, ph, pw)]


def assemble(patches: list, H: int, W: int, ph: int = 64, pw: int = 64) -> np.ndarray:
    out = np.empty((H, W, 3), np.uint8)
    for p, (y0, y1, x0, x1) in zip(patches, patch_grid(H, W, ph, pw)):
        out[y0:y1, x0:x1] = p
    return out


def compress_frames(frames, model=None, config: CodecConfig = CodecConfig(), ph: int = 64, pw: int = 64):
    """Frames (list or (F, H, W, 3)) -> (buffer, offsets) of F * n_patches blobs."""
    patches = [p for f in frames for p in split_frame(np.asarray(f), ph, pw)]
    return compress_batch(patches, model, config)


def decompress_frames(buffer, offsets, n_frames: int, H: int, W: int, model=None, ph: int = 64, pw: int = 64):
    out = decompress_batch(buffer, offsets, model)
    per = len(patch_grid(H, W, ph, pw))
    if isinstance(out, np.ndarray):
        out = list(out)
    return np.stack([assemble(out[f * per:(f + 1) * per], H, W, ph, pw) for f in range(n_frames)])
