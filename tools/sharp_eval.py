"""bits/dim of the fast numerics against the exact (reference-identical)
numerics for a model file, on N synthetic CIFAR-shaped images.

    python tools/sharp_eval.py model.pilw [N]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2206_05279_b200 as pc  # noqa: E402
from paper_2206_05279_b200 import vqvae  # noqa: E402
from paper_2206_05279_b200.synth import smooth_images  # noqa: E402

m = pc.ModelWeights.load(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
for H in (32, 64):
    imgs = smooth_images(n if H == 32 else n // 4, H, H, seed=77)
    out = {}
    for num in ("exact", "fast"):
        buf, off = pc.compress_batch(imgs, m, pc.CodecConfig(backend="twar-vqvae", numerics=num))
        assert np.array_equal(pc.decompress_batch(buf, off, m), imgs)
        out[num] = 8.0 * float(off[-1]) / imgs.size
    sbuf, soff = pc.compress_batch(imgs)
    idx_f = np.stack([vqvae.encode_to_indices(im, m, exact=False) for im in imgs[:64]])
    idx_e = np.stack([vqvae.encode_to_indices(im, m) for im in imgs[:64]])
    print(f"{H}x{H} n={len(imgs)}: bpd exact {out['exact']:.5f} fast {out['fast']:.5f} "
          f"rel {(out['fast'] - out['exact']) / out['exact']:+.5%}  static {8.0 * float(soff[-1]) / imgs.size:.4f}  "
          f"codes used {(m.histogram > 0).sum()}  index agreement (64 imgs) {(idx_f == idx_e).mean():.6f}")
