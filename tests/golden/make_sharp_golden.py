"""tests/golden/vqvae_sharp.npz: pixelcodec's own twar-vqvae containers for
the sharp model (sharp.pilw, make_sharp.py) on 6 synthetic images, with the
reference's indices / mu / s. Run in the build container (imports the
reference read-only, like make_golden.py):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_sharp_golden.py
"""

import os
import sys

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from pixelcodec import container, vqvae  # noqa: E402
from pixelcodec.weights import ModelWeights  # noqa: E402

from paper_2206_05279_b200.synth import smooth_images  # noqa: E402

if __name__ == "__main__":
    model = ModelWeights.load(os.path.join(HERE, "sharp.pilw"))
    out, blobs = {}, []
    for k, (h, w) in enumerate([(32, 32), (32, 32), (64, 64), (17, 13), (1, 1), (31, 33)]):
        img = smooth_images(1, h, w, seed=500 + k)[0]
        idx = vqvae.encode_to_indices(img, model)
        mu, s = vqvae.decode_to_params(idx, model, (h, w))
        blob = container.compress(img, model, container.CodecConfig(backend="twar-vqvae", lanes=1 + (k % 2)))
        assert np.array_equal(container.decompress(blob, model), img)
        out.update({f"img{k}": img, f"idx{k}": idx, f"mu{k}": mu, f"s{k}": s})
        blobs.append(blob)
    sizes = np.array([len(b) for b in blobs], np.int64)
    offs = np.zeros(len(blobs) + 1, np.int64)
    np.cumsum(sizes, out=offs[1:])
    out["buf"], out["offs"], out["n"] = np.frombuffer(b"".join(blobs), np.uint8), offs, np.array(len(blobs))
    np.savez_compressed(os.path.join(HERE, "vqvae_sharp.npz"), **out)
    print("bpd", [round(8 * len(b) / (out[f"img{k}"].size), 3) for k, b in enumerate(blobs)])
