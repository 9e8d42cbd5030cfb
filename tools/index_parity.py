"""Codebook-index agreement of the GPU encoder with the oracle (numpy/BLAS
restatement of the reference, bit-identical to pixelcodec on the same BLAS)
over a sample of synthetic images.
Usage: python tools/index_parity.py [n] [H] [random|trained] [smooth|noise]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import vqvae
from paper_2206_05279_b200.synth import smooth_images
from oracle import oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
wts = sys.argv[3] if len(sys.argv) > 3 else "random"
kind = sys.argv[4] if len(sys.argv) > 4 else "smooth"
m = (pc.ModelWeights.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                       "trained.pilw")) if wts == "trained" else pc.random_weights(seed=1))
om = O.Model.from_bytes(m.to_bytes())
if kind == "noise":
    imgs = np.random.default_rng(123).integers(0, 256, (n, H, H, 3), dtype=np.uint8)
else:
    imgs = smooth_images(n, H, H, seed=123)
t0 = time.time()
import torch
from paper_2206_05279_b200.device import as_device_u8, require_device
dev = require_device()
stream = torch.cuda.current_stream(dev)
gpu = np.concatenate([vqvae.encode_indices_device(as_device_u8(imgs[i:i + 512], dev, stream), m, dev, stream, exact=False).cpu().numpy()
                      for i in range(0, n, 512)])
ref = np.stack([O.encode_indices(im, om) for im in imgs])
bad = int((gpu != ref).sum())
print(f"{wts} weights, {kind} images {n} {H}x{H}: index mismatches {bad} / {ref.size} ({time.time() - t0:.1f} s)")
