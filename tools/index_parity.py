"""Codebook-index agreement of the GPU encoder with the oracle (numpy/BLAS
restatement of the reference, bit-identical to pixelcodec on the same BLAS)
over a sample of synthetic images. Usage: python tools/index_parity.py [n] [H]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import vqvae
from paper_2206_05279_b200.synth import smooth_images
from oracle import oracle as O

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
H = int(sys.argv[2]) if len(sys.argv) > 2 else 32
m = pc.random_weights(seed=1)
om = O.Model.from_bytes(m.to_bytes())
imgs = smooth_images(n, H, H, seed=123)
t0 = time.time()
gpu = np.stack([vqvae.encode_to_indices(im, m) for im in imgs])
ref = np.stack([O.encode_indices(im, om) for im in imgs])
bad = int((gpu != ref).sum())
print(f"images {n} {H}x{H}: index mismatches {bad} / {ref.size} ({time.time() - t0:.1f} s)")
