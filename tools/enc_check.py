import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import vqvae
from paper_2206_05279_b200.synth import smooth_images
m = pc.random_weights(seed=1)
for (H, W) in [(32, 32), (17, 13), (64, 64)]:
    img = smooth_images(1, H, W, seed=1)[0]
    zt = vqvae.encoder_latents(img, m)
    zf = vqvae.encoder_latents(img, m, precise=True)
    print(H, W, float(np.abs(zt - zf).max()), float(np.abs(zf).max()), flush=True)
