"""Digest of the fast encoder's z and indices (and the fast decoder's outputs)
for fixed inputs -- compare two builds (PILC_LIB_PATH) for bit identity:
python tools/z_digest.py [H] [N]"""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import vqvae
from paper_2206_05279_b200.device import as_device_u8
from paper_2206_05279_b200.logistic import default_grid
from paper_2206_05279_b200.synth import smooth_images
H = int(sys.argv[1]) if len(sys.argv) > 1 else 32
N = int(sys.argv[2]) if len(sys.argv) > 2 else 512
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev)
m = pc.random_weights(seed=1)
imgs = smooth_images(N, H, H, seed=3)
gh, gw = vqvae.latent_shape(H, H)
z = torch.empty((N, gh, gw, 32), dtype=torch.float32, device=dev)
idx = vqvae.encode_indices_device(as_device_u8(imgs, dev, stream), m, dev, stream, z_out=z, exact=False)
r = vqvae.decode_head_device(idx, m, H, H, default_grid(), dev, stream, want_params=True, exact=False)
torch.cuda.synchronize()
for name, t in [("z", z), ("idx", idx)] + list(zip(("shift", "d", "mu", "s"), r)):
    print(name, hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16])
