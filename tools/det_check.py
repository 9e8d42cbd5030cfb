"""Determinism of the tcgen05 decoder: identical calls must give identical (shift, d)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import vqvae
from paper_2206_05279_b200.logistic import default_grid
dev = torch.device("cuda", 0); s = torch.cuda.current_stream(dev)
m = pc.random_weights(seed=1)
for n in (1, 7, 512, 4096):
    idx = torch.from_numpy(np.random.default_rng(n).integers(0, 256, (n, 16, 16), dtype=np.uint8)).to(dev)
    outs = [tuple(t.cpu().numpy() for t in vqvae.decode_head_device(idx, m, 32, 32, default_grid(), dev, s)) for _ in range(4)]
    same = all(np.array_equal(outs[0][0], o[0]) and np.array_equal(outs[0][1], o[1]) for o in outs[1:])
    print(n, "deterministic" if same else "NOT deterministic",
          [int((outs[0][0] != o[0]).sum()) for o in outs[1:]])
