"""Per-launch encoder kernel times with the encoder block fusion on / off
(pilc_set_tuning key 0): python tools/bk_exp.py 1 0"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import _lib, vqvae
from paper_2206_05279_b200.synth import smooth_images
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
m = pc.random_weights(seed=1)
imgs = torch.from_numpy(smooth_images(8192, 32, 32, seed=0)).to(dev)
for v in [int(b) for b in sys.argv[1:]] or [1, 0]:
    prev = _lib.set_tuning(_lib.TUNE_BLOCK_FUSION, v)
    for _ in range(3):
        vqvae.encode_indices_device(imgs, m, dev, stream)
    torch.cuda.synchronize()
    _lib.prof_reset(True)
    for _ in range(5):
        vqvae.encode_indices_device(imgs, m, dev, stream)
    torch.cuda.synchronize()
    r = _lib.prof_read()
    print("fusion", v, {k: (v_[0] // 5, round(1000 * v_[1] / 5, 1)) for k, v_ in r.items()}, "(launches, us per encode)")
    _lib.set_tuning(_lib.TUNE_BLOCK_FUSION, prev)
