"""Per-launch device times of one compress + decompress step (live, CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import _lib, container as ct
from paper_2206_05279_b200.synth import smooth_images
H = int(sys.argv[1]) if len(sys.argv) > 1 else 32
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev)
NUM = sys.argv[3] if len(sys.argv) > 3 else "fast"
for kv in filter(None, os.environ.get("PILC_TUNING", "").split(",")):  # e.g. PILC_TUNING=1=1,3=0
    k, v = kv.split("=")
    _lib.set_tuning(int(k), int(v))
model = pc.random_weights(seed=1); cfg = pc.CodecConfig(backend="twar-vqvae", numerics=NUM)
img_d = torch.from_numpy(smooth_images(N, H, H, seed=0)).to(dev)
def step():
    o, off = ct._compress_device(img_d, model, cfg, dev, stream)
    ct._decompress_device(o, off, img_d.shape[0], model, dev, stream)
for _ in range(3): step()
torch.cuda.synchronize(); _lib.prof_reset(True); step(); torch.cuda.synchronize()
tot = 0
for k, ms, u in _lib.prof_records():
    tot += ms
    print(f"{k:22s} {ms*1e3:9.1f} us  units={u:.3g}")
print("sum", tot)
