"""Step time of the bench's device loop with / without per-launch event timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import _lib, container as ct
from paper_2206_05279_b200.synth import smooth_images
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev)
model = pc.random_weights(seed=1); cfg = pc.CodecConfig(backend="twar-vqvae")
img_d = torch.from_numpy(smooth_images(8192, 32, 32, seed=0)).to(dev)
def step():
    o, off = ct._compress_device(img_d, model, cfg, dev, stream)
    ct._decompress_device(o, off, 8192, model, dev, stream)
for _ in range(3): step()
for timing in (False, True, False):
    _lib.prof_reset(timing)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(10): step()
    t1 = time.perf_counter()
    e1.record(stream); torch.cuda.synchronize()
    print(f"timing={timing}: device {e0.elapsed_time(e1) / 10:.3f} ms/step, host enqueue {1e3 * (t1 - t0) / 10:.3f} ms/step")
_lib.prof_reset(False)
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); step(); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
