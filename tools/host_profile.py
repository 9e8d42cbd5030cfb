"""Where does host time go in one compress + decompress of the bench batch?"""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import container as ct
from paper_2206_05279_b200.synth import smooth_images
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
model = pc.random_weights(seed=1)
cfg = pc.CodecConfig(backend="twar-vqvae", numerics="fast")
imgs = smooth_images(8192, 32, 32, seed=0)
img_d = torch.from_numpy(imgs).to(dev)
def step():
    out_d, off_d = ct._compress_device(img_d, model, cfg, dev, stream)
    r = ct._decompress_device(out_d, off_d, img_d.shape[0], model, dev, stream)
    torch.cuda.synchronize()
    return r
for _ in range(3):
    step()
t0 = time.perf_counter(); step(); print("step wall", time.perf_counter() - t0)
pr = cProfile.Profile(); pr.enable(); step(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
t0 = time.perf_counter()
buf, off = pc.compress_batch(imgs, model, cfg)
t1 = time.perf_counter()
out = pc.decompress_batch(buf, off, model)
t2 = time.perf_counter()
print("e2e compress", t1 - t0, "decompress", t2 - t1)
pr = cProfile.Profile(); pr.enable(); buf, off = pc.compress_batch(imgs, model, cfg); out = pc.decompress_batch(buf, off, model); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
