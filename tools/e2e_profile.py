"""Phase timings of the public batch API (host buffers in, host buffers out)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import container as ct, device as dv
from paper_2206_05279_b200.synth import smooth_images
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev)
model = pc.random_weights(seed=1); cfg = pc.CodecConfig(backend="twar-vqvae", numerics="fast")
imgs = smooth_images(8192, 32, 32, seed=0)
for _ in range(3):
    buf, off = pc.compress_batch(imgs, model, cfg); out = pc.decompress_batch(buf, off, model)
T = {}
def tic(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    t0 = tic(); img_d = dv.as_device_u8(imgs, dev, stream); t1 = tic()
    o, offd = ct._compress_device(img_d, model, cfg, dev, stream); t2 = tic()
    buf, off = pc.compress_batch(imgs, model, cfg); t3 = tic()
    out = pc.decompress_batch(buf, off, model); t4 = tic()
    bd = dv.h2d(buf, dev, stream, pad=16); t5 = tic()
    print(f"h2d imgs {1e3*(t1-t0):.2f} ms | compress kernels {1e3*(t2-t1):.2f} | compress_batch {1e3*(t3-t2):.2f} | "
          f"decompress_batch {1e3*(t4-t3):.2f} | h2d blobs {1e3*(t5-t4):.2f}")
t0 = time.perf_counter(); p = dv.pinned(imgs.nbytes); print("pinned alloc", 1e3*(time.perf_counter()-t0))
print("cpus", len(os.sched_getaffinity(0)))
a = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True); d = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
pg = torch.empty(64 << 20, dtype=torch.uint8)
for name, src, dst in [("pinned h2d", a, d), ("pageable h2d", pg, d), ("pinned d2h", d, a), ("pageable d2h", d, pg)]:
    for _ in range(2): dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5): dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
    print(f"{name}: {64 * 1.048576 / dt / 1e3:.1f} GB/s")
print("returned blob buffer is page-locked:", torch.from_numpy(buf).is_pinned())
