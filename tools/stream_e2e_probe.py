"""Steady-state StreamCodec intervals as bench.py measures them (two
compresses queued ahead), repeated, with the completion pool size as a knob:
python tools/stream_e2e_probe.py [workers] [reps] [steps]"""
import os, statistics, sys, time
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200.device import pinned
from paper_2206_05279_b200.stream import StreamCodec
from paper_2206_05279_b200.synth import smooth_images

workers = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
K = int(sys.argv[3]) if len(sys.argv) > 3 else 13
N, H = 8192, 32
m = pc.random_weights(seed=1)
cfg = pc.CodecConfig(backend="twar-vqvae", numerics="fast")
imgs0 = smooth_images(N, H, H, seed=0)
imgs = pinned(imgs0.nbytes).numpy().reshape(imgs0.shape)
imgs[...] = imgs0
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
pre = os.environ.get("PROBE_PRE", "")
if "dev" in pre:  # the bench's device-timed steps first
    from paper_2206_05279_b200 import container as ct
    img_d = torch.from_numpy(imgs0).to(dev)
    s0 = torch.cuda.current_stream(dev)
    for _ in range(6):
        o, off = ct._compress_device(img_d, m, cfg, dev, s0)
        ct._decompress_device(o, off, N, m, dev, s0)
    torch.cuda.synchronize()
if "sync" in pre:  # the bench's synchronous API rounds
    for _ in range(6):
        b, o = pc.compress_batch(imgs, m, cfg)
        pc.decompress_batch(b, o, m)
for rep in range(reps):
    done = []
    with StreamCodec(m, cfg, dev) as codec:
        if workers != 1:
            codec._done.shutdown()
            codec._done = ThreadPoolExecutor(max_workers=workers)
        def comp(k):
            with torch.cuda.stream(codec.kern):
                flush.fill_(k & 0xFF)
            return codec.compress(imgs)
        fcs, pend = [comp(k) for k in range(2)], None
        for k in range(K):
            b, o = fcs.pop(0).result()
            if k + 2 < K:
                fcs.append(comp(k + 2))
            fd = codec.decompress(b, o)
            if pend is not None:
                pend.result(); done.append(time.perf_counter())
            pend = fd
        pend.result(); done.append(time.perf_counter())
    iv = [1e3 * (b - a) for a, b in zip(done[:-1], done[1:])]
    print(f"workers {workers} rep {rep}: median {statistics.median(iv):.2f} ms  " + " ".join(f"{x:.2f}" for x in iv))
