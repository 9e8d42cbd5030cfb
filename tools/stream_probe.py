"""Timeline of StreamCodec round trips (diagnostic): python tools/stream_probe.py [H] [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_05279_b200 as pc  # noqa: E402
from paper_2206_05279_b200.device import pinned  # noqa: E402
from paper_2206_05279_b200.stream import StreamCodec  # noqa: E402
from paper_2206_05279_b200.synth import smooth_images  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 32
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
m = pc.random_weights(seed=1)
cfg = pc.CodecConfig(backend="twar-vqvae", numerics="fast")
imgs0 = smooth_images(N, H, H, seed=0)
imgs = pinned(imgs0.nbytes).numpy().reshape(imgs0.shape)
imgs[...] = imgs0
for rep in range(3):
    with StreamCodec(m, cfg) as codec:
        T = time.perf_counter
        t0 = T()
        log = []
        fc = codec.compress(imgs)
        log.append(("submit c0", T() - t0))
        pend = None
        for k in range(5):
            buf, off = fc.result()
            log.append((f"c{k} done", T() - t0))
            if k + 1 < 5:
                fc = codec.compress(imgs)
                log.append((f"submit c{k+1}", T() - t0))
            fd = codec.decompress(buf, off)
            log.append((f"submit d{k}", T() - t0))
            if pend is not None:
                pend.result()
                log.append((f"d{k-1} done", T() - t0))
            pend = fd
        pend.result()
        log.append(("d4 done", T() - t0))
        print(f"rep {rep}: {1e3 * (T() - t0) / 5:.2f} ms/step  " + "  ".join(f"{a}@{1e3 * b:.1f}" for a, b in log))
t0 = time.perf_counter()
for k in range(5):
    b, o = pc.compress_batch(imgs, m, cfg)
    pc.decompress_batch(b, o, m)
print(f"sync: {1e3 * (time.perf_counter() - t0) / 5:.2f} ms/step")
