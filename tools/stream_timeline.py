"""GPU timeline of StreamCodec steady state (events around each request's
kernels on the kernel stream): kernel time per request and the idle gap
before it. PROBE_PRE=dev runs the bench's device-timed steps first.
python tools/stream_timeline.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_05279_b200 as pc
from paper_2206_05279_b200 import stream as st
from paper_2206_05279_b200 import container as ct
from paper_2206_05279_b200.device import pinned
from paper_2206_05279_b200.synth import smooth_images

N, H = 8192, 32
m = pc.random_weights(seed=1)
cfg = pc.CodecConfig(backend="twar-vqvae", numerics="fast")
imgs0 = smooth_images(N, H, H, seed=0)
imgs = pinned(imgs0.nbytes).numpy().reshape(imgs0.shape)
imgs[...] = imgs0
dev = torch.device("cuda", 0)
if "dev" in os.environ.get("PROBE_PRE", ""):
    img_d = torch.from_numpy(imgs0).to(dev)
    s0 = torch.cuda.current_stream(dev)
    for _ in range(6):
        o, off = ct._compress_device(img_d, m, cfg, dev, s0)
        ct._decompress_device(o, off, N, m, dev, s0)
    torch.cuda.synchronize()
marks = []
oc, od = st._compress_device, st._decompress_device
def wrap(fn, tag):
    def f(*a, **k):
        s = torch.cuda.current_stream()
        h0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True); e0.record(s)
        r = fn(*a, **k)
        e1 = torch.cuda.Event(enable_timing=True); e1.record(s)
        marks.append((tag, e0, e1, time.perf_counter() - h0))
        return r
    return f
st._compress_device = wrap(oc, "C")
st._decompress_device = wrap(od, "D")
K = 13
from paper_2206_05279_b200 import _lib
prof = "prof" in os.environ.get("PROBE_PRE", "")
with st.StreamCodec(m, cfg, dev) as codec:
    if prof:
        _lib.prof_reset(True)
    fcs, pend = [codec.compress(imgs) for _ in range(2)], None
    for k in range(K):
        b, o = fcs.pop(0).result()
        if k + 2 < K:
            fcs.append(codec.compress(imgs))
        fd = codec.decompress(b, o)
        if pend is not None:
            pend.result()
        pend = fd
    pend.result()
torch.cuda.synchronize()
if prof:
    agg = {}
    for k_, ms, u in _lib.prof_records():
        a = agg.setdefault(k_, [0, 0.0])
        a[0] += 1
        a[1] += ms
    for k_, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k_:22s} {c:4d} launches {1e3 * ms / c:8.1f} us each")
t0 = marks[0][1]
prev_end = None
durs = {"C": [], "D": []}
for i, (tag, e0, e1, th) in enumerate(marks):
    s, e = t0.elapsed_time(e0), t0.elapsed_time(e1)
    gap = s - prev_end if prev_end is not None else 0.0
    if os.environ.get("VERBOSE"):
        print(f"{tag} start {s:8.2f} ms  dur {e - s:6.2f}  gap {gap:6.2f}  host call {1e3 * th:6.2f} ms")
    if 4 <= i < len(marks) - 3:
        durs[tag].append(e - s)
    prev_end = e
import statistics
print("steady C %.2f ms  D %.2f ms" % (statistics.median(durs["C"]), statistics.median(durs["D"])))
