"""One strided-lane coder configuration (coder-only config 5) for ncu:
python tools/coder_probe.py L [n_log2]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2206_05279_b200 import _lib, tables  # noqa: E402
from paper_2206_05279_b200.device import ptr, sptr  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 24)
M = 12
syms, d, pmfs = bench._bench_symbols(M, n)
enc, dec = tables.build_tables(pmfs, M)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
s_d = torch.from_numpy(syms).to(dev)
d_d = torch.from_numpy(d.astype(np.uint8)).to(dev)
for _ in range(3):
    scr, cap, nb, stt = tables.encode_lanes_device(s_d, 1, n, L, enc, dev, st, dsched=d_d)
    lane_off = torch.arange(L, dtype=torch.int64, device=dev) * (cap * 4)
    out = torch.empty(n, dtype=torch.uint8, device=dev)
    lstat = torch.zeros(L, dtype=torch.uint8, device=dev)
    _lib.call("pilc_rans_decode", ptr(scr), ptr(lane_off), ptr(nb), ptr(stt), ptr(d_d), None, 1, n, L,
              ptr(dec.device_words(dev)), dec.D, M, None, ptr(out), ptr(lstat), sptr(st))
torch.cuda.synchronize()
assert torch.equal(out, s_d)
print("ok")
