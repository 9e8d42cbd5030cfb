"""Host->device copy strategies for a pageable 25 MB image batch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
dev = torch.device("cuda", 0)
arr = np.random.default_rng(0).integers(0, 256, (8192, 32, 32, 3), dtype=np.uint8)
d = torch.empty(arr.size, dtype=torch.uint8, device=dev)
pin = torch.empty(arr.size, dtype=torch.uint8, pin_memory=True)
pool = ThreadPoolExecutor(8)
flat = arr.reshape(-1)
def par_copy(dst, src, k=8):
    step = -(-src.size // k)
    list(pool.map(lambda i: np.copyto(dst[i:i + step], src[i:i + step]), range(0, src.size, step)))
def t(name, fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(f"{name:40s} {1e3 * min(ts):6.2f} ms (min) {1e3 * np.median(ts):6.2f} ms (median)")
t("torch copy_ pageable (blocking)", lambda: d.copy_(torch.from_numpy(flat)))
t("torch copy_ pageable non_blocking", lambda: d.copy_(torch.from_numpy(flat), non_blocking=True))
t("par_copy(8) -> pinned + async copy", lambda: (par_copy(pin.numpy(), flat), d.copy_(pin, non_blocking=True)))
t("par_copy(16) -> pinned + async copy", lambda: (par_copy(pin.numpy(), flat, 16), d.copy_(pin, non_blocking=True)))
t("np.copyto -> pinned + async", lambda: (np.copyto(pin.numpy(), flat), d.copy_(pin, non_blocking=True)))
def chunked():
    # 4 MB chunks: memcpy chunk k+1 while DMA of chunk k runs
    ch = 4 << 20
    s = torch.cuda.current_stream()
    for i in range(0, flat.size, ch):
        np.copyto(pin.numpy()[i:i + ch], flat[i:i + ch])
        d[i:i + ch].copy_(pin[i:i + ch], non_blocking=True)
t("chunked memcpy+DMA overlap", chunked)
def reg():
    cr = torch.cuda.cudart()
    r = cr.cudaHostRegister(flat.ctypes.data, flat.nbytes, 0)
    d.copy_(torch.from_numpy(flat), non_blocking=True); torch.cuda.synchronize()
    cr.cudaHostUnregister(flat.ctypes.data)
t("cudaHostRegister + DMA + unregister", reg)
import threading
def threaded(k):
    def go():
        step = -(-flat.size // k)
        streams = [torch.cuda.Stream() for _ in range(k)]
        def work(i):
            with torch.cuda.stream(streams[i]):
                d[i * step:(i + 1) * step].copy_(torch.from_numpy(flat[i * step:(i + 1) * step]))
        ts = [threading.Thread(target=work, args=(i,)) for i in range(k)]
        for t_ in ts: t_.start()
        for t_ in ts: t_.join()
    return go
for k in (2, 4, 8):
    t(f"{k} threads, pageable copy_ per slice", threaded(k))
