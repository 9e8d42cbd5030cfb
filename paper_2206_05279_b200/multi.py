"""One process, several GPUs: the batch API over a list of devices.

Images and blobs are independent: a batch splits into
contiguous shares, one per device, each driven by its own host thread (the
CUDA library calls release the GIL) on that device's current stream, with
the device's own cached tables and packed model. Nothing is exchanged
between devices. The host side is zero-copy:

  compress    each device encodes its share and reports its total blob
              bytes; once every share is sized, one page-locked output
              buffer is allocated and every device copies its blobs straight
              into its slice of it (offsets rebased by the preceding shares'
              totals) -- no per-device host buffer, no concatenation.
  decompress  each device gets a view of its blobs (offsets rebased to the
              share's first blob) and, when the batch is one shape (read from
              blob 0's header), copies its images straight into its rows of
              one page-locked (N, H, W, 3) output.

Outputs are byte-identical to a one-device call: every per-image result is
independent of batch composition and device.
"""

from __future__ import annotations

import struct
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from .device import pinned, require_device
from .shard import shard_range

_POOLS: dict = {}


def _pool(k: int) -> ThreadPoolExecutor:
    if k not in _POOLS:
        _POOLS[k] = ThreadPoolExecutor(max_workers=k, thread_name_prefix="pilc-dev")
    return _POOLS[k]


def _run(k: int, fn):
    """fn(i) on k threads; the first exception (in share order) is raised --
    a share's own error before the broken barriers it left the others."""
    futs = [_pool(k).submit(fn, i) for i in range(k)]
    res, errs = [], []
    for f in futs:
        try:
            res.append(f.result())
        except BaseException as e:  # noqa: BLE001
            res.append(None)
            errs.append(e)
    if errs:
        own = [e for e in errs if not isinstance(e, threading.BrokenBarrierError)]
        raise (own or errs)[0]
    return res


def compress_multi(images, model, config, devices):
    from .container import compress_batch

    devs = [require_device(d) for d in devices]
    k = len(devs)
    if isinstance(images, torch.Tensor):
        images = images.cpu().numpy()
    arr = np.asarray(images)
    N = arr.shape[0]
    spans = [shard_range(N, i, k) for i in range(k)]
    sized = threading.Barrier(k)
    placed = threading.Barrier(k)
    totals = [0] * k
    host = {}

    def work(i):
        dev = devs[i]
        torch.cuda.set_device(dev)
        s, e = spans[i]
        try:
            if e > s:
                out_d, off_d, total = compress_batch(arr[s:e], model, config, device=dev, return_device=True)
                offs = off_d.cpu().numpy().view(np.uint64)
            else:
                out_d, offs, total = None, np.zeros(1, np.uint64), 0
            totals[i] = total
            sized.wait()
            if i == 0:
                host["buf"] = pinned(sum(totals) + 8)
                host["off"] = np.zeros(N + 1, np.uint64)
            placed.wait()
            base = sum(totals[:i])
            if total:
                stream = torch.cuda.current_stream(dev)
                with torch.cuda.stream(stream):
                    host["buf"][base: base + total].copy_(out_d[:total], non_blocking=True)
                stream.synchronize()
            host["off"][s + 1: e + 1] = offs[1:] + np.uint64(base)
        except BaseException:
            sized.abort()
            placed.abort()
            raise

    _run(k, work)
    total = sum(totals)
    return host["buf"].numpy()[:total], host["off"]


def decompress_multi(buffer, offsets, model, devices, raise_on_error: bool = True):
    from .container import check_offsets, decompress_batch
    from .errors import FormatError

    devs = [require_device(d) for d in devices]
    k = len(devs)
    offs = check_offsets(offsets)
    buf = np.frombuffer(buffer, np.uint8) if isinstance(buffer, (bytes, bytearray, memoryview)) \
        else np.ascontiguousarray(buffer, dtype=np.uint8)
    n = offs.size - 1
    if int(offs[-1]) > buf.size:
        raise FormatError("container truncated")
    spans = [shard_range(n, i, k) for i in range(k)]
    # one shape (the usual batch): every share decodes into its rows of one
    # page-locked output; a share that turns out otherwise returns its own
    shape = None
    if n and int(offs[1]) - int(offs[0]) >= 17 and bytes(buf[int(offs[0]): int(offs[0]) + 4]) == b"PILC":
        W, H = struct.unpack_from("<II", buf, int(offs[0]) + 9)
        if 0 < W * H <= (1 << 31) and n * H * W * 3 <= (1 << 40):
            shape = (H, W)
    out = pinned(n * shape[0] * shape[1] * 3).numpy().reshape(n, *shape, 3) if shape else None

    def work(i):
        dev = devs[i]
        torch.cuda.set_device(dev)
        s, e = spans[i]
        if e == s:
            return [], {}
        sub = buf[int(offs[s]): int(offs[e])]
        soff = offs[s: e + 1] - offs[s]
        dst = out[s:e] if out is not None else None
        return decompress_batch(sub, soff, model, device=dev, raise_on_error=False, out=dst)

    parts = _run(k, work)
    errors = {}
    uniform = out is not None
    for (s, e), (imgs, errs) in zip(spans, parts):
        errors.update({s + j: err for j, err in errs.items()})
        if e > s and not (isinstance(imgs, np.ndarray) and out is not None
                          and imgs.__array_interface__["data"][0] == out[s:e].__array_interface__["data"][0]):
            uniform = False
    if uniform and not errors:
        res = out
    else:
        res = [None] * n
        for (s, e), (imgs, _) in zip(spans, parts):
            for j in range(e - s):
                res[s + j] = None if (s + j) in errors else imgs[j]
    if errors and raise_on_error:
        raise errors[min(errors)]
    return (res, errors) if not raise_on_error else res
