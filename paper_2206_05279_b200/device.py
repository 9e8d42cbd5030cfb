"""Device plumbing: torch owns device memory and streams, the CUDA library
owns the compute. Pointers cross the C ABI as plain integers.

Every GPU entry point calls `require_device()`, which raises if there is no
sm_100 device or the library is not built: no silent CPU fallback exists.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _lib

_checked: set = set()
_lock = threading.Lock()


def require_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.LibraryError("paper_2206_05279_b200 needs a CUDA device (B200, sm_100a); none is visible")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
    with _lock:
        if dev.index not in _checked:
            _lib.load()
            major, minor = torch.cuda.get_device_capability(dev)
            if major != 10:
                raise _lib.LibraryError(f"device {dev} is sm_{major}{minor}; this build targets sm_100a only")
            _checked.add(dev.index)
    return dev


def ptr(t) -> ctypes.c_void_p | None:
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return ctypes.c_void_p(t.ctypes.data)
    return ctypes.c_void_p(t.data_ptr())


def sptr(stream: torch.cuda.Stream) -> ctypes.c_void_p:
    return ctypes.c_void_p(stream.cuda_stream)


def pinned(nbytes: int) -> torch.Tensor:
    """Page-locked host buffer (torch's caching host allocator). Buffers the
    batch API returns (blob buffers, decoded images) live here, so feeding
    them back (decompress_batch(compress_batch(...))) DMAs with no staging."""
    return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)


_READBACK: dict = {}


def readback(host: torch.Tensor, src: torch.Tensor, stream: torch.cuda.Stream) -> torch.cuda.Event:
    """Small device result -> page-locked host, after `stream`'s work so far,
    on a per-device read-back stream; returns the copy's completion event.
    Issued on `stream` itself the copy would wait on the copy engine behind
    other streams' large transfers (a pipelined caller's image and blob
    downloads) and hold back every kernel queued after it (measured: +0.7 ms
    per CIFAR-8192 decompress under StreamCodec)."""
    key = src.device.index
    rb = _READBACK.get(key)
    if rb is None:
        rb = _READBACK.setdefault(key, torch.cuda.Stream(src.device))
    after = torch.cuda.Event()
    after.record(stream)
    rb.wait_event(after)
    src.record_stream(rb)
    with torch.cuda.stream(rb):
        host.copy_(src, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(rb)
    return ev


def h2d(arr: np.ndarray, dev: torch.device, stream: torch.cuda.Stream, pad: int = 0) -> torch.Tensor:
    """Host numpy -> device tensor on `stream`. Page-locked sources (any
    cudaHostAlloc'd / registered memory, e.g. buffers this package returned)
    DMA asynchronously; pageable ones go through the driver's staged copy
    (measured ~30 GB/s on the B200 box, faster than a host memcpy into a
    pinned buffer followed by a DMA)."""
    a = np.ascontiguousarray(arr)
    flat = a.view(np.uint8).reshape(-1)
    out = torch.empty(flat.size + pad, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(stream):
        if flat.size:
            if not flat.flags.writeable:  # e.g. np.frombuffer(bytes): torch only wraps writable arrays
                flat = flat.copy()
            src = torch.from_numpy(flat)
            out[: flat.size].copy_(src, non_blocking=src.is_pinned())
            out._pilc_host = src  # type: ignore[attr-defined]  # alive until the copy has run
        if pad:
            out[flat.size:].zero_()
    return out


def as_device_u8(images, dev, stream) -> torch.Tensor:
    if isinstance(images, torch.Tensor):
        t = images.to(device=dev, dtype=torch.uint8, non_blocking=True)
        return t.contiguous()
    return h2d(np.asarray(images, dtype=np.uint8), dev, stream).view(*np.shape(images))


class DeviceCache:
    """Immutable per-device artefacts (coder tables, packed model) keyed by
    content hash. Thread-safe; never evicted within a process."""

    def __init__(self):
        self._d: dict = {}
        self._lock = threading.Lock()

    def get(self, key, dev: torch.device, make):
        k = (key, dev.index)
        with self._lock:
            v = self._d.get(k)
        if v is None:
            v = make()
            with self._lock:
                self._d.setdefault(k, v)
                v = self._d[k]
        return v


CACHE = DeviceCache()
