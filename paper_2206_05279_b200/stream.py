"""Pipelined batch codec on one GPU (a serving-side extension; pixelcodec
has no counterpart).

`compress_batch` / `decompress_batch` are synchronous: each call uploads its
inputs, runs its kernels and downloads its results in series, so the PCIe
transfers (~2 ms per CIFAR-8192 round trip) add to the kernels (~5.5 ms).
StreamCodec keeps three CUDA streams -- uploads, kernels, downloads -- and a
completion thread, so the upload of request k + 1 and the download of
request k - 1 run under the kernels of request k. Requests return futures;
each request's bytes are exactly what the synchronous calls return (the
same device functions, and every per-image result is independent of batch
composition).

    codec = StreamCodec(model, CodecConfig(backend="twar-vqvae"))
    f = codec.compress(images)            # Future[(buffer, offsets)]
    g = codec.decompress(*f.result())     # Future[images]
    images_back = g.result()

Frames split into patch containers (patches.compress_frames /
decompress_frames, BASELINE config 4) go through compress_frames /
decompress_frames the same way.

Kernels of different requests run in submission order on the one kernel
stream (never concurrently: the persistent-grid kernels would only slow
each other down).
"""

from __future__ import annotations

from concurrent.futures import Future, ThreadPoolExecutor

import numpy as np
import torch

from .container import (CodecConfig, SpeculationMiss, _compress_device, _decompress_device, _resolve_errors,
                        _verify, check_offsets)
from .device import pinned, readback, require_device
from .errors import FormatError, ParameterError
from . import patches as _pt


class StreamCodec:
    def __init__(self, model=None, config: CodecConfig = CodecConfig(), device=None):
        self.dev = require_device(device)
        self.model, self.config = model, config
        self.up = torch.cuda.Stream(self.dev)
        self.kern = torch.cuda.Stream(self.dev)
        self.down = torch.cuda.Stream(self.dev)
        self._done = ThreadPoolExecutor(max_workers=1, thread_name_prefix="pilc-stream")  # FIFO completion

    def close(self) -> None:
        self._done.shutdown(wait=True)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- helpers ------------------------------------------------------------

    def _upload(self, host: np.ndarray, nbytes_pad: int = 0) -> tuple:
        """host -> new device tensor on the upload stream; returns (tensor, event,
        keep-alive). Page-locked sources copy asynchronously."""
        flat = np.ascontiguousarray(host).view(np.uint8).reshape(-1)
        with torch.cuda.device(self.dev):
            d = torch.empty(flat.size + nbytes_pad, dtype=torch.uint8, device=self.dev)
        d.record_stream(self.up)
        d.record_stream(self.kern)
        src = torch.from_numpy(flat if flat.flags.writeable else flat.copy())
        with torch.cuda.stream(self.up):
            if flat.size:
                d[: flat.size].copy_(src, non_blocking=src.is_pinned())
            if nbytes_pad:
                d[flat.size:].zero_()
            ev = torch.cuda.Event()
            ev.record(self.up)
        return d, ev, src

    def _download(self, src: torch.Tensor, after: torch.cuda.Event, nbytes: int) -> np.ndarray:
        """device bytes -> page-locked host, on the download stream (completion thread)."""
        host = pinned(nbytes + 8)
        src.record_stream(self.down)
        with torch.cuda.stream(self.down):
            self.down.wait_event(after)
            if nbytes:
                host[:nbytes].copy_(src.reshape(-1)[:nbytes], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.down)
        ev.synchronize()
        return host.numpy()[:nbytes]

    # -- compress -----------------------------------------------------------

    def compress(self, images) -> Future:
        arr = np.asarray(images)
        if arr.dtype != np.uint8 or arr.ndim != 4 or arr.shape[-1] != 3 or arr.shape[1] < 1 or arr.shape[2] < 1:
            raise ParameterError("expected a uint8 (N, H, W, 3) array")
        n = arr.shape[0]
        if n == 0:
            f: Future = Future()
            f.set_result((np.zeros(0, np.uint8), np.zeros(1, np.uint64)))
            return f
        img_d, ev_up, keep = self._upload(arr)
        self.kern.wait_event(ev_up)
        with torch.cuda.stream(self.kern):
            out_d, off_d = _compress_device(img_d.view(arr.shape), self.model, self.config, self.dev, self.kern)
            offs_h = pinned(8 * (n + 1))
            ev_k = readback(offs_h, off_d.view(torch.uint8), self.kern)  # after the kernels; off the kernel stream

        def finish():
            ev_k.synchronize()
            offs = offs_h.numpy().view(np.uint64).copy()
            buf = self._download(out_d, ev_k, int(offs[-1]))
            assert keep is not None  # the pageable / pinned source stays alive until here
            return buf, offs

        return self._done.submit(finish)

    # -- decompress ---------------------------------------------------------

    def decompress(self, buffer, offsets) -> Future:
        offs = check_offsets(offsets)
        buf_host = np.frombuffer(buffer, np.uint8) if isinstance(buffer, (bytes, bytearray, memoryview)) \
            else np.ascontiguousarray(buffer, dtype=np.uint8)
        n = offs.size - 1
        if int(offs[-1]) > buf_host.size:
            raise FormatError("container truncated")
        if n <= 0:
            f: Future = Future()
            f.set_result(np.zeros((0, 1, 1, 3), np.uint8))
            return f
        buf_d, ev_b, keep_b = self._upload(buf_host[: int(offs[-1])], nbytes_pad=16)
        off_d, ev_o, keep_o = self._upload(offs.view(np.uint8))
        self.kern.wait_event(ev_b)
        self.kern.wait_event(ev_o)
        with torch.cuda.stream(self.kern):
            res = _decompress_device(buf_d, off_d.view(torch.int64), n, self.model, self.dev, self.kern,
                                     buf_host, offs)
            ev_k = torch.cuda.Event()
            ev_k.record(self.kern)

        def finish():
            results, errors, hdr = res
            ev_k.synchronize()
            done = ev_k
            try:
                _verify(results)
            except SpeculationMiss:  # another batch layout ran last: redo this one, non-speculatively
                with torch.cuda.stream(self.kern):
                    results, errors, hdr = _decompress_device(buf_d, off_d.view(torch.int64), n, self.model,
                                                              self.dev, self.kern, buf_host, offs,
                                                              speculate=False)
                    done = torch.cuda.Event()
                    done.record(self.kern)
                done.synchronize()
            with torch.cuda.stream(self.down):  # status reads: not on the kernel stream
                self.down.wait_event(done)
                errors = _resolve_errors(results, errors, hdr)
            if errors:
                raise errors[min(errors)]
            assert keep_b is not None and keep_o is not None
            if len(results) == 1 and np.asarray(results[0][0]).size == n:
                img = results[0][1]
                return self._download(img, done, img.numel()).reshape(tuple(img.shape))
            imgs: list = [None] * n
            for ids, img, *_ in results:
                arr = self._download(img, done, img.numel()).reshape(tuple(img.shape))
                for j, i in enumerate(np.asarray(ids)):
                    imgs[int(i)] = arr[j]
            return imgs

        return self._done.submit(finish)

    # -- frames as patch containers (patches.py) ----------------------------

    def compress_frames(self, frames, ph: int = 64, pw: int = 64) -> Future:
        """Future[(buffer, offsets)] of patches.compress_frames(frames, ...)."""
        arr = np.asarray(frames)
        if arr.dtype != np.uint8 or arr.ndim != 4 or arr.shape[-1] != 3 or arr.shape[1] < 1 or arr.shape[2] < 1:
            raise ParameterError("expected uint8 (F, H, W, 3) frames")
        _pt._check_patch(ph, pw)
        F, H, W = arr.shape[:3]
        if F == 0:
            f: Future = Future()
            f.set_result((np.zeros(0, np.uint8), np.zeros(1, np.uint64)))
            return f
        fr_d, ev_up, keep = self._upload(arr)
        n_groups = len(_pt._groups(H, W, ph, pw))
        parts, offs_h, evs = _pt._compress_launch(fr_d.view(arr.shape), self.model, self.config, ph, pw, self.dev,
                                                  [self.kern] * n_groups, ev_up)

        def finish():
            for ev in evs:
                ev.synchronize()
                self.down.wait_event(ev)
            host, offsets = _pt._compress_gather(parts, offs_h, F, H, W, ph, pw, self.down)
            done = torch.cuda.Event()
            done.record(self.down)
            done.synchronize()
            assert keep is not None
            return host.numpy()[: int(offsets[-1])], offsets

        return self._done.submit(finish)

    def decompress_frames(self, buffer, offsets, n_frames: int, H: int, W: int, ph: int = 64,
                          pw: int = 64) -> Future:
        """Future[frames] of patches.decompress_frames(buffer, offsets, ...)."""
        buf_host, offs = _pt._check_frame_offsets(buffer, offsets, n_frames, H, W, ph, pw)
        if n_frames == 0:
            f: Future = Future()
            f.set_result(np.zeros((0, H, W, 3), np.uint8))
            return f
        buf_d, ev_b, keep_b = self._upload(buf_host[: int(offs[-1])], nbytes_pad=16)
        with torch.cuda.device(self.dev):
            frames_d = torch.empty((n_frames, H, W, 3), dtype=torch.uint8, device=self.dev)
        n_groups = len(_pt._groups(H, W, ph, pw))
        launched = _pt._decode_launch(buf_d, offs, n_frames, H, W, self.model, ph, pw, self.dev,
                                      [self.kern] * n_groups, ev_b)
        # the patches into the frames right behind each group's decode, on the
        # kernel stream (speculatively: redone there if the batch layout
        # missed); a copy kernel on another stream would share the SMs with
        # the next request's persistent kernels
        assembled = []
        for g, s, _gb, _go, _gh, res, _k, _ev in launched:
            ev = None
            _r, _c, nr, nc, h, w = g
            # only when the speculated layout has this group's shape (else the
            # speculation misses and finish() redoes decode + assembly)
            if res[0] and tuple(res[0][0][1].shape) == (n_frames * nr * nc, h, w, 3):
                _pt._assemble(g, res[0][0][1], frames_d, s)
                ev = torch.cuda.Event()
                ev.record(s)
            assembled.append(ev)

        def finish():
            evs = _pt._decode_finish(launched, frames_d, self.model, self.dev, out_stream=self.down,
                                     assembled=assembled)
            ev = evs[-1] if evs else torch.cuda.Event()
            if not evs:
                ev.record(self.down)
            assert keep_b is not None
            return self._download(frames_d, ev, frames_d.numel()).reshape(n_frames, H, W, 3)

        return self._done.submit(finish)
