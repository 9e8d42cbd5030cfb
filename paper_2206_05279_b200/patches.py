"""High-resolution frames as independent patch containers (BASELINE config 4).

The paper evaluates high-resolution images as fixed-size crops
(`PAPER.md:431-432`). A frame is split into a grid of ph x pw patches (the
last row / column may be smaller) and each patch is a self-contained PILC
blob, so a frame compresses and decompresses as one batch of patches (two or
four shape groups) and the patches shard across CTAs and GPUs with no
exchange.
"""

from __future__ import annotations

import numpy as np
import torch

from .container import (CodecConfig, SpeculationMiss, _compress_device, _decompress_device, _resolve_errors, _verify,
                        check_offsets)
from .errors import FormatError, ParameterError
from .device import h2d, pinned, readback, require_device


_SIDE: dict = {}


def _side_stream(dev, i: int) -> torch.cuda.Stream:
    """Per-device side streams for the shape groups of a frame batch."""
    key = (dev.index, i)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(dev)
    return _SIDE[key]


def patch_grid(H: int, W: int, ph: int = 64, pw: int = 64):
    """[(y0, y1, x0, x1)] in raster order."""
    return [(y, min(y + ph, H), x, min(x + pw, W)) for y in range(0, H, ph) for x in range(0, W, pw)]


def split_frame(frame: np.ndarray, ph: int = 64, pw: int = 64) -> list:
    H, W = frame.shape[:2]
    return [np.ascontiguousarray(frame[y0:y1, x0:x1]) for (y0, y1, x0, x1) in patch_grid(H, W, ph, pw)]


def assemble(patches: list, H: int, W: int, ph: int = 64, pw: int = 64) -> np.ndarray:
    out = np.empty((H, W, 3), np.uint8)
    for p, (y0, y1, x0, x1) in zip(patches, patch_grid(H, W, ph, pw)):
        out[y0:y1, x0:x1] = p
    return out


def _groups(H: int, W: int, ph: int, pw: int):
    """Shape groups of the patch grid: (row slice, col slice, n_rows, n_cols,
    patch h, patch w) for the full patches and the ragged bottom row / right
    column / corner (those that exist)."""
    fh, fw = H // ph, W // pw
    hr, wr = H - fh * ph, W - fw * pw
    out = []
    for rows, nr, h in ((slice(0, fh * ph), fh, ph), (slice(fh * ph, H), 1 if hr else 0, hr)):
        for cols, nc, w in ((slice(0, fw * pw), fw, pw), (slice(fw * pw, W), 1 if wr else 0, wr)):
            if nr and nc:
                out.append((rows, cols, nr, nc, h, w))
    return out


def _raster_index(H: int, W: int, ph: int, pw: int):
    """For each group, the raster positions (within a frame) of its patches."""
    fh, fw = H // ph, W // pw
    ncols = fw + (1 if W - fw * pw else 0)
    idx = []
    for rows, cols, nr, nc, h, w in _groups(H, W, ph, pw):
        r0 = 0 if rows.start == 0 else fh
        c0 = 0 if cols.start == 0 else fw
        rr, cc = np.meshgrid(np.arange(r0, r0 + nr), np.arange(c0, c0 + nc), indexing="ij")
        idx.append((rr * ncols + cc).reshape(-1))
    return idx


def _group_patches(frames, g):
    """(F*nr*nc, h, w, 3) patches of one shape group, raster order within it
    (numpy array or device tensor)."""
    rows, cols, nr, nc, h, w = g
    F = frames.shape[0]
    v = frames[:, rows, cols].reshape(F, nr, h, nc, w, 3)
    if isinstance(v, torch.Tensor):
        return v.permute(0, 1, 3, 2, 4, 5).contiguous().reshape(F * nr * nc, h, w, 3)
    return np.ascontiguousarray(v.transpose(0, 1, 3, 2, 4, 5)).reshape(F * nr * nc, h, w, 3)


def _compress_launch(frames_d, model, config, ph, pw, dev, streams, after):
    """Queue every shape group's compress (group i on streams[i], after the
    event `after`) and the D2H of its offsets; returns (parts, pinned
    offsets, events)."""
    F, H, W = frames_d.shape[:3]
    parts, offs_h, evs = [], [], []
    for gi, g in enumerate(_groups(H, W, ph, pw)):
        s = streams[gi]
        s.wait_event(after)
        frames_d.record_stream(s)
        with torch.cuda.stream(s):
            # straight to the device compress: no host read before the next
            # group (or the next request) is queued
            out_d, off_d = _compress_device(_group_patches(frames_d, g), model, config, dev, s)
            h = pinned(off_d.numel() * 8)
            ev = readback(h, off_d.view(torch.uint8), s)
        parts.append((out_d, off_d))
        offs_h.append(h)
        evs.append(ev)
    return parts, offs_h, evs


def _compress_gather(parts, offs_h, F, H, W, ph, pw, stream):
    """Frame-ordered offsets (host, once the groups' offsets are back) and
    the D2H of each (frame, group) run of blobs into its place in one
    page-locked buffer, on `stream`; returns (host tensor, offsets)."""
    ridx = _raster_index(H, W, ph, pw)
    per = sum(len(r) for r in ridx)
    goffs = [h.numpy().view(np.uint64) for h in offs_h]
    sizes = np.zeros((F, per), np.uint64)
    for off, r in zip(goffs, ridx):
        sizes[:, r] = np.diff(off).reshape(F, -1)
    offsets = np.zeros(F * per + 1, np.uint64)
    np.cumsum(sizes.reshape(-1), out=offsets[1:])
    host = pinned(int(offsets[-1]) + 8)
    with torch.cuda.stream(stream):
        for (out_d, _), off, r in zip(parts, goffs, ridx):
            out_d.record_stream(stream)
            k = len(r)
            for f in range(F):
                if bool(np.all(np.diff(r) == 1)):  # one run per frame
                    runs = [(0, k)]
                else:
                    runs = [(j, j + 1) for j in range(k)]
                for j0, j1 in runs:
                    s0, s1 = int(off[f * k + j0]), int(off[f * k + j1])
                    d0 = int(offsets[f * per + r[j0]])
                    host[d0:d0 + s1 - s0].copy_(out_d[s0:s1], non_blocking=True)
    return host, offsets


def compress_frames(frames, model=None, config: CodecConfig = CodecConfig(), ph: int = 64, pw: int = 64,
                    device=None):
    """Frames (F, H, W, 3) -> (buffer, offsets) of F * n_patches blobs, frame
    by frame, raster order within a frame. The frames go to the GPU once; each
    shape group of the patch grid is cut there and compressed as one batch
    (each group on its own stream: their latency-bound coder kernels
    overlap); each (frame, group) run of blobs is copied from the device
    straight to its place in the page-locked result (no host-side
    shuffling)."""
    _check_patch(ph, pw)
    dev = require_device(device)
    stream = torch.cuda.current_stream(dev)
    if isinstance(frames, torch.Tensor):
        frames_d = frames.to(dev)
    else:  # page-locked frames (e.g. ones this package returned) upload asynchronously
        arr = np.asarray(frames, dtype=np.uint8)
        frames_d = h2d(arr, dev, stream).view(arr.shape)
    if frames_d.dim() != 4 or frames_d.shape[-1] != 3 or frames_d.dtype != torch.uint8:
        raise ParameterError("expected uint8 (F, H, W, 3) frames")
    F, H, W = frames_d.shape[:3]
    if F == 0:
        return np.zeros(0, np.uint8), np.zeros(1, np.uint64)
    ev_in = torch.cuda.Event()
    ev_in.record(stream)
    n_groups = len(_groups(H, W, ph, pw))
    streams = [stream] + [_side_stream(dev, i) for i in range(1, n_groups)]
    parts, offs_h, evs = _compress_launch(frames_d, model, config, ph, pw, dev, streams, ev_in)
    for ev in evs:
        ev.synchronize()
        stream.wait_event(ev)
    host, offsets = _compress_gather(parts, offs_h, F, H, W, ph, pw, stream)
    stream.synchronize()
    return host.numpy()[: int(offsets[-1])], offsets


def _check_patch(ph: int, pw: int) -> None:
    if int(ph) < 1 or int(pw) < 1:
        raise ParameterError("patch sizes must be at least 1")


def _check_frame_offsets(buffer, offsets, n_frames, H, W, ph, pw):
    _check_patch(ph, pw)
    if int(n_frames) < 0 or int(H) < 1 or int(W) < 1:
        raise ParameterError("expected n_frames >= 0 frames of at least 1 x 1 pixels")
    buffer = np.asarray(buffer, dtype=np.uint8)
    offsets = check_offsets(offsets)
    per = sum(len(r) for r in _raster_index(H, W, ph, pw))
    if offsets.size != n_frames * per + 1 or int(offsets[-1]) > buffer.size:
        raise FormatError(f"expected {n_frames * per + 1} blob offsets within the buffer for {n_frames} frame(s) of "
                          f"{per} patches")
    return buffer, offsets


def _decode_launch(buf_d, offsets, F, H, W, model, ph, pw, dev, streams, after):
    """Queue every shape group's decode (group i on streams[i], after the
    event `after`): its blobs gathered on the device, then the speculative
    decode; no host read. Returns the launched groups."""
    groups = _groups(H, W, ph, pw)
    ridx = _raster_index(H, W, ph, pw)
    per = sum(len(r) for r in ridx)
    launched = []
    for gi, (g, r) in enumerate(zip(groups, ridx)):
        k = len(r)
        s = streams[gi]
        s.wait_event(after)
        buf_d.record_stream(s)
        pos = (np.arange(F)[:, None] * per + r[None, :]).reshape(-1)
        lens = offsets[pos + 1] - offsets[pos]
        goff_h = pinned(8 * (F * k + 1))
        goff = goff_h.numpy().view(np.uint64)
        goff[0] = 0
        np.cumsum(lens, out=goff[1:])
        with torch.cuda.stream(s):
            gbuf = torch.empty(int(goff[-1]) + 16, dtype=torch.uint8, device=dev)
            gbuf[int(goff[-1]):].zero_()
            contiguous = bool(np.all(np.diff(r) == 1))
            for f in range(F):
                runs = [(0, k)] if contiguous else [(j, j + 1) for j in range(k)]
                for j0, j1 in runs:
                    s0, s1 = int(offsets[f * per + r[j0]]), int(offsets[f * per + r[j1 - 1] + 1])
                    d0 = int(goff[f * k + j0])
                    gbuf[d0:d0 + s1 - s0].copy_(buf_d[s0:s1], non_blocking=True)
            goff_d = torch.empty(F * k + 1, dtype=torch.int64, device=dev)
            goff_d.view(torch.uint8).copy_(goff_h, non_blocking=True)
            res = _decompress_device(gbuf, goff_d, F * k, model, dev, s)
            ev_dec = torch.cuda.Event()  # this group's decode, recorded now (later work may follow on s)
            ev_dec.record(s)
        launched.append((g, s, gbuf, goff_d, goff_h, res, k, ev_dec))
    return launched


def _assemble(g, img, frames_d, stream):
    """The group's decoded patches into their places in frames_d, on stream."""
    rows, cols, nr, nc, h, w = g
    F = frames_d.shape[0]
    with torch.cuda.stream(stream):
        img.record_stream(stream)
        frames_d.record_stream(stream)
        frames_d[:, rows, cols] = img.reshape(F, nr, nc, h, w, 3).permute(0, 1, 3, 2, 4, 5).reshape(
            F, nr * h, nc * w, 3)


def _decode_finish(launched, frames_d, model, dev, out_stream=None, assembled=None):
    """Check each launched group (blocks on its summary), raise its first
    error, and write its patches into frames_d (on the group's stream, or on
    out_stream after the group's decode when given). `assembled`: per group
    the event recorded right after its patches were written into frames_d
    on its stream at launch (redone there only when the speculated batch
    layout missed). Returns the events the frames are complete after."""
    F = frames_d.shape[0]
    evs = []
    for gi, (g, s, gbuf, goff_d, goff_h, (results, errors, hdr), k, done) in enumerate(launched):
        redo = False
        with torch.cuda.stream(s):
            try:
                _verify(results)
            except SpeculationMiss:
                results, errors, hdr = _decompress_device(gbuf, goff_d, F * k, model, dev, s, speculate=False)
                redo = True
                done = torch.cuda.Event()
                done.record(s)
        ws = out_stream if out_stream is not None else s
        with torch.cuda.stream(ws):
            ws.wait_event(done)
            errors = _resolve_errors(results, errors, hdr)
            if errors:
                raise errors[min(errors)]
        if assembled is not None and assembled[gi] is not None and not redo:
            done = assembled[gi]
        else:
            _assemble(g, results[0][1], frames_d, s if assembled is not None else ws)
            done = torch.cuda.Event()
            done.record(s if assembled is not None else ws)
        evs.append(done)
    return evs


def decompress_frames(buffer, offsets, n_frames: int, H: int, W: int, model=None, ph: int = 64, pw: int = 64,
                      device=None):
    """Inverse of compress_frames: the blob buffer goes to the GPU once, each
    shape group is gathered there (device copies of its (frame, group) runs)
    and decoded as one batch on its own stream (the groups' latency-bound
    coder and wavefront kernels overlap; every group is queued before any
    host read), written into device frames, and the frames come back in one
    copy."""
    dev = require_device(device)
    stream = torch.cuda.current_stream(dev)
    buffer, offsets = _check_frame_offsets(buffer, offsets, n_frames, H, W, ph, pw)
    F = n_frames
    if F == 0:
        return np.zeros((0, H, W, 3), np.uint8)
    buf_d = h2d(buffer[: int(offsets[-1])], dev, stream)
    frames_d = torch.empty((F, H, W, 3), dtype=torch.uint8, device=dev)
    ev_buf = torch.cuda.Event()
    ev_buf.record(stream)
    n_groups = len(_groups(H, W, ph, pw))
    streams = [stream] + [_side_stream(dev, i) for i in range(1, n_groups)]
    launched = _decode_launch(buf_d, offsets, F, H, W, model, ph, pw, dev, streams, ev_buf)
    for ev in _decode_finish(launched, frames_d, model, dev):
        stream.wait_event(ev)
    host = pinned(frames_d.numel())
    with torch.cuda.stream(stream):
        host.copy_(frames_d.view(-1), non_blocking=True)
    stream.synchronize()
    return host.numpy().reshape(F, H, W, 3)
