"""Benchmark rows in the reference's report format, measured on the GPU.

Mirrors `pixelcodec.report` (report.py:24-104): `run_bench(...)` returns
rows {phase, lanes, bytes, seconds, mb_per_s} and `write_rows` emits them as
JSON lines. Phases (the reference's, run on the B200 path):

  coder-encode-fast / coder-decode-fast   GPU lanes (pilc_rans_encode /
      pilc_rans_decode) over `lane_counts`, symbols from the reference's
      Table-6 generator (`_bench_symbols`, report.py:34-44), device-resident,
      CUDA-event timed; the decode is checked against the input
  model-inference        encode_to_indices + decode_to_params of one image
  ar-decode-parallel     predictor.decode_parallel of one image
  roundtrip-batch        compress_batch + decompress_batch of `batch` images
      (host arrays in and out), the codec's public batch API

The reference coder (`coder-*-ref`, a pure-Python rANS) and the sequential
predictor decode have no GPU counterpart and are not timed; figures
(render_figures) need matplotlib, which this image lacks.

    python -m paper_2206_05279_b200.report [--symbols N] [--batch B]
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np
import torch

from . import _lib, logistic, predictor, tables, vqvae
from .device import ptr, require_device, sptr
from .weights import random_weights


def _row(phase: str, lanes: int, nbytes: int, seconds: float) -> dict:
    """report.py:24-31: bytes are raw symbols / pixels, MB = 1e6 B."""
    return {
        "phase": phase,
        "lanes": lanes,
        "bytes": nbytes,
        "seconds": round(seconds, 6),
        "mb_per_s": round(nbytes / 1e6 / seconds, 3) if seconds > 0 else float("inf"),
    }


def _bench_symbols(M: int, grid: logistic.ScaleGrid, n: int, seed: int = 0):
    """report.py:34-44: d uniform over the grid, symbol ~ PMF_d."""
    rng = np.random.default_rng(seed)
    pmfs = logistic.residual_distributions(grid, M)
    d = rng.integers(0, grid.D, n).astype(np.uint16)
    syms = np.empty(n, dtype=np.uint8)
    for i, pmf in enumerate(pmfs):
        sel = d == i
        p = pmf.P.astype(np.float64) / (1 << M)
        syms[sel] = rng.choice(256, int(sel.sum()), p=p)
    return syms, d, pmfs


def _timed(fn, stream, reps: int) -> float:
    """Median seconds of `reps` CUDA-event-timed calls after one warm-up."""
    fn()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        out.append(a.elapsed_time(b) / 1e3)
    return float(np.median(out))


def run_bench(M: int = 12, D: int = 8, lane_counts=(1, 2, 4, 8), n_symbols: int = 1 << 20,
              image_hw: tuple[int, int] = (96, 96), seed: int = 0, batch: int = 1024, reps: int = 5) -> list[dict]:
    dev = require_device()
    stream = torch.cuda.current_stream(dev)
    grid = logistic.default_grid(D)
    syms, d, pmfs = _bench_symbols(M, grid, n_symbols, seed)
    enc, dec = tables.build_tables(pmfs, M)
    rows = []
    s_d = torch.from_numpy(syms).to(dev)
    d_d = torch.from_numpy(d.astype(np.uint8)).to(dev)
    n = syms.size
    for L in lane_counts:
        box = {}

        def encode():
            box["e"] = tables.encode_lanes_device(s_d, 1, n, L, enc, dev, stream, dsched=d_d)

        te = _timed(encode, stream, reps)
        scr, cap, nb, st = box["e"]
        lane_off = torch.arange(L, dtype=torch.int64, device=dev) * (cap * 4)
        out = torch.empty(n, dtype=torch.uint8, device=dev)
        lstat = torch.zeros(L, dtype=torch.uint8, device=dev)

        def decode():
            _lib.call("pilc_rans_decode", ptr(scr), ptr(lane_off), ptr(nb), ptr(st), ptr(d_d), None, 1, n, L,
                      ptr(dec.device_words(dev)), dec.D, M, None, ptr(out), ptr(lstat), sptr(stream))

        td = _timed(decode, stream, reps)
        if not torch.equal(out, s_d) or int(lstat.max()) != 0:
            raise AssertionError("bench round trip failed")
        rows.append(_row("coder-encode-fast", L, n, te))
        rows.append(_row("coder-decode-fast", L, n, td))

    # model inference and predictor phases on one synthetic image (report.py:84-103)
    rng = np.random.default_rng(seed)
    H, W = image_hw
    img = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
    weights = random_weights(seed=seed)
    idx = vqvae.encode_to_indices(img, weights)  # warm-up (model upload, workspace)
    vqvae.decode_to_params(idx, weights, (H, W))
    t0 = time.perf_counter()
    idx = vqvae.encode_to_indices(img, weights)
    vqvae.decode_to_params(idx, weights, (H, W))
    rows.append(_row("model-inference", 1, img.size, time.perf_counter() - t0))

    params = predictor.default_params()
    res = predictor.forward_residual(img, params)
    predictor.decode_parallel(res, params)
    t0 = time.perf_counter()
    predictor.decode_parallel(res, params)
    rows.append(_row("ar-decode-parallel", 1, img.size, time.perf_counter() - t0))

    if batch:
        from . import container
        from .synth import smooth_images

        imgs = smooth_images(batch, 32, 32, seed=seed)
        cfg = container.CodecConfig(backend="twar-vqvae")
        buf, off = container.compress_batch(imgs, weights, cfg)
        container.decompress_batch(buf, off, weights)
        t0 = time.perf_counter()
        buf, off = container.compress_batch(imgs, weights, cfg)
        back = container.decompress_batch(buf, off, weights)
        rows.append(_row("roundtrip-batch", 1, imgs.size, time.perf_counter() - t0))
        if not np.array_equal(back, imgs):
            raise AssertionError("batch round trip failed")
    return rows


def write_rows(rows: list[dict], stream) -> None:
    """report.py:107-109."""
    for row in rows:
        stream.write(json.dumps(row) + "\n")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="GPU benchmark rows in the reference report format")
    ap.add_argument("--symbols", type=int, default=1 << 20)
    ap.add_argument("--lanes", default="1,2,4,8,1024,65536")
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args(argv)
    rows = run_bench(lane_counts=tuple(int(x) for x in a.lanes.split(",")), n_symbols=a.symbols, seed=a.seed,
                     batch=a.batch)
    write_rows(rows, sys.stdout)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
