#!/usr/bin/env python
"""PILC on B200: round-trip (compress + decompress) raw-image throughput.

Workload (BASELINE.json configs[1]): CIFAR10-shaped 32x32x3 synthetic
"smooth" images (trainer data.ts generator, seed = rank), batch 8192 per GPU,
twar-vqvae backend, full model random_weights(ModelConfig(), seed=1)
(K=256, Dc=32, C=32, B=4), M=12, one lane per stream.

One step = compress_batch of the whole batch + decompress_batch of the
resulting blobs. `value` = raw MB (1e6 B) per step x ranks / max-over-ranks
step time, measured with CUDA events on the launching stream with the
images already resident in HBM; L2 is flushed (256 MiB write) before each
timed step. `e2e` is the same metric through the public host API
(pinned host images in, host blobs out, host blobs in, host images out).
Images/patches shard across GPUs with no data-path collective ("weak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

BATCH = 8192
H = W = 32
WORKLOAD = "cifar10-32x32x3-synthetic-smooth, batch 8192/GPU, twar-vqvae full model (K256 Dc32 C32 B4, seed 1), M=12, L=1"
METRIC = "PILC round-trip (compress+decompress) raw-image MB/s"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference)


def _cpu_worker(args):
    seed, count, model_bytes = args
    import numpy as np  # noqa: F401  (threads pinned by the parent's env)

    from oracle import oracle as O
    from paper_2206_05279_b200.synth import smooth_images

    imgs = smooth_images(count, H, W, seed=seed)
    m = O.Model.from_bytes(model_bytes)
    O.compress(imgs[0], m, "twar-vqvae")  # warm tables + C library
    t0 = time.perf_counter()
    nbytes = 0
    for im in imgs:
        blob = O.compress(im, m, "twar-vqvae")
        out = O.decompress(blob, m)
        assert (out == im).all()
        nbytes += im.size
    return nbytes, time.perf_counter() - t0


def cpu_oracle_run(per_proc: int, procs: int, seed0: int = 1000):
    """Times the oracle port on `procs` processes (one core each)."""
    import multiprocessing as mp

    import paper_2206_05279_b200 as pc

    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        os.environ[k] = "1"
    model_bytes = pc.random_weights(seed=1).to_bytes()
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        pool.map(_cpu_worker, [(seed0 + i, 1, model_bytes) for i in range(procs)])  # spawn + warm-up
        res = pool.map(_cpu_worker, [(seed0 + i, per_proc, model_bytes) for i in range(procs)])
    # each worker times its own compress+decompress loop (after its warm-up);
    # the job takes as long as the slowest worker
    wall = max(r[1] for r in res)
    nbytes = sum(r[0] for r in res)
    return nbytes / 1e6 / wall, nbytes, wall


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    procs = len(os.sched_getaffinity(0))
    per_proc = 2
    vals = []
    for _ in range(args.warmup):
        cpu_oracle_run(1, procs)
    t_all = 0.0
    for _ in range(args.steps):
        v, nbytes, wall = cpu_oracle_run(per_proc, procs)
        vals.append(v)
        t_all += wall
    value = statistics.median(vals)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 4),
        "unit": "MB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1000 * t_all / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32/f64 (numpy+BLAS network), int (C coder)",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample_images_per_step": per_proc * procs},
        "cpu_baseline": {
            "value": round(value, 4), "unit": "MB/s", "cores": procs, "kind": "port",
            "sample": f"{per_proc} images/process x {procs} processes per step, oracle/ "
                      "(numpy restatement of pixelcodec + C lanes/predictor), one thread per process",
        },
        "e2e": {"value": round(value, 4), "unit": "MB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# GPU arm


def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2206_05279_b200 as pc
    from paper_2206_05279_b200 import _lib
    from paper_2206_05279_b200 import container as ct
    from paper_2206_05279_b200.synth import smooth_images

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)
    model = pc.random_weights(seed=1)
    cfg = pc.CodecConfig(backend="twar-vqvae")
    imgs = smooth_images(BATCH, H, W, seed=rank)
    raw_bytes = imgs.size
    img_d = torch.from_numpy(imgs).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if ws > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    def step_device():
        out_d, off_d, total = ct._compress_device(img_d, model, cfg, dev, stream)
        offs_host = off_d.cpu().numpy().view(np.uint64)
        results, errors, hdr = ct._decompress_device(out_d, off_d, offs_host, model, dev, stream)
        return out_d, offs_host, results, errors

    # warm-up (+ correctness of the device path, outside the timed region)
    for _ in range(args.warmup):
        out_d, offs_host, results, errors = step_device()
    torch.cuda.synchronize(dev)
    assert not errors, errors
    dec = results[0][1].cpu().numpy()
    lossless = bool(np.array_equal(dec, imgs))
    blob_sizes = np.diff(offs_host.astype(np.int64))
    bpd = float(np.mean(8.0 * blob_sizes / (H * W * 3)))

    # timed region: device-resident inputs
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    _lib.prof_reset(True)
    barrier()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)  # evict L2 between steps (outside the events)
            e0, e1, e2 = ev[k]
            e0.record(stream)
            out_d, off_d, total = ct._compress_device(img_d, model, cfg, dev, stream)
            e1.record(stream)
            offs_host = off_d.cpu().numpy().view(np.uint64)
            ct._decompress_device(out_d, off_d, offs_host, model, dev, stream)
            e2.record(stream)
        barrier()
    launches = _lib.prof_launches()
    prof = _lib.prof_read()
    _lib.prof_reset(False)
    t_c = sum(a.elapsed_time(b) for a, b, _ in ev) / 1000.0
    t_d = sum(b.elapsed_time(c) for _, b, c in ev) / 1000.0
    t_step = (t_c + t_d) / args.steps
    tt = torch.tensor([t_step, t_c / args.steps, t_d / args.steps], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_step, t_cs, t_ds = (float(x) for x in tt.cpu())
    value = raw_bytes * ws / 1e6 / t_step

    # end to end through the public API with host buffers
    e2e_times = []
    h2d = d2h = 0
    barrier()
    for k in range(max(1, args.steps)):
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        buf, off = pc.compress_batch(imgs, model, cfg)
        out = pc.decompress_batch(buf, off, model)
        torch.cuda.synchronize(dev)
        e2e_times.append(time.perf_counter() - t0)
        h2d = imgs.nbytes + buf.nbytes + off.nbytes
        d2h = buf.nbytes + off.nbytes + out.nbytes
    assert np.array_equal(out, imgs)
    te = torch.tensor([statistics.median(e2e_times)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = raw_bytes * ws / 1e6 / float(te.item())

    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
            src = "measured"
        except OSError:
            peaks = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
            src = "fallback"
        dom = max(prof.items(), key=lambda kv: kv[1][1]) if prof else None
        roofline = None
        if dom:
            name, (n, ms, units) = dom
            if name in ("conv_kernel", "argmin_kernel"):
                ach = units / (ms / 1e3) / 1e12
                peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
                roofline = {"kernel": name, "bound": "tensor", "achieved": round(ach, 3), "peak": peak,
                            "unit": "TFLOP/s", "frac": round(ach / peak, 5), "traffic": None,
                            "peak_source": f"{src} bf16 dense (sustained)",
                            "note": "SIMT fp32 path; algorithmic FLOPs = 2*N*Ho*Wo*Co*Ci*k^2 per launch"}
            else:
                roofline = {"kernel": name, "bound": "hbm", "achieved": None, "peak": peaks.get("hbm_gbs"),
                            "unit": "GB/s", "frac": None, "traffic": None}
            tr = _traffic(name)
            if tr is not None and roofline:
                roofline["traffic"] = tr
        stages = {k: {"launches": v[0], "ms_per_step": round(v[1] / args.steps, 4)} for k, v in prof.items()}
        cpu = None
        if ws == 1 and not args.no_cpu:
            procs = len(os.sched_getaffinity(0))
            v, nbytes, wall = cpu_oracle_run(2, procs)
            cpu = {"value": round(v, 4), "unit": "MB/s", "cores": procs, "kind": "port",
                   "sample": f"{2 * procs} CIFAR images ({nbytes} B) compress+decompress, oracle/ numpy+C, "
                             f"{procs} processes x 1 thread, {wall:.1f} s"}
        line = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "MB/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(1000 * t_step, 3),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32 (network, SIMT), f64 (argmin), int (coder/predictor/container)",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "global_batch": BATCH * ws, "image": [H, W, 3],
                       "parallelism": f"shard{ws}", "l2": "flushed (256 MiB write) before each step"},
            "compress_mb_s": round(raw_bytes * ws / 1e6 / t_cs, 3),
            "decompress_mb_s": round(raw_bytes * ws / 1e6 / t_ds, 3),
            "bpd": round(bpd, 4),
            "lossless": lossless,
            "e2e": {"value": round(e2e_value, 3), "unit": "MB/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "roofline": roofline,
            "stages": stages,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return 0


def _traffic(kernel: str):
    """dram bytes per launch for `kernel` from the committed ncu summary."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        return s.get("dram_bytes_per_launch", {}).get(kernel)
    except OSError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
