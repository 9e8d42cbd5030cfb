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
# BASELINE.json configs: [1] is the default line; the others are --workload
WORKLOADS = {
    "cifar": dict(H=32, W=32, N=8192, desc=WORKLOAD),
    "in64": dict(H=64, W=64, N=4096, desc="imagenet64-64x64x3-synthetic-smooth, batch 4096/GPU, twar-vqvae full "
                                          "model (seed 1), M=12, L=1"),
    "1080p": dict(H=1080, W=1920, N=8, desc="1920x1080x3 synthetic-smooth frames, 8/GPU, split into 64x64 patch "
                                           "containers (510/frame), twar-vqvae full model (seed 1), M=12, L=1"),
}


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


def bench_model(name: str):
    """--weights: `random` = random_weights(ModelConfig(), seed=1) (the
    BASELINE config); `trained` = tests/golden/trained.pilw, the same
    architecture briefly trained by the trainer port (one-code histogram)."""
    import paper_2206_05279_b200 as pc

    if name == "trained":
        return pc.ModelWeights.load(os.path.join(REPO, "tests", "golden", "trained.pilw"))
    return pc.random_weights(seed=1)


def cpu_oracle_run(per_proc: int, procs: int, seed0: int = 1000, weights: str = "random"):
    """Times the oracle port on `procs` processes (one core each)."""
    import multiprocessing as mp

    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        os.environ[k] = "1"
    model_bytes = bench_model(weights).to_bytes()
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        pool.map(_cpu_worker, [(seed0 + i, 1, model_bytes) for i in range(procs)])  # spawn + warm-up
        res = pool.map(_cpu_worker, [(seed0 + i, per_proc, model_bytes) for i in range(procs)])
    # each worker times its own compress+decompress loop (after its warm-up);
    # the job takes as long as the slowest worker
    wall = max(r[1] for r in res)
    nbytes = sum(r[0] for r in res)
    return nbytes / 1e6 / wall, nbytes, wall


def cpu_sample_size(procs: int, target_s: float, weights: str = "random") -> int:
    """Images per process so one oracle run lasts about target_s seconds."""
    _, _, wall = cpu_oracle_run(2, procs, weights=weights)
    return max(2, int(round(2 * target_s / max(wall, 1e-3))))


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    procs = len(os.sched_getaffinity(0))
    # each step is a bounded sample; the whole run stays within ~3 minutes
    per_proc = cpu_sample_size(procs, max(1.0, min(10.0, 150.0 / (args.steps + args.warmup))), args.weights)
    vals = []
    for _ in range(args.warmup):
        cpu_oracle_run(2, procs, weights=args.weights)
    t_all = 0.0
    for _ in range(args.steps):
        v, nbytes, wall = cpu_oracle_run(per_proc, procs, weights=args.weights)
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
        "config": {"workload": WORKLOAD, "weights": args.weights, "sample_images_per_step": per_proc * procs},
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
    """SM clock and throttle reasons sampled on a thread while the timed
    region runs (NVML, ~5 ms period; nvidia-smi as fallback). One sample is
    taken on entry and one on exit, so even a short region has samples."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nv = None
        try:  # NVML polls in microseconds; nvidia-smi takes ~0.1 s per sample
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            bits = (pynvml.nvmlClocksThrottleReasonHwSlowdown, pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                    pynvml.nvmlClocksThrottleReasonSwThermalSlowdown, pynvml.nvmlClocksThrottleReasonSwPowerCap)
            self._nv = (pynvml, h, bits, pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nv = None

    def _sample(self):
        if self._nv is not None:
            pynvml, h, bits, mx = self._nv
            try:
                r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append([str(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)), str(mx)]
                                    + ["Active" if r & b else "Not Active" for b in bits])
                return
            except Exception:
                pass
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            if out:
                self.samples.append([x.strip() for x in out.split(",")])
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.005 if self._nv is not None else 0.2)

    def __enter__(self):
        self._sample()
        self._t.start()
        return self

    def __exit__(self, *a):
        self._sample()
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
    model = bench_model(args.weights)
    cfg = pc.CodecConfig(backend="twar-vqvae")
    wl = WORKLOADS[args.workload]
    if args.workload == "1080p":
        from paper_2206_05279_b200 import patches as pt
        frames = np.stack([smooth_images(1, wl["H"], wl["W"], seed=1000 * rank + f)[0] for f in range(wl["N"])])
        plist = [p for f in frames for p in pt.split_frame(f)]
        shapes = sorted({p.shape for p in plist})
        groups_h = [np.stack([p for p in plist if p.shape == sh]) for sh in shapes]
        imgs = frames
    else:
        imgs = smooth_images(wl["N"], wl["H"], wl["W"], seed=rank)
        groups_h = [imgs]
    raw_bytes = imgs.size
    groups_d = [torch.from_numpy(g).to(dev) for g in groups_h]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if ws > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(dev)

    def step_device():
        outs = []
        for img_d in groups_d:
            out_d, off_d = ct._compress_device(img_d, model, cfg, dev, stream)
            results, errors, hdr = ct._decompress_device(out_d, off_d, img_d.shape[0], model, dev, stream)
            ct._verify(results)  # the speculated summary matched (raises otherwise)
            outs.append((off_d.cpu().numpy().view(np.uint64), results, errors))
        return outs

    # warm-up (+ correctness of the device path, outside the timed region)
    for _ in range(max(1, args.warmup)):
        outs = step_device()
    torch.cuda.synchronize(dev)
    lossless = True
    bits = 0.0
    for g, (offs_host, results, errors) in zip(groups_h, outs):
        assert not errors, errors
        lossless &= bool(np.array_equal(results[0][1].cpu().numpy(), g))
        bits += 8.0 * float(np.diff(offs_host.astype(np.int64)).sum())
    bpd = bits / float(sum(g.size for g in groups_h))

    # timed region: device-resident inputs. Pass 1 measures the step with no
    # per-launch instrumentation (counted launches only); pass 2 repeats the
    # same K steps with a CUDA event pair around every launch for the stage
    # table and the roofline (the events themselves cost ~3% of the step).
    def timed(profile: bool):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
               torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        _lib.prof_reset(profile)
        barrier()
        with ClockSampler(local) as clk:
            for k in range(args.steps):
                flush.fill_(k & 0xFF)  # evict L2 between steps (outside the events)
                e0, e1, e2 = ev[k]
                e0.record(stream)
                packed = [ct._compress_device(img_d, model, cfg, dev, stream) for img_d in groups_d]
                e1.record(stream)
                for (out_d, off_d), img_d in zip(packed, groups_d):
                    ct._decompress_device(out_d, off_d, img_d.shape[0], model, dev, stream)
                e2.record(stream)
            barrier()
        launches = _lib.prof_launches()
        prof = _lib.prof_read() if profile else {}
        _lib.prof_reset(False)
        t_c = sum(a.elapsed_time(b) for a, b, _ in ev) / 1000.0
        t_d = sum(b.elapsed_time(c) for _, b, c in ev) / 1000.0
        return clk, launches, prof, t_c, t_d

    clk, launches, _, t_c, t_d = timed(False)
    _, _, prof, _, _ = timed(True)
    t_step = (t_c + t_d) / args.steps
    tt = torch.tensor([t_step, t_c / args.steps, t_d / args.steps], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_step, t_cs, t_ds = (float(x) for x in tt.cpu())
    value = raw_bytes * ws / 1e6 / t_step

    # end to end through the public API with host buffers (after the same
    # number of untimed warm-up calls as the device loop: the first calls
    # page-lock their host buffers)
    e2e_times, e2e_c, e2e_d = [], [], []
    h2d = d2h = 0
    lat = None
    for _ in range(max(1, args.warmup)):
        if args.workload == "1080p":
            buf, off = pt.compress_frames(imgs, model, cfg)
            out = pt.decompress_frames(buf, off, len(imgs), wl["H"], wl["W"], model)
        else:
            buf, off = pc.compress_batch(imgs, model, cfg)
            out = pc.decompress_batch(buf, off, model)
    barrier()
    for k in range(max(1, args.steps)):
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        if args.workload == "1080p":
            buf, off = pt.compress_frames(imgs, model, cfg)
            torch.cuda.synchronize(dev)
            t1 = time.perf_counter()
            out = pt.decompress_frames(buf, off, len(imgs), wl["H"], wl["W"], model)
        else:
            buf, off = pc.compress_batch(imgs, model, cfg)
            torch.cuda.synchronize(dev)
            t1 = time.perf_counter()
            out = pc.decompress_batch(buf, off, model)
        torch.cuda.synchronize(dev)
        t2 = time.perf_counter()
        e2e_times.append(t2 - t0)
        e2e_c.append(t1 - t0)
        e2e_d.append(t2 - t1)
        h2d = imgs.nbytes + buf.nbytes + off.nbytes
        d2h = buf.nbytes + off.nbytes + out.nbytes
    assert np.array_equal(out, imgs)
    if args.workload == "1080p":
        # single-frame decompress latency: blobs in host RAM -> frame in RAM
        per = len(pt.patch_grid(wl["H"], wl["W"]))
        fb = buf[: int(off[per])]
        fo = off[: per + 1]
        ts = []
        for _ in range(5):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            fr = pt.decompress_frames(fb, fo, 1, wl["H"], wl["W"], model)
            ts.append(time.perf_counter() - t0)
        assert np.array_equal(fr[0], imgs[0])
        lat = round(1000 * statistics.median(ts), 3)
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
        notes = {
            "tc3_conv_kernel": "encoder block convs, 3-product fp16 split on tcgen05 kind::f16 (per K=16 step A_hi x [W_hi|W_lo] "
                               "N=64 + A_lo x W_hi N=32, fp32 TMEM); algorithmic FLOPs = 2*N*H*W*Cout*Cin*9 per launch "
                               "(MMA FLOPs issued = 3x that)",
            "tc_conv_kernel": "bf16 tcgen05 decoder convs; algorithmic FLOPs = 2*N*H*W*Cout*Cin*9 per launch",
            "enc_front_kernel": "encoder stem + stride-2 down, both 3-product fp16 MMAs (down over the space-to-depth stem); "
                                "algorithmic FLOPs = 2*N*(4*gh*gw*32*27 + gh*gw*32*32*9)",
            "conv_kernel": "fp32 SIMT convs (non-default model shapes); algorithmic FLOPs = 2*N*Ho*Wo*Cout*Cin*k^2 per launch",
            "tc3_block_kernel": "one encoder residual block per launch (conv1 + conv2, intermediate in shared memory), "
                                "3-product fp16 split on tcgen05 kind::f16; algorithmic FLOPs = 2 convs x 2*N*H*W*32*32*9 "
                                "(MMA FLOPs issued = 3x that)",
            "dec_trunk_kernel": "decoder trunk (gather + all 2B bf16 block convs, activations in shared memory, G images per "
                                "CTA iteration); algorithmic FLOPs = 2B x 2*N*gh*gw*32*32*9",
            "argmin_kernel": "codebook distance GEMM (3xTF32 tcgen05) + proven-margin screen + exact f64 rescore (3*n*K*Dc FLOPs)",
        }
        if dom:
            name, (n, ms, units) = dom
            if name in notes:
                ach = units / (ms / 1e3) / 1e12
                peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
                roofline = {"kernel": name, "bound": "tensor", "achieved": round(ach, 3), "peak": peak,
                            "unit": "TFLOP/s", "frac": round(ach / peak, 5), "traffic": None,
                            "launches_per_step": n / args.steps, "ms_per_launch": round(ms / n, 4),
                            "timing": "per-launch CUDA events over a second pass of the K timed steps",
                            "peak_source": f"{src} bf16 dense, sustained (kind::f16 fp16/bf16 MMAs run at this rate)",
                            "note": notes[name]}
            else:
                gbs = units / (ms / 1e3) / 1e9
                roofline = {"kernel": name, "bound": "hbm", "achieved": round(gbs, 2), "peak": peaks.get("hbm_gbs"),
                            "unit": "GB/s", "frac": round(gbs / peaks.get("hbm_gbs"), 5), "traffic": None}
            # attainable rate for these MMA shapes: SS-mode tcgen05 MMAs (M=128,
            # K=16) cost max(44 cycles, operand bytes / 128 B/cycle) each on this
            # B200 (tools/micro/mma_rate.cu: N=16/32 44, N=64 48, N=128 64), so
            # N=32-output convs cannot approach the dense peak. Cycles per
            # 128-row K=16 step (algorithmic 2*128*32*16 FLOP): bf16 convs 44;
            # the 3-product fp16 encoder (N=64 + N=32 MMAs) 92.
            floor_cyc = {"tc_conv_kernel": 44.0, "dec_trunk_kernel": 44.0, "tc3_block_kernel": 92.0,
                         "tc3_conv_kernel": 92.0}.get(name)
            if floor_cyc and roofline and roofline.get("bound") == "tensor":
                sm = peaks.get("sm_count", 148)
                mhz = clk.summary().get("sm_mhz") or 1965.0
                att = 2.0 * 128 * 32 * 16 / floor_cyc * sm * mhz * 1e6 / 1e12
                roofline["mma_floor"] = {"peak": round(att, 1), "unit": "TFLOP/s",
                                         "frac": round(roofline["achieved"] / att, 4),
                                         "note": f"{floor_cyc:.0f} cycles per 128x32x16 step (measured per-MMA floor), "
                                                 f"{sm} SMs at the sampled SM clock; ignores the padded border rows"}
            tr = _traffic(name)
            if tr is not None and roofline:
                roofline["traffic"] = tr
                roofline["traffic_gbs"] = round(tr / (ms / n / 1e3) / 1e9, 1)
                roofline["traffic_frac_of_hbm"] = round(tr / (ms / n / 1e3) / 1e9 / peaks.get("hbm_gbs"), 4)
        # per-stage rooflines: tensor kernels against the dense bf16 peak (and
        # the per-MMA floor), every kernel's DRAM bytes (committed ncu capture,
        # per launch) against the measured HBM bandwidth
        ncu_name = {"enc_front_kernel": "enc_front_tc_kernel", "argmin_kernel": "argmin_tc_kernel",
                    "gather_kernel": "dec_table_kernel", "blob_sizes+scan": "blob_sizes_kernel"}
        hbm_peak = peaks.get("hbm_gbs")
        tpeak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
        # (up conv and head share tc_conv_kernel with different N: no single floor)
        floor = {"dec_trunk_kernel": 44.0, "tc3_block_kernel": 92.0, "tc3_conv_kernel": 92.0}
        mhz = clk.summary().get("sm_mhz") or 1965.0
        stages = {}
        for k, (n, ms, units) in prof.items():
            e = {"launches": n, "ms_per_step": round(ms / args.steps, 4)}
            tr = _traffic(ncu_name.get(k, k))
            if tr is not None and ms > 0:
                gbs = tr * n / (ms / 1e3) / 1e9
                e["hbm_gbs"] = round(gbs, 1)
                e["hbm_frac"] = round(gbs / hbm_peak, 4)
            if k in notes and ms > 0:
                tf = units / (ms / 1e3) / 1e12
                e["tflops"] = round(tf, 2)
                e["tensor_frac"] = round(tf / tpeak, 4)
                if k in floor:
                    att = 2.0 * 128 * 32 * 16 / floor[k] * peaks.get("sm_count", 148) * mhz * 1e6 / 1e12
                    e["mma_floor_frac"] = round(tf / att, 4)
            stages[k] = e
        cpu = None
        if ws == 1 and not args.no_cpu:
            procs = len(os.sched_getaffinity(0))
            per_proc = cpu_sample_size(procs, 10.0, args.weights)
            v, nbytes, wall = cpu_oracle_run(per_proc, procs, weights=args.weights)
            cpu = {"value": round(v, 4), "unit": "MB/s", "cores": procs, "kind": "port",
                   "sample": f"{per_proc * procs} CIFAR images ({nbytes} B) compress+decompress, oracle/ numpy+C, "
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
            "dtype": "bf16 tcgen05 decoder, fp32-class encoder (3-product fp16 split on tcgen05), 3xTF32 + f64 argmin, "
                     "int coder/predictor/container",
            "data": "synthetic",
            "config": {"workload": wl["desc"], "weights": args.weights, "global_batch": wl["N"] * ws, "image": [wl["H"], wl["W"], 3],
                       "parallelism": f"shard{ws}", "l2": "flushed (256 MiB write) before each step"},
            "frame_decompress_latency_ms": lat,
            "compress_mb_s": round(raw_bytes * ws / 1e6 / t_cs, 3),
            "decompress_mb_s": round(raw_bytes * ws / 1e6 / t_ds, 3),
            "bpd": round(bpd, 4),
            "lossless": lossless,
            "e2e": {"value": round(e2e_value, 3), "unit": "MB/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "compress_mb_s": round(raw_bytes / 1e6 / statistics.median(e2e_c), 3),
                    "decompress_mb_s": round(raw_bytes / 1e6 / statistics.median(e2e_d), 3)},
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


def run_coder(args):
    """configs[4]: coder only. n = 2^26 symbols from the paper's Table-6
    generator (report._bench_symbols, report.py:34-44: d uniform over the 8
    default-grid distributions, symbol ~ PMF_d, seed 0); symbol i -> lane
    i mod L. Encode and decode each timed with CUDA events (device-resident
    symbols / d / lane payloads); GB/s counts algorithmic bytes (symbol + d +
    payload), the SURVEY §8d unit."""
    import numpy as np
    import torch

    from paper_2206_05279_b200 import _lib, tables
    from paper_2206_05279_b200.device import ptr, sptr
    from paper_2206_05279_b200.logistic import default_grid, residual_distributions

    _, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    M, n = 12, 1 << 26
    pmfs = residual_distributions(default_grid(), M)
    rng = np.random.default_rng(0)
    d = rng.integers(0, 8, n).astype(np.uint8)
    syms = np.empty(n, np.uint8)
    for i, pmf in enumerate(pmfs):
        sel = d == i
        syms[sel] = rng.choice(256, int(sel.sum()), p=pmf.P.astype(np.float64) / (1 << M))
    enc, dec = tables.build_tables(pmfs, M)
    s_d = torch.from_numpy(syms).to(dev)
    d_d = torch.from_numpy(d).to(dev)
    rows = []
    for L in [1 << k for k in (10, 12, 14, 16, 18, 20)]:
        def encode():
            return tables.encode_lanes_device(s_d, 1, n, L, enc, dev, stream, dsched=d_d)
        scr, cap, nb, st = encode()
        lane_off = torch.arange(L, dtype=torch.int64, device=dev) * (cap * 4)
        out = torch.empty(n, dtype=torch.uint8, device=dev)
        lstat = torch.zeros(L, dtype=torch.uint8, device=dev)

        def decode():
            lstat.zero_()
            _lib.call("pilc_rans_decode", ptr(scr), ptr(lane_off), ptr(nb), ptr(st), ptr(d_d), None, 1, n, L,
                      ptr(dec.device_words(dev)), dec.D, M, None, ptr(out), ptr(lstat), sptr(stream))
        decode()
        torch.cuda.synchronize(dev)
        assert torch.equal(out, s_d) and int(lstat.max()) == 0
        payload = float(nb.to(torch.int64).sum().item()) / 8.0
        te, td = [], []
        for _ in range(max(args.steps, 1)):
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record(stream)
            encode()
            b.record(stream)
            decode()
            c.record(stream)
            torch.cuda.synchronize(dev)
            te.append(a.elapsed_time(b) / 1e3)
            td.append(b.elapsed_time(c) / 1e3)
        algo = 2.0 * n + payload
        rows.append({"lanes": L, "bits_per_symbol": round(8 * payload / n, 4),
                     "encode_gb_s": round(algo / statistics.median(te) / 1e9, 2),
                     "decode_gb_s": round(algo / statistics.median(td) / 1e9, 2),
                     "encode_msym_s": round(n / statistics.median(te) / 1e6, 1),
                     "decode_msym_s": round(n / statistics.median(td) / 1e6, 1)})
    if rank == 0:
        peak = None
        try:
            with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
                peak = json.load(f).get("hbm_gbs")
        except OSError:
            peak = 6650.0
        best = max(rows, key=lambda r: r["decode_gb_s"])
        print(json.dumps({"metric": "rANS coder-only decode GB/s (algorithmic bytes)", "value": best["decode_gb_s"],
                          "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                          "higher_is_better": True, "data": "synthetic",
                          "config": {"workload": "coder-only sweep, n=2^26 Table-6 symbols, D=8, M=12"},
                          "roofline": {"bound": "hbm", "peak": peak, "unit": "GB/s",
                                       "frac": round(best["decode_gb_s"] / (peak / 1.0), 4)},
                          "sweep": rows}), flush=True)
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
    ap.add_argument("--workload", default="cifar", choices=sorted(WORKLOADS) + ["coder"],
                    help="BASELINE config: cifar (configs[1], default), in64 (configs[2]), 1080p (configs[3]), "
                         "coder (configs[4], coder-only lane sweep)")
    ap.add_argument("--weights", default="random", choices=["random", "trained"],
                    help="random_weights(seed=1) (default) or tests/golden/trained.pilw")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "coder":
        return run_coder(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
