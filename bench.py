#!/usr/bin/env python
"""Benchmark of the DGAL hot path on B200 (driver contract: one JSON line).

Headline workload = BASELINE cfg3: paired IoU loss forward + backward over 2^24
KITTI-like rotated-box pairs Poly2<float,4> per GPU (one "step" = one
dgal_iou_paired_fwd + one dgal_iou_paired_bwd over the whole batch, i.e. every
§8(a) row of the paired path a0-a12).  Multi-GPU (torchrun, one process per
GPU): weak scaling, each rank owns its own 2^24-pair shard, no collective on the
data path; elapsed = max over ranks of the CUDA-event time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--impl reference times the CPU oracle (oracle/, double precision, all host
cores) on a bounded sample of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IoU pairs/sec fwd+bwd (1/2/4/8 B200), % of FP32/HBM roofline vs CPU oracle"
UNIT = "pairs/s"
N_PAIRS = 1 << 24        # cfg3 per GPU
K = 4
# algorithmic bytes per pair: fwd reads 4 planes x 16 B, writes
# iou 4 + nx 1 + xflags 8; bwd reads 64 + g 4 + nx 1 + xflags 8, writes 64.
FWD_BYTES = 64 + 4 + 1 + 8
BWD_BYTES = 64 + 4 + 1 + 8 + 64


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """Per-launch DRAM bytes of the kernels from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while running (10 ms period)."""

    REASONS = {
        0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index):
        self.samples = []
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()
        self.window = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                t = time.perf_counter()
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((t, mhz, rs))
            except Exception:
                pass
            time.sleep(0.01)

    def start(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.th.join()

    def summary(self, t0, t1):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "NVML unavailable"}
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        if not win:  # region shorter than the period: nearest samples
            win = sorted(self.samples, key=lambda s: abs(s[0] - 0.5 * (t0 + t1)))[:3]
        mhz = [s[1] for s in win]
        reasons = set()
        for s in win:
            for bit, name in self.REASONS.items():
                if s[2] & bit:
                    reasons.add(name)
        return {"sm_mhz": float(np.median(mhz)) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(win)}


def cpu_oracle_rate(batch, seconds=10.0, threads=0):
    """Time the oracle (fwd + bwd, as it stands) on a bounded prefix of the workload."""
    import oracle
    nt = threads or oracle.max_threads()
    probe = batch.take(np.arange(min(20000, batch.n)))
    t = time.perf_counter()
    oracle.iou_paired_fwd(probe.p1, probe.p2, nthreads=nt)
    oracle.iou_paired_bwd(probe.p1, probe.p2, probe.grad, nthreads=nt)
    rate = probe.n / (time.perf_counter() - t)
    n = int(min(batch.n, max(probe.n, rate * seconds)))
    s = batch.take(np.arange(n))
    t = time.perf_counter()
    oracle.iou_paired_fwd(s.p1, s.p2, nthreads=nt)
    oracle.iou_paired_bwd(s.p1, s.p2, s.grad, nthreads=nt)
    dt = time.perf_counter() - t
    return n / dt, nt, n, dt


def run_reference(args, rank):
    import synth
    if rank != 0:
        return 0
    batch = synth.gen_cfg3_pairs(1 << 20)
    import oracle
    nt = oracle.max_threads()
    # each step = fwd+bwd over a bounded sample (sized from a probe to ~2 s/step)
    rate, nt, _, _ = cpu_oracle_rate(batch, seconds=1.0)
    n = int(min(batch.n, max(20000, rate * 2.0)))
    s = batch.take(np.arange(n))
    for _ in range(args.warmup):
        oracle.iou_paired_fwd(s.p1, s.p2, nthreads=nt)
        oracle.iou_paired_bwd(s.p1, s.p2, s.grad, nthreads=nt)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle.iou_paired_fwd(s.p1, s.p2, nthreads=nt)
        oracle.iou_paired_bwd(s.p1, s.p2, s.grad, nthreads=nt)
    dt = time.perf_counter() - t
    v = n * args.steps / dt
    sample = f"first {n} pairs of the cfg3 workload per step (of {N_PAIRS} per GPU), fwd+bwd, float64"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "cfg3 paired IoU fwd+bwd, KITTI-like rotated boxes, K=4 (CPU oracle sample)",
                   "pairs_per_step": n},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": nt, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="dgal", choices=["dgal", "reference"])
    ap.add_argument("--pairs", type=int, default=N_PAIRS, help="pairs per GPU (default: cfg3's 2^24)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        return run_reference(args, rank)

    import torch
    import paper_2011_11134_b200 as dgal
    import synth
    from paper_2011_11134_b200.hostpipe import HostPipeline

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    # ---- inputs: this rank's shard, resident in HBM ----
    n = args.pairs
    batch = synth.gen_cfg3_pairs(n, seed=synth.seed_for(3, rank))
    T = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    x1, y1 = T(batch.p1.x.reshape(n, K)), T(batch.p1.y.reshape(n, K))
    x2, y2 = T(batch.p2.x.reshape(n, K)), T(batch.p2.y.reshape(n, K))
    g = torch.full((n,), -1.0 / n, dtype=torch.float32, device=dev)   # d(mean(1-IoU))/dIoU
    iou = torch.empty(n, dtype=torch.float32, device=dev)
    nx = torch.empty(n, dtype=torch.uint8, device=dev)
    xf = torch.empty((n, 2 * K), dtype=torch.uint8, device=dev)
    grads = tuple(torch.empty((n, K), dtype=torch.float32, device=dev) for _ in range(4))

    def step():
        dgal.iou_paired_fwd(x1, y1, x2, y2, out=(iou, nx, xf))
        dgal.iou_paired_bwd(x1, y1, x2, y2, g, nx, xf, out=grads)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.05)
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for s in range(args.steps):
        e0, e1, e2 = ev[s]
        e0.record(stream)
        dgal.iou_paired_fwd(x1, y1, x2, y2, out=(iou, nx, xf))
        e1.record(stream)
        dgal.iou_paired_bwd(x1, y1, x2, y2, g, nx, xf, out=grads)
        e2.record(stream)
    end.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    if dist:
        dist.barrier()
    time.sleep(0.02)
    sampler.stop()

    ms = start.elapsed_time(end)
    fwd_ms = sum(a.elapsed_time(b) for a, b, _ in ev) / args.steps
    bwd_ms = sum(b.elapsed_time(c) for _, b, c in ev) / args.steps
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_pairs = n * args.steps * world
    value = total_pairs / (ms * 1e-3)

    # ---- e2e: host buffers, H2D + fwd + bwd + D2H inside the timed region ----
    e2e = None
    if not args.no_e2e:
        pipe = HostPipeline(K, device=dev)
        x4h = torch.stack([x1, y1, x2, y2]).cpu().pin_memory()
        gh = g.cpu().pin_memory()
        iouh = torch.empty(n, dtype=torch.float32).pin_memory()
        g4h = torch.empty((4, n, K), dtype=torch.float32).pin_memory()
        pipe.run(x4h, gh, iouh, g4h)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            pipe.run(x4h, gh, iouh, g4h)
        b.record(stream)
        torch.cuda.synchronize()
        ems = a.elapsed_time(b)
        if dist:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": n * args.e2e_steps * world / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(x4h.numel() * 4 + gh.numel() * 4),
               "d2h_bytes_per_step": int(iouh.numel() * 4 + g4h.numel() * 4),
               "ms_per_step": ems / args.e2e_steps,
               "path": "pinned host -> chunked 3-stream pipeline (H2D, fwd, bwd, D2H)"}
        # sanity: the e2e result equals the device result
        assert torch.equal(iouh, iou.cpu()), "e2e IoU differs from device IoU"

    if dist:
        dist.destroy_process_group()
    if rank != 0:
        return 0

    peak, peak_src = measured_peaks()
    fwd_gbs = n * FWD_BYTES / (fwd_ms * 1e-3) / 1e9
    bwd_gbs = n * BWD_BYTES / (bwd_ms * 1e-3) / 1e9
    dom = "paired_fwd" if fwd_ms >= bwd_ms else "paired_bwd"
    dom_gbs = fwd_gbs if dom == "paired_fwd" else bwd_gbs
    traffic = ncu_traffic().get(f"{dom}_k4_bytes_per_launch")
    clocks = sampler.summary(t_wall0, t_wall1)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        sample = synth.gen_cfg3_pairs(1 << 20, seed=synth.seed_for(3, rank))
        rate, nt, ns, dt = cpu_oracle_rate(sample, seconds=10.0)
        cpu = {"value": rate, "unit": UNIT, "cores": nt, "kind": "oracle",
               "sample": f"first {ns} pairs of this cfg3 workload, fwd+bwd in float64 ({dt:.1f} s)"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "cfg3: paired IoU loss fwd+bwd, KITTI-like rotated-box pairs, Poly2<float,4>",
                   "pairs_per_gpu": n, "global_pairs": n * world, "K": K,
                   "parallelism": f"dp{world} (contiguous pair shards, no collective)",
                   "l2": "inputs 1.07 GB/GPU > 126 MB L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": dom_gbs, "peak": peak, "unit": "GB/s",
                     "frac": dom_gbs / peak, "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_pair": {"paired_fwd": FWD_BYTES, "paired_bwd": BWD_BYTES},
                     "paired_fwd": {"ms": fwd_ms, "GB/s": fwd_gbs, "frac": fwd_gbs / peak},
                     "paired_bwd": {"ms": bwd_ms, "GB/s": bwd_gbs, "frac": bwd_gbs / peak},
                     "step_frac": (n * (FWD_BYTES + BWD_BYTES) / (ms / args.steps * 1e-3) / 1e9) / peak},
        "clocks": clocks,
        "gpu_launches": 2 * args.steps,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())
