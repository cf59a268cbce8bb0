#!/usr/bin/env python
"""bench.py -- batched dual-select FFT throughput on B200 (driver contract).

Workload (BASELINE.json configs[1]): N=1024, FP16, dual-select, batch 2^20
transforms per GPU, synthetic uniform[-1,1) complex data generated on the
device before timing.  One step = one forward pass over the whole batch
(one kernel launch).  Inputs (4 GiB) and outputs (4 GiB) exceed the 126 MB L2,
so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dsfft|reference]

Multi-GPU: one process per GPU (torchrun); each rank transforms its own
2^20-transform shard (weak scaling, no data-path collective -- batched FFTs
exchange nothing); the step time is the max over ranks (all_reduce MAX on the
per-rank CUDA-event times).

Reported on rank 0 as one JSON line: value = transforms/s of the whole job,
roofline (HBM bytes = 2*N*sizeof(complex) per transform vs the measured copy
bandwidth in MEASURED_PEAKS.json), e2e through the C ABI with pinned host
buffers (dsfft_execute_host: H2D + kernels + D2H inside the timed region),
accuracy of every transform of the batch vs an FP64 reference transform on the
device (plus the LF comparison and the paper's bound), cpu_baseline (the
reference's own CPU path, oracle/_ref, on this host's cores), clocks sampled
during the run.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_N = 1024
DEFAULT_BATCH = 1 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dsfft", choices=["dsfft", "reference"])
    ap.add_argument("--n", type=int, default=DEFAULT_N)
    ap.add_argument("--batch", type=int, default=None,
                    help="transforms per GPU (default 2^20 for N<=4096, else 1 GiB of input)")
    ap.add_argument("--precision", default="fp16", choices=["fp16", "fp32"])
    ap.add_argument("--strategy", default="dual")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(args):
    """dram bytes per launch from the committed ncu capture, when present."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        key = f"n{args.n}_{args.precision}_{args.strategy}"
        e = s.get(key)
        if e and e.get("batch"):
            # scale the captured per-launch bytes to this run's batch
            return float(e["dram_bytes"]) * args.batch / float(e["batch"])
    except Exception:
        pass
    return None


class ClockSampler:
    """Polls NVML during the timed region (SM clock + throttle reasons)."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device_index: int):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[device_index]) if vis else device_index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["nvml unavailable"]}
        names = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max,
                "reasons": names, "samples": len(self.samples)}


def cpu_reference_rate(args, seconds: float, threads: int = 0):
    """The reference's own CPU forward (oracle/_ref = fmafft compiled from its
    sources; else the oracle port) on this host's cores, on a bounded sample
    of the same workload.  Returns (transforms/s, sample transforms, kind, cores)."""
    import oracle
    kind = "reference" if oracle.ref_available() else "port"
    lib = oracle.load_ref() if kind == "reference" else oracle.load_oracle()
    cores = threads or os.cpu_count() or 1
    x = lib.random_buffer(args.n, 42, batch=max(cores, 64))
    t0 = time.perf_counter()
    lib.forward(x, args.strategy, args.precision, threads=cores)
    dt = time.perf_counter() - t0
    rate0 = x.shape[0] / max(dt, 1e-9)
    count = int(max(cores, min(rate0 * seconds, 1 << 20)))
    xs = lib.random_buffer(args.n, 43, batch=count)
    t0 = time.perf_counter()
    lib.forward(xs, args.strategy, args.precision, threads=cores)
    dt = time.perf_counter() - t0
    return count / dt, count, kind, cores, dt


def workload_config(args, world):
    """The same config block on both arms (BASELINE configs[1] by default)."""
    which = "configs[1]" if args.n == 1024 and args.precision == "fp16" else \
        ("configs[4]" if args.n > 4096 else "configs[2]")
    return {"workload": f"N={args.n} {args.precision} {args.strategy}-select forward, "
                        f"batch {args.batch} per GPU (BASELINE {which})",
            "n": args.n, "precision": args.precision, "strategy": args.strategy,
            "batch_per_gpu": args.batch, "global_batch": args.batch * world,
            "l2": "inputs (and outputs) > L2 per step; no flush needed"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path timed on this host's cores."""
    if rank != 0:
        return
    rates = []
    per_step = max(1.0, min(20.0, 60.0 / max(1, args.steps + args.warmup)))
    for i in range(args.warmup):
        cpu_reference_rate(args, per_step * 0.25)
    sample = kind = cores = None
    for i in range(args.steps):
        r, sample, kind, cores, _ = cpu_reference_rate(args, per_step)
        rates.append(r)
    value = float(statistics.median(rates))
    line = {
        "impl": "reference", "metric": "batched FFT transforms/s", "value": value,
        "unit": "transforms/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sample / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f16" if args.precision == "fp16" else "f32", "data": "synthetic",
        "config": workload_config(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": "transforms/s", "cores": cores, "kind": kind,
                         "sample": f"{sample} transforms of the workload per step"},
        "e2e": {"value": value, "unit": "transforms/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def accuracy_sample(y_host: np.ndarray, x_host: np.ndarray, n: int):
    """Max / median rel-L2 error vs an FP64 DFT (numpy, float64) on a sample."""
    x = x_host.astype(np.float64).view(np.complex128)[..., 0]
    y = y_host.astype(np.float64).view(np.complex128)[..., 0]
    ref = np.fft.fft(x, axis=-1)
    num = np.sqrt(np.sum(np.abs(y - ref) ** 2, axis=-1))
    den = np.sqrt(np.sum(np.abs(ref) ** 2, axis=-1))
    err = num / den
    fin = np.isfinite(err)
    return float(np.max(err)) if fin.all() else float("inf"), float(np.median(err[fin]))


def main():
    args = parse()
    if args.batch is None:  # BASELINE configs[1] / configs[4]
        sb = 4 if args.precision == "fp16" else 8
        args.batch = DEFAULT_BATCH if args.n <= 4096 else max(1, (1 << 30) // (args.n * sb))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_2604_00567_b200 as dsfft

    # one process per GPU; DSFFT_DIST_BACKEND=gloo exercises the control plane
    # with several ranks sharing one device (no data-path collective either way)
    backend = os.environ.get("DSFFT_DIST_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def reduce_max(v: float) -> float:
        """Control-plane MAX over ranks (NCCL tensors live on the device)."""
        if not dist:
            return float(v)
        t = torch.tensor([float(v)], dtype=torch.float64,
                         device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    n, batch, prec = args.n, args.batch, args.precision
    plan = dsfft.make_plan(n, args.strategy, prec, device=local_dev)
    wdt = torch.float16 if prec == "fp16" else torch.float32
    sbytes = 4 if prec == "fp16" else 8
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    x = (torch.rand((batch, n, 2), device=dev, generator=g, dtype=torch.float32) * 2 - 1).to(wdt)
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)

    def step():
        dsfft.forward(plan, x, out=y, stream=stream.cuda_stream)

    for _ in range(max(3, args.warmup)):
        step()
    launches_per_step = dsfft.last_launch_count()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = reduce_max(ev0.elapsed_time(ev1) / args.steps)  # the job's step = slowest rank
    total = batch * world
    value = total / (ms * 1e-3)
    algo_bytes = 2.0 * n * sbytes * batch  # per launch, read once + write once
    achieved = algo_bytes / (ms * 1e-3) / 1e9
    peak, peak_kind = load_peaks()
    traffic = load_traffic(args)

    # accuracy of every transform of the batch, on the device: rel-L2 vs an
    # FP64 reference transform (dsfft_error_device, measure_error semantics)
    acc = None
    if not args.no_accuracy:
        rep = dsfft.error_device(plan, x, "forward")
        acc = {"max_rel_l2_vs_fp64": rep["rel_l2_max"], "median_rel_l2": rep["rel_l2_median"],
               "nonfinite": rep["nonfinite_trials"], "transforms": rep["trials"],
               "how": "dsfft_error_device over the whole batch (FP64 reference transform)"}
        # the paper's claim on the same batch: dual-select within Eq. 11's bound
        # and below Linzer-Feig-with-clamp (north_star; analysis.cpp:61-63)
        if args.strategy == "dual" and prec in ("fp16", "fp32"):
            eps = 2.0 ** -11 if prec == "fp16" else 2.0 ** -24
            tab = dsfft.build_table(n, "dual", "fp64")
            acc["paper_bound"] = (1.0 + float(np.abs(tab["ratio"]).max()) * eps) ** \
                int(np.log2(n)) - 1.0
            lf = dsfft.error_device(dsfft.make_plan(n, "lf", prec, device=local_dev), x,
                                    "forward")
            acc["lf_max"], acc["lf_median"] = lf["rel_l2_max"], lf["rel_l2_median"]
            acc["dual_beats_lf"] = rep["rel_l2_median"] < lf["rel_l2_median"]
            acc["within_bound"] = rep["rel_l2_max"] <= acc["paper_bound"]
        # host cross-check on a few transforms: numpy FP64 FFT
        idx = torch.arange(0, batch, max(1, batch // 16), device=dev)[:16]
        acc["numpy_check_max"], _ = accuracy_sample(y[idx].cpu().numpy(), x[idx].cpu().numpy(),
                                                    n)

    # e2e through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        ksteps = args.e2e_steps or max(2, min(args.steps, 5))
        eb = batch  # e2e batch: the whole shard unless pinned host memory runs short
        while True:
            try:
                hx = torch.empty((eb, n, 2), dtype=x.dtype, pin_memory=True)
                hy = torch.empty((eb, n, 2), dtype=x.dtype, pin_memory=True)
                break
            except RuntimeError:
                if eb <= 1024:
                    raise
                eb //= 4
        hx.copy_(x[:eb])
        hxn, hyn = hx.numpy(), hy.numpy()
        dsfft.execute_host(plan, 0, hxn, hyn, eb, stream.cuda_stream)  # warm-up
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ksteps):
            dsfft.execute_host(plan, 0, hxn, hyn, eb, stream.cuda_stream)
        dt = reduce_max((time.perf_counter() - t0) / ksteps)
        e2e = {"value": eb * world / dt, "unit": "transforms/s",
               "h2d_bytes_per_step": int(hx.numel() * hx.element_size()),
               "d2h_bytes_per_step": int(hy.numel() * hy.element_size()),
               "ms_per_step": dt * 1e3, "path": "dsfft_execute_host (pinned)",
               "transforms_per_step": eb * world}
        del hx, hy

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            r, sample, kind, cores, secs = cpu_reference_rate(args, args.cpu_seconds)
            cpu = {"value": r, "unit": "transforms/s", "cores": cores, "kind": kind,
                   "sample": f"{sample} transforms (N={n} {prec} {args.strategy}), {secs:.1f} s"}
        except Exception as e:  # the checker is optional on a bare box
            cpu = {"value": None, "unit": "transforms/s", "cores": None, "kind": None,
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": "batched FFT transforms/s", "value": value, "unit": "transforms/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f16" if prec == "fp16" else "f32", "data": "synthetic",
            "config": workload_config(args, world),
            "gflops": 5.0 * n * np.log2(n) * value / 1e9,
            "hbm_gbs": achieved * world,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_kind": peak_kind, "kernel": "fft_small_kernel",
                         "algorithmic_bytes_per_launch": algo_bytes},
            "accuracy": acc,
            "e2e": e2e,
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
