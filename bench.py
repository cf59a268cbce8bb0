#!/usr/bin/env python
"""bench.py -- batched dual-select FFT throughput on B200 (driver contract).

Workload (BASELINE.json configs[1], and configs[3] across GPUs): N=1024, FP16,
dual-select, one global batch of 2^20 transforms, synthetic uniform[-1,1)
complex data generated on the device from the GLOBAL transform index
(dsfft_fill_uniform) before timing.  One step = one forward pass over the
whole batch (one kernel launch per GPU).  Inputs (4 GiB) and outputs (4 GiB)
exceed the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dsfft|reference]
                  [--n N] [--precision fp16|fp32] [--strategy dual|lf|cosine|standard]
                  [--global-batch B | --batch B_per_gpu]

Multi-GPU: one process per GPU.  `--gpus N` without a
torchrun environment re-launches itself under `torch.distributed.run` with N
ranks; under torchrun WORLD_SIZE must equal --gpus.  Default is STRONG
scaling: the 2^20-transform global batch is split into contiguous shards
(distributed.shard_range); `--batch B` selects weak scaling (B transforms per
GPU, rank r owns global transforms [rB, (r+1)B)).  Shards need no data-path
collective (batched FFTs exchange nothing); NCCL carries only the barrier and
the MAX of per-rank CUDA-event step times.  Because inputs are keyed by the
global index, every shard equals the same rows of the 1-GPU run
(tests/test_gpu_distributed.py checks this bit for bit).
DSFFT_DIST_BACKEND=gloo runs the control plane over gloo, which lets several
ranks share one GPU (tests only).

Reported on rank 0 as one JSON line: value = transforms/s of the whole job,
roofline (HBM bytes = 2*N*sizeof(complex) per transform vs the measured copy
bandwidth in MEASURED_PEAKS.json), e2e through the C ABI with pinned host
buffers (dsfft_execute_host: H2D + kernels + D2H inside the timed region),
accuracy of every transform vs the FP64 dft_oracle on the device (plus the LF
comparison and the paper's bound), a sustained leg (>= 3 s back to back, with
its own clock / power samples: the board's power cap shows there), the
reference's own CPU path (oracle/_ref) on this host's cores, clocks sampled
during the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_N = 1024
DEFAULT_GLOBAL_BATCH = 1 << 20
SEED = 20260419


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dsfft", choices=["dsfft", "reference"])
    ap.add_argument("--n", type=int, default=DEFAULT_N)
    g = ap.add_mutually_exclusive_group()
    g.add_argument("--global-batch", type=int, default=None,
                   help="strong scaling: total transforms split over the GPUs "
                        "(default 2^20 for N<=8192)")
    g.add_argument("--batch", type=int, default=None,
                   help="weak scaling: transforms per GPU (default for N>8192: 1 GiB of input)")
    ap.add_argument("--precision", default="fp16", choices=["fp16", "fp32"])
    ap.add_argument("--strategy", default="dual")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--sustained-seconds", type=float, default=3.0,
                    help="back-to-back leg after the timed steps (0 disables)")
    ap.add_argument("--dump", default=None,
                    help="directory: each rank saves its output shard (tests)")
    return ap.parse_args()


def resolve_batches(args, world):
    """(mode, global_batch, per_rank) for the run."""
    sb = 4 if args.precision == "fp16" else 8
    if args.batch is not None:
        return "weak", args.batch * world, args.batch
    if args.global_batch is not None:
        return "strong", args.global_batch, None
    if args.n <= 8192:  # BASELINE configs[1] / configs[3]
        return "strong", DEFAULT_GLOBAL_BATCH, None
    per = max(1, (1 << 30) // (args.n * sb))  # configs[4]: 1 GiB of input per GPU
    return "weak", per * world, per


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def kernel_name(n: int, launches_per_step: int) -> str:
    """The dominant kernel of the workload: the single kernel for N <= 8192;
    above, the fused one-launch kernel when the library chose it (one launch
    per step), else the pass-group kernel."""
    if n <= 8192:
        return "fft_small_kernel"
    return "mp_fused_kernel" if launches_per_step == 1 else "mp_kernel"


def load_traffic(args, batch):
    """ncu dram bytes per launch from the committed capture of this workload,
    scaled to this run's batch (None when no capture exists)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        e = s.get(f"n{args.n}_{args.precision}_{args.strategy}")
        if e and e.get("batch"):
            return float(e["dram_bytes"]) * batch / float(e["batch"]), e.get("kernel")
    except Exception:
        pass
    return None, None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """Polls NVML during a timed region: SM clock, throttle reasons, power."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device_index: int, period: float = 0.005):
        self.ok = False
        self.period = period
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
        self.samples, self.power, self.reasons = [], [], 0
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            except Exception:
                pass
            time.sleep(self.period)

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
        out = {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max,
               "reasons": names, "samples": len(self.samples)}
        if self.power:
            out["power_w_median"] = float(statistics.median(self.power))
            out["power_w_max"] = float(max(self.power))
        return out


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


def workload_config(args, world, mode, global_batch, per_rank):
    """The same config block on both arms."""
    which = "configs[1]/[3]" if args.n == 1024 and args.precision == "fp16" else \
        ("configs[4]" if args.n > 8192 else "configs[2]")
    if mode == "strong":
        desc = f"global batch {global_batch} split over {world} GPU(s)"
    else:
        desc = f"batch {per_rank} per GPU"
    return {"workload": f"N={args.n} {args.precision} {args.strategy}-select forward, {desc} "
                        f"(BASELINE {which})",
            "n": args.n, "precision": args.precision, "strategy": args.strategy,
            "global_batch": global_batch, "batch_per_gpu": per_rank if per_rank else
            -(-global_batch // world), "parallelism": f"batch shards x{world}, no collectives",
            "inputs": "device-generated from the global transform index (dsfft_fill_uniform)",
            "l2": "inputs (and outputs) > L2 per step; no flush needed"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path timed on this host's cores
    (rank 0 only; other ranks exit without work)."""
    if rank != 0:
        return
    mode, gb, per = resolve_batches(args, max(args.gpus, 1))
    rates = []
    per_step = max(1.0, min(20.0, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_reference_rate(args, per_step * 0.25)
    sample = kind = cores = None
    for _ in range(args.steps):
        r, sample, kind, cores, _ = cpu_reference_rate(args, per_step)
        rates.append(r)
    value = float(statistics.median(rates))
    line = {
        "impl": "reference", "metric": "batched FFT transforms/s", "value": value,
        "unit": "transforms/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sample / value,
        "higher_is_better": True, "scaling": mode, "vs_baseline": None,
        "dtype": "f16" if args.precision == "fp16" else "f32", "data": "synthetic",
        "config": workload_config(args, max(args.gpus, 1), mode, gb, per),
        "cpu_baseline": {"value": value, "unit": "transforms/s", "cores": cores, "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{sample} transforms of the workload per step"},
        "e2e": {"value": value, "unit": "transforms/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args) -> int:
    """--gpus N outside torchrun: run this script under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", "--", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    from paper_2604_00567_b200.distributed import env_rank, max_over_ranks
    rank, world, local = env_rank()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} "
                 "(launch one process per GPU)")

    import torch

    import paper_2604_00567_b200 as dsfft
    from paper_2604_00567_b200.distributed import make_shard, sharded_forward

    # one process per GPU; DSFFT_DIST_BACKEND=gloo exercises the control plane
    # with several ranks sharing one device (no data-path collective either way)
    backend = os.environ.get("DSFFT_DIST_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    if ndev == 0:
        sys.exit("bench.py: no CUDA device (the product has no CPU path)")
    if backend == "nccl" and world > ndev:
        sys.exit(f"bench.py: {world} ranks need {world} GPUs, found {ndev}")
    local_dev = local % ndev
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    red_dev = dev if backend == "nccl" else None

    mode, global_batch, per_rank = resolve_batches(args, world)
    n, prec = args.n, args.precision
    plan = dsfft.make_plan(n, args.strategy, prec, device=local_dev)
    sbytes = 4 if prec == "fp16" else 8
    shard = make_shard(plan, rank, world, SEED,
                       global_batch=global_batch if mode == "strong" else None,
                       per_rank_batch=per_rank if mode == "weak" else None)
    batch = shard.count
    stream = torch.cuda.current_stream(dev)

    def step():
        sharded_forward(plan, shard, stream=stream.cuda_stream)

    for _ in range(max(3, args.warmup)):
        step()
    launches_per_step = dsfft.last_launch_count()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_dev) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_rank = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms_rank, red_dev)  # the job's step = slowest rank
    value = global_batch / (ms * 1e-3)
    algo_bytes = 2.0 * n * sbytes * batch  # per launch on this rank, read once + write once
    achieved = algo_bytes / (ms_rank * 1e-3) / 1e9
    peak, peak_kind = load_peaks()
    traffic, traffic_kernel = load_traffic(args, batch)

    if args.dump:
        os.makedirs(args.dump, exist_ok=True)
        torch.cuda.synchronize()
        np.save(os.path.join(args.dump, f"shard{rank}.npy"), shard.y.cpu().numpy())
        np.save(os.path.join(args.dump, f"range{rank}.npy"), np.array([shard.start, shard.stop]))

    # sustained: back-to-back steps for >= S seconds with their own samples
    sustained = None
    if args.sustained_seconds > 0:
        k = max(args.steps, int(np.ceil(args.sustained_seconds / (ms_rank * 1e-3))))
        if dist:
            dist.barrier()
        with ClockSampler(local_dev, period=0.02) as sclk:
            ev0.record(stream)
            for _ in range(k):
                step()
            ev1.record(stream)
            torch.cuda.synchronize()
        sms = max_over_ranks(ev0.elapsed_time(ev1) / k, red_dev)
        sustained = {"value": global_batch / (sms * 1e-3), "ms_per_step": sms, "steps": k,
                     "seconds": sms * k * 1e-3,
                     "roofline_frac": algo_bytes / (sms * 1e-3) / 1e9 / peak,
                     "clocks": sclk.summary()}

    # accuracy of every transform of the shard, on the device: rel-L2 vs the
    # FP64 dft_oracle (bit-identical to fft.cpp:103-121; fp64 FFT for N > 4096)
    acc = None
    if not args.no_accuracy and batch:
        rep = dsfft.error_device(plan, shard.x, "forward")
        how = "FP64 DFT (device dft_oracle)" if n <= 4096 else "FP64 FFT (device fp64 path)"
        acc = {"max_rel_l2_vs_fp64": rep["rel_l2_max"], "median_rel_l2": rep["rel_l2_median"],
               "nonfinite": rep["nonfinite_trials"], "transforms": rep["trials"],
               "how": f"dsfft_error_device over every transform of rank 0's shard vs {how}"}
        # the paper's claim on the same batch: dual-select within Eq. 11's bound
        # and below Linzer-Feig-with-clamp (north_star; analysis.cpp:61-63)
        if args.strategy == "dual":
            eps = 2.0 ** -11 if prec == "fp16" else 2.0 ** -24
            tab = dsfft.build_table(n, "dual", "fp64")
            acc["paper_bound"] = (1.0 + float(np.abs(tab["ratio"]).max()) * eps) ** \
                int(np.log2(n)) - 1.0
            lf = dsfft.error_device(dsfft.make_plan(n, "lf", prec, device=local_dev), shard.x,
                                    "forward")
            acc["lf_max"], acc["lf_median"] = lf["rel_l2_max"], lf["rel_l2_median"]
            acc["dual_beats_lf"] = rep["rel_l2_median"] < lf["rel_l2_median"]
            acc["within_bound"] = rep["rel_l2_max"] <= acc["paper_bound"]

    # e2e through the C ABI with pinned host buffers (each rank its shard)
    e2e = None
    if not args.no_e2e and batch:
        ksteps = args.e2e_steps or max(2, min(args.steps, 5))
        eb = batch  # e2e batch: the whole shard unless pinned host memory runs short
        while True:
            try:
                hx = torch.empty((eb, n, 2), dtype=shard.x.dtype, pin_memory=True)
                hy = torch.empty((eb, n, 2), dtype=shard.x.dtype, pin_memory=True)
                break
            except RuntimeError:
                if eb <= 1024:
                    raise
                eb //= 4
        hx.copy_(shard.x[:eb])
        hxn, hyn = hx.numpy(), hy.numpy()
        dsfft.execute_host(plan, 0, hxn, hyn, eb, stream.cuda_stream)  # warm-up
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ksteps):
            dsfft.execute_host(plan, 0, hxn, hyn, eb, stream.cuda_stream)
        dt = max_over_ranks((time.perf_counter() - t0) / ksteps, red_dev)
        e2e = {"value": eb * world / dt, "unit": "transforms/s",
               "h2d_bytes_per_step": int(hx.numel() * hx.element_size()),
               "d2h_bytes_per_step": int(hy.numel() * hy.element_size()),
               "ms_per_step": dt * 1e3, "path": "dsfft_execute_host (pinned), per rank",
               "transforms_per_step": eb * world}
        del hx, hy

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            r, sample, kind, cores, secs = cpu_reference_rate(args, args.cpu_seconds)
            cpu = {"value": r, "unit": "transforms/s", "cores": cores, "kind": kind,
                   "cpu_model": cpu_model(),
                   "sample": f"{sample} transforms (N={n} {prec} {args.strategy}), {secs:.1f} s"}
        except Exception as e:  # the checker is optional on a bare box
            cpu = {"value": None, "unit": "transforms/s", "cores": None, "kind": None,
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": "batched FFT transforms/s", "value": value, "unit": "transforms/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": mode, "vs_baseline": None,
            "dtype": "f16" if prec == "fp16" else "f32", "data": "synthetic",
            "config": workload_config(args, world, mode, global_batch, per_rank),
            "gflops": 5.0 * n * np.log2(n) * value / 1e9,
            "hbm_gbs": 2.0 * n * sbytes * value / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_kind": peak_kind, "kernel": kernel_name(n, launches_per_step),
                         "traffic_from": traffic_kernel,
                         "launches_per_step": launches_per_step,
                         "algorithmic_bytes_per_step": algo_bytes,
                         "how": "2*N*sizeof(complex) per transform of rank 0's shard / "
                                "rank 0's CUDA-event step time"},
            "sustained": sustained,
            "accuracy": acc,
            "e2e": e2e,
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
