"""FEAST B200 benchmark (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1]): dfeast_sygv, N = 4096 dense real
symmetric generalized pencil, M0 = 160, Ne = 8, interval around the ~100
eigenvalues nearest 0; seeded synthetic matrices (workloads.c2_sygv; the
paper's datasets are not shipped).  One STEP = one complete FEAST solve
(factorize all Ne shifts, all refinement passes to convergence).

  value  FEAST iterations/s = sum(loop+1) / device time, inputs resident in HBM
  e2e    same metric through the public API with pinned HOST inputs: H2D of A
         and B and D2H of the result (e, X, res) inside the timed region
  lu     shifted-LU FP64 TFLOP/s = (8/3) N^3 per fb_zgetrf / its mean duration
         (CUDA events on the launching stream) -> the roofline object
  --gpus N > 1: contour points sharded over ranks (point k -> rank k mod N),
         partial Q summed with an NCCL all-reduce each pass ("strong" scaling)
  --impl reference: the CPU oracle port (reference kernel restated in numpy +
         LAPACK zgetrf/zgetrs) on the host cores, same workload and metric.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "FEAST iterations/sec & shifted-LU FP64 TFLOP/s (vs peak)"
UNIT = "iterations/s"
FP64_DMMA_PEAK = 37.1   # TFLOP/s, measured: tools/fp64_peak.cu (profiles/r01_fp64_peak.txt)


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region, in-process
    through NVML (no nvidia-smi subprocesses competing with the launching
    thread); falls back to nvidia-smi when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits: hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
    BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            dev = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(index)).split(",")[index]) \
                if os.environ.get("CUDA_VISIBLE_DEVICES") else index
            self._h = pynvml.nvmlDeviceGetHandleByIndex(dev)
            self._nvml = pynvml
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        return [str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in self.BITS]

    def _loop(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    self.samples.append(self._sample_nvml())
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def cpu_reference_solve(w, threads):
    """One oracle solve (reference algorithm restated, LAPACK linear algebra)."""
    from oracle import oracle_feast_sy
    t0 = time.perf_counter()
    r = oracle_feast_sy(w.a, w.emin, w.emax, w.m0, b=w.b,
                        fpm=[0] + [w.fpm().slot(i) for i in range(1, 65)], reduced="lapack")
    dt = time.perf_counter() - t0
    return r, dt


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    from paper_1203_4031_b200 import workloads as W
    w = W.c2_sygv()
    for _ in range(args.warmup):
        cpu_reference_solve(w, threads)
    total_it, total_t, loops = 0, 0.0, []
    for _ in range(args.steps):
        r, dt = cpu_reference_solve(w, threads)
        total_it += r.loop + 1
        total_t += dt
        loops.append(r.loop)
    v = total_it / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64/c128",
        "data": "synthetic (seeded, workloads.c2_sygv)",
        "config": {"workload": "c2_dfeast_sygv N=4096 M0=160 Ne=8 (BASELINE configs[1])",
                   "m_found": int(r.m), "loops": loops},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} full C2 solves (oracle/feast_oracle.py: reference "
                                   "kernel restated + LAPACK zgetrf/zgetrs, OpenBLAS threads=cores)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1203_4031_b200 as fb
    from paper_1203_4031_b200 import workloads as W
    from paper_1203_4031_b200.dense import DeviceDenseOps
    from paper_1203_4031_b200.device import get_device

    world, rank, local = _dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = get_device()
    w = W.c2_sygv()
    n, m0 = w.n, w.m0
    A_d = torch.from_numpy(w.a).to(dev.tdev)
    B_d = torch.from_numpy(w.b).to(dev.tdev)
    A_h = torch.from_numpy(w.a).pin_memory()
    B_h = torch.from_numpy(w.b).pin_memory()
    fpm = w.fpm()

    def solve_once(a, b):
        if world > 1:
            from paper_1203_4031_b200.distributed import feast_sy_distributed
            return feast_sy_distributed(a, w.emin, w.emax, m0, b=b, fpm=fpm.copy())
        return fb.feast_sy(a, w.emin, w.emax, m0, b=b, fpm=fpm.copy())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        r = solve_once(A_d, B_d)
    # -- device-resident timed region -------------------------------------
    # the host issues ~1300 launches per step: keep Python's cyclic GC from
    # pausing the launching thread inside the timed regions
    import gc
    gc.collect()
    gc.disable()
    barrier()
    launches0 = dev.launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    its, loops = 0, []
    lu_events = []
    DeviceDenseOps.lu_event_sink = lu_events
    with ClockSampler(local) as clk:
        step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        ev0.record()
        step_ev[0].record()
        for i in range(args.steps):
            r = solve_once(A_d, B_d)
            its += r.loop + 1
            loops.append(r.loop)
            step_ev[i + 1].record()
        ev1.record()
        barrier()
    step_ms = [round(step_ev[i].elapsed_time(step_ev[i + 1]), 2) for i in range(args.steps)]
    DeviceDenseOps.lu_event_sink = None
    launches = dev.launches() - launches0
    t = ev0.elapsed_time(ev1) / 1e3
    if world > 1:
        tt = torch.tensor([t], device=dev.tdev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    value = its / t

    # -- LU roofline: fb_zgetrf calls inside the timed region (events on its stream)
    lu_ms = sum(a.elapsed_time(b) for a, b, _ in lu_events) / max(1, sum(c for _, _, c in lu_events))
    lu_flops = 8.0 / 3.0 * n ** 3
    lu_tf = lu_flops / (lu_ms / 1e3) / 1e12

    # -- end to end through the public API with pinned host inputs ----------
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e2e_its = 0
    e0.record()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r2 = solve_once(A_h, B_h)        # uploads A, B; result arrays come back to the host
        e2e_its += r2.loop + 1
    e1.record()
    barrier()
    t_e2e = max(e0.elapsed_time(e1) / 1e3, time.perf_counter() - t0)
    if world > 1:
        tt = torch.tensor([t_e2e], device=dev.tdev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    gc.enable()
    h2d = 2 * n * n * 8
    d2h = n * m0 * 8 + 2 * m0 * 8

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        rr, dt = cpu_reference_solve(w, threads)
        cpu = {"value": (rr.loop + 1) / dt, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": "1 full C2 solve with the CPU oracle (reference kernel restated in numpy "
                         "+ LAPACK zgetrf/zgetrs, OpenBLAS threads=cores)",
               "m_found": int(rr.m), "loops": int(rr.loop), "seconds": dt}

    # DRAM bytes of one batched LU call (all its kernels) from the committed ncu
    # capture of the same workload (tools/prof_final.sh -> profiles/), or null
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_lu_traffic.json")) as f:
            tj = json.load(f)
        if tj.get("n") == n and tj.get("count") == w.ne:
            traffic = tj["dram_bytes_per_call"]
    except (OSError, ValueError, KeyError):
        pass

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64/c128",
            "data": "synthetic (seeded, workloads.c2_sygv)",
            "config": {"workload": "c2_dfeast_sygv N=4096 M0=160 Ne=8 (BASELINE configs[1])",
                       "global_batch": 1, "seq_len": n, "parallelism": f"contour-points x{world}",
                       "l2": "working set (A, B, 8 factors = 2.4 GB) larger than L2",
                       "m_found": int(r.m), "loops": loops, "info": int(r.info), "step_ms": step_ms},
            "lu_tflops": lu_tf, "lu_ms": lu_ms,
            "roofline": {"bound": "tensor", "achieved": lu_tf, "peak": FP64_DMMA_PEAK, "unit": "TFLOP/s",
                         "frac": lu_tf / FP64_DMMA_PEAK, "traffic": traffic,
                         "traffic_unit": "bytes per fb_zgetrf_batched call (Ne shifts), ncu dram read+write",
                         "kernel": "fb_zgetrf_batched (Ne shifted complex LUs per call, (8/3)N^3 flop each)",
                         "peak_source": "measured DMMA m8n8k4 f64 microbenchmark (tools/fp64_peak.cu); "
                                        "MEASURED_PEAKS.json has no FP64 entry"},
            "e2e": {"value": e2e_its / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
