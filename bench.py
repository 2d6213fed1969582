"""FEAST B200 benchmark (contract: one JSON line on rank 0).

Workload (default --config c2 = BASELINE.json configs[1]): dfeast_sygv,
N = 4096 dense real symmetric generalized pencil, M0 = 160, Ne = 8, interval
around the ~100 eigenvalues nearest 0; seeded synthetic matrices
(workloads.py; the paper's datasets are not shipped).  --config c1 | c3 | c4
select the other single-GPU BASELINE configurations (c3 = zfeast_heev
N = 8192, Ne = 16: the multi-GPU scaling configuration).  One STEP = one
complete FEAST solve (factorize all Ne shifts, all refinement passes to
convergence).

  value   FEAST iterations/s = sum(loop+1) / device time, inputs resident in HBM
          (first-pass factorizations included)
  steady  the same passes / (time - factorization time): cached factors
  points  contour-point throughput = Ne * sum(loop+1) / time
  e2e     value's metric through the public API with pinned HOST inputs: H2D of
          A and B and D2H of the result (e, X, res) inside the timed region
  lu      shifted-LU FP64 TFLOP/s = (8/3) N^3 per factorization / its duration
          (CUDA events on the launching stream) -> the roofline object
  banded  config 4 (dfeast_sbgv N = 1e6, kd = 16) measured in the same run:
          one contour pass of the band solve (8 shifts x 96 right-hand sides)
          as GB/s and FP64 fraction, the band multiply, and a full solve
  --gpus N > 1: one rank per GPU (NCCL); started by the driver's torchrun, or
          spawned here when WORLD_SIZE is absent.  Contour points are sharded
          over the ranks (point k -> rank k mod N), dense pencils also shard
          the rows of the N^2 M0 products ("strong" scaling: the job is fixed).
  --impl reference: the reference's own RCI kernel (feastlib, unmodified, from
          oracle/_ref) pumped by its own run_rci and answered by LAPACK
          zgetrf/zgetrs on the host cores -- same workload, metric and config
          keys; falls back to the oracle's restatement if oracle/_ref is absent.
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


FP64_DFMA_PEAK = 34.2   # TFLOP/s, measured DFMA microbenchmark (same tool / profile)
CONFIGS = {
    "c1": ("c1_syev", "c1_dfeast_syev N=2000 M0=150 Ne=8 (BASELINE configs[0])"),
    "c2": ("c2_sygv", "c2_dfeast_sygv N=4096 M0=160 Ne=8 (BASELINE configs[1])"),
    "c3": ("c3_heev", "c3_zfeast_heev N=8192 M0=256 Ne=16 (BASELINE configs[2])"),
    "c4": ("c4_sbgv", "c4_dfeast_sbgv N=1000000 kd=16 M0=96 Ne=8 (BASELINE configs[3])"),
}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"
    except (OSError, ValueError, KeyError):
        return 6550.0, "B200_PROFILING.md fallback"


def _config(args, w, world, loops, info, step_ms, m_found):
    """config object shared by both arms (same keys: the driver compares them)."""
    work = (f"A, B and {w.ne} factors larger than L2" if w.kind == "dense"
            else "band factors (6.3 GB) and right-hand sides larger than L2")
    return {"workload": CONFIGS[args.config][1], "global_batch": 1, "seq_len": int(w.n),
            "parallelism": f"contour-points x{world}" + (" + row-sharded products" if world > 1 and w.kind == "dense" else ""),
            "l2": work, "m_found": int(m_found), "loops": [int(v) for v in loops], "info": int(info),
            "step_ms": step_ms}


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region, in-process
    through NVML (no nvidia-smi subprocesses competing with the launching
    thread); falls back to nvidia-smi when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits: hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
    BITS = (0x8, 0x40, 0x20, 0x4)

    def __init__(self, index, disabled=False):
        self.index = index
        self.disabled = disabled
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
        # NVML queries take the driver lock for tens of ms and stall the launching
        # thread (a +40-60 ms step whenever one lands inside it): first sample
        # 0.15 s into the timed region, then one per second
        if self._stop.wait(0.15):
            return
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
            self._stop.wait(1.0)

    def __enter__(self):
        if not self.disabled:
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
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


def cpu_reference_solve(w):
    """One CPU solve of the workload: feastlib's own kernel + run_rci answered
    by LAPACK (oracle/_ref present) or the oracle's restatement of it."""
    from oracle import ref
    t0 = time.perf_counter()
    if ref.available():
        r = ref.reference_solve(w)
        kind = "reference"
    else:
        from oracle import oracle_feast_he, oracle_feast_sy
        from oracle.feast_oracle import oracle_feast_sb
        fpm = [0] + [w.fpm().slot(i) for i in range(1, 65)]
        if w.kind == "band":
            r = oracle_feast_sb(w.a, w.kla, w.emin, w.emax, w.m0, b=w.b, klb=w.klb, uplo=w.uplo, fpm=fpm)
        else:
            fn = oracle_feast_he if w.hermitian else oracle_feast_sy
            r = fn(w.a, w.emin, w.emax, w.m0, b=w.b, fpm=fpm, reduced="lapack")
        kind = "port"
    return r, time.perf_counter() - t0, kind


_CPU_SAMPLE = {"reference": "full solves by the reference's own RCI kernel + run_rci (feastlib, unmodified, "
                            "oracle/_ref) answered by LAPACK zgetrf/zgetrs / zgbtrf/zgbtrs, OpenBLAS threads=cores",
               "port": "full solves by the oracle (reference kernel restated in numpy + LAPACK), OpenBLAS threads=cores"}


def run_reference(args):
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    from paper_1203_4031_b200 import workloads as W
    w = getattr(W, CONFIGS[args.config][0])()
    for _ in range(args.warmup):
        cpu_reference_solve(w)
    total_it, total_t, loops, step_ms = 0, 0.0, [], []
    for _ in range(args.steps):
        r, dt, kind = cpu_reference_solve(w)
        total_it += r.loop + 1
        total_t += dt
        loops.append(r.loop)
        step_ms.append(round(1e3 * dt, 2))
    v = total_it / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64/c128",
        "data": f"synthetic (seeded, workloads.{CONFIGS[args.config][0]})",
        "config": _config(args, w, max(1, args.gpus), loops, r.info, step_ms, r.m),
        "contour_points_per_s": w.ne * v,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{args.steps} {_CPU_SAMPLE[kind]}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def banded_leg(dev, torch, reps=5):
    """Config 4 on this GPU: one contour pass of the band solve (all Ne shifts
    x M0 right-hand sides: sweeps + interface + correction/accumulation) timed
    with CUDA events, the band multiply, and one full feast_sb solve."""
    import paper_1203_4031_b200 as fb
    from paper_1203_4031_b200 import workloads as W
    from paper_1203_4031_b200.banded import DeviceBandOps, expand_band_device
    from paper_1203_4031_b200.quadrature import build_contour, gauss_legendre
    w = W.c4_sbgv()
    n, kl, m0, ne = w.n, w.kla, w.m0, w.ne
    FA = expand_band_device(dev, w.a, w.kla, w.uplo, False, kl)
    FB = expand_band_device(dev, w.b, w.klb, w.uplo, False, kl)
    FBc = expand_band_device(dev, w.b, w.klb, w.uplo, False, w.klb)
    ops = DeviceBandOps(dev, FA, FB, kl, False, mv_b=(FBc, w.klb))
    ct = build_contour(gauss_legendre(ne), w.emin, w.emax)
    zs = [complex(z) for z in ct.z]
    e0, e1 = _events(torch)
    torch.cuda.synchronize()
    e0.record()
    ops.prefactorize(zs)
    e1.record()
    torch.cuda.synchronize()
    t_fac = e0.elapsed_time(e1)
    Y = dev.empty(n, m0, False)
    Y.plane(0).copy_(torch.rand(n, m0, dtype=torch.float64, device=dev.tdev) - 0.5)
    Q = dev.zeros(n, m0, False)
    X = dev.empty(n, m0, False)
    spec = [(z, False, 0, ct.weights[k], ct.theta[k]) for k, z in enumerate(zs)]

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = _events(torch)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    t_pass = timed(lambda: ops.solve_pass_accumulate(Y, spec, ct.radius, Q))
    t_mva = timed(lambda: ops.multiply_a(Y, X))
    t_mvb = timed(lambda: ops.multiply_b(Y, X))
    del ops, FA, FB, FBc, Y, Q, X
    torch.cuda.empty_cache()
    fb.feast_sb(w.a, w.kla, w.emin, w.emax, m0, b=w.b, klb=w.klb, uplo=w.uplo, fpm=w.fpm())   # warm-up (allocations)
    a, b = _events(torch)
    a.record()
    r = fb.feast_sb(w.a, w.kla, w.emin, w.emax, m0, b=w.b, klb=w.klb, uplo=w.uplo, fpm=w.fpm())
    b.record()
    torch.cuda.synchronize()
    t_solve = a.elapsed_time(b)
    hbm, src = _hbm_peak()
    bytes_pass = ne * ((3 * kl + 1) * n * 16 + 2 * n * m0 * 16)      # 3.856 GB per shift
    flop_pass = ne * 8.0 * 3 * kl * n * m0                           # 3.69e10 per shift
    mv_bytes = (2 * kl + 1) * n * 8 + 2 * n * m0 * 8
    mvb_bytes = (2 * w.klb + 1) * n * 8 + 2 * n * m0 * 8
    gbs = bytes_pass / t_pass / 1e6
    return {
        "workload": CONFIGS["c4"][1],
        "solve_pass_ms": t_pass, "solve_pass_gbs": gbs, "hbm_frac": gbs / hbm, "hbm_peak_gbs": hbm,
        "hbm_peak_source": src,
        "solve_pass_tflops": flop_pass / t_pass / 1e9, "fp64_frac": flop_pass / t_pass / 1e9 / FP64_DFMA_PEAK,
        "fp64_peak_tflops": FP64_DFMA_PEAK,
        "what": "one contour pass: Ne=8 shifts x M0=96 right-hand sides, partition sweeps + interface solve + "
                "fused spike-correction/quadrature kernel (fb_band_solve_accumulate), CUDA events; bytes and "
                "flop are BASELINE.md §3's algorithmic counts",
        "factor_ms": t_fac, "matvec_a_ms": t_mva, "matvec_a_gbs": mv_bytes / t_mva / 1e6,
        "matvec_b_ms": t_mvb, "matvec_b_gbs": mvb_bytes / t_mvb / 1e6,
        "full_solve": {"ms": t_solve, "iterations_per_s": (r.loop + 1) / (t_solve / 1e3),
                       "contour_points_per_s": ne * (r.loop + 1) / (t_solve / 1e3),
                       "info": int(r.info), "m_found": int(r.m), "loops": int(r.loop),
                       "max_res": float(r.res[:r.m].max()) if r.m else None,
                       "inputs": "host band arrays (272 MB uploaded inside the timed region)"},
    }


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1203_4031_b200 as fb
    from paper_1203_4031_b200 import distributed as D
    from paper_1203_4031_b200 import workloads as W
    from paper_1203_4031_b200.banded import DeviceBandOps
    from paper_1203_4031_b200.dense import DeviceDenseOps
    from paper_1203_4031_b200.device import get_device

    world, rank, local = _dist_env()
    if world != max(1, args.gpus):
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = get_device()
    w = getattr(W, CONFIGS[args.config][0])()
    n, m0 = w.n, w.m0
    band = w.kind == "band"
    A_d = torch.from_numpy(w.a).to(dev.tdev)
    B_d = None if w.b is None else torch.from_numpy(w.b).to(dev.tdev)
    A_h = torch.from_numpy(w.a).pin_memory()
    B_h = None if w.b is None else torch.from_numpy(w.b).pin_memory()
    fpm = w.fpm()

    def solve_once(a, b):
        if band:
            fn = D.feast_sb_distributed if world > 1 else fb.feast_sb
            return fn(a, w.kla, w.emin, w.emax, m0, b=b, klb=w.klb, uplo=w.uplo, fpm=fpm.copy())
        if world > 1:
            fn = D.feast_he_distributed if w.hermitian else D.feast_sy_distributed
        else:
            fn = fb.feast_he if w.hermitian else fb.feast_sy
        return fn(a, w.emin, w.emax, m0, b=b, fpm=fpm.copy())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(t):
        if world > 1:
            tt = torch.tensor([t], device=dev.tdev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return float(tt.item())
        return t

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
    ev0, ev1 = _events(torch)
    its, loops = 0, []
    fac_events = []
    DeviceDenseOps.lu_event_sink = fac_events
    DeviceBandOps.factor_event_sink = fac_events
    with ClockSampler(local, disabled=args.no_clocks) as clk:
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
    DeviceBandOps.factor_event_sink = None
    launches = dev.launches() - launches0
    t = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
    value = its / t
    # factorization time inside the timed region (events on the launching stream)
    t_fac = max_over_ranks(sum(a.elapsed_time(b) for a, b, _ in fac_events) / 1e3)
    n_fac = sum(c for _, _, c in fac_events)
    steady = its / max(t - t_fac, 1e-9)

    # -- end to end through the public API with pinned host inputs ----------
    barrier()
    e0, e1 = _events(torch)
    e2e_its = 0
    e0.record()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r2 = solve_once(A_h, B_h)        # uploads A, B; result arrays come back to the host
        e2e_its += r2.loop + 1
    e1.record()
    barrier()
    t_e2e = max_over_ranks(max(e0.elapsed_time(e1) / 1e3, time.perf_counter() - t0))
    gc.enable()
    esz = 16 if w.hermitian else 8
    h2d = int(A_h.numel() * A_h.element_size() + (0 if B_h is None else B_h.numel() * B_h.element_size()))
    d2h = n * m0 * esz + 2 * m0 * 8

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
        rr, dt, kind = cpu_reference_solve(w)
        cpu = {"value": (rr.loop + 1) / dt, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": "1 " + _CPU_SAMPLE[kind], "m_found": int(rr.m), "loops": int(rr.loop), "seconds": dt}

    banded = None
    if rank == 0 and world == 1 and not args.no_banded and not band:
        del A_d, B_d
        torch.cuda.empty_cache()
        banded = banded_leg(dev, torch)

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64/c128",
            "data": f"synthetic (seeded, workloads.{CONFIGS[args.config][0]})",
            "config": _config(args, w, world, loops, r.info, step_ms, r.m),
            "steady_state": {"value": steady, "unit": UNIT,
                             "how": "same passes / (timed region - batched factorization time, CUDA events)",
                             "factorization_s": t_fac, "factorizations": n_fac},
            "contour_points_per_s": w.ne * value,
            "e2e": {"value": e2e_its / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if band:
            hbm, src = _hbm_peak()
            line["roofline"] = {"bound": "hbm", "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None,
                                "traffic": None, "note": "run the default config for the banded roofline object"}
        else:
            # LU roofline: batched factorizations inside the timed region
            lu_ms = 1e3 * t_fac / max(1, n_fac)
            lu_flops = 8.0 / 3.0 * n ** 3
            lu_tf = lu_flops / (lu_ms / 1e3) / 1e12 if lu_ms > 0 else 0.0
            # DRAM bytes of one batched LU call (all its kernels) from the committed ncu
            # capture of the same workload (tools/prof_final.sh -> profiles/), or null
            traffic = None
            try:
                with open(os.path.join(ROOT, "profiles", "r02_lu_traffic.json")) as f:
                    tj = json.load(f)
                if tj.get("n") == n and tj.get("count") == w.ne and world == 1:
                    traffic = tj["dram_bytes_per_call"]
            except (OSError, ValueError, KeyError):
                pass
            line["lu_tflops"] = lu_tf
            line["lu_ms"] = lu_ms
            line["roofline"] = {
                "bound": "tensor", "achieved": lu_tf, "peak": FP64_DMMA_PEAK, "unit": "TFLOP/s",
                "frac": lu_tf / FP64_DMMA_PEAK, "traffic": traffic,
                "traffic_unit": "bytes per fb_zgetrf_batched call (Ne shifts), ncu dram read+write "
                                "(committed capture of this workload; 9x the 4.3 GB minimum, harmless at 37 flop/B)",
                "kernel": "fb_zgetrf_batched (this rank's shifted complex LUs per call, (8/3)N^3 flop each)",
                "peak_source": "measured DMMA m8n8k4 f64 microbenchmark (tools/fp64_peak.cu); "
                               "MEASURED_PEAKS.json has no FP64 entry"}
        if banded is not None:
            line["banded"] = banded
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-banded", action="store_true")
    ap.add_argument("--no-clocks", action="store_true",
                    help="diagnosis only: no NVML sampling thread during the timed region")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # started without torchrun: spawn the ranks (one per GPU) and relay the JSON line
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
               *sys.argv[1:]]
        return subprocess.call(cmd)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
