"""Kernel timeline of one warm FEAST solve through torch.profiler (CUPTI):
GPU busy time (union of kernel intervals, overlap across streams counted
once), idle gaps, per-kernel totals, and the share of each phase.  Unlike an
ncu launch list, kernels run concurrently and at full clocks here.

Usage: python tools/trace_step.py [c1|c2|c3|c4] [--out gpurun_out/trace_c2.json]
"""
import argparse
import collections
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1203_4031_b200 as fb  # noqa: E402
from paper_1203_4031_b200 import workloads as W  # noqa: E402


def run(w, A, B):
    if w.kind == "band":
        return fb.feast_sb(w.a, w.kla, w.emin, w.emax, w.m0, b=w.b, klb=w.klb, uplo=w.uplo, fpm=w.fpm())
    fn = fb.feast_he if w.hermitian else fb.feast_sy
    return fn(A, w.emin, w.emax, w.m0, b=B, fpm=w.fpm())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", nargs="?", default="c2")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    w = {"c1": W.c1_syev, "c2": W.c2_sygv, "c3": W.c3_heev, "c4": W.c4_sbgv}[args.cfg]()
    A = torch.from_numpy(w.a).cuda() if w.kind == "dense" else None
    B = torch.from_numpy(w.b).cuda() if (w.kind == "dense" and w.b is not None) else None
    for _ in range(2):
        r = run(w, A, B)
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        r = run(w, A, B)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in evs)
    per = collections.defaultdict(lambda: [0, 0.0])
    for s, e, n in iv:
        k = n.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:60]
        per[k][0] += 1
        per[k][1] += (e - s)
    busy, cur_s, cur_e, gaps = 0.0, None, None, []
    for s, e, _ in iv:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
                gaps.append(s - cur_e)
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        busy += cur_e - cur_s
    span = (iv[-1][1] - iv[0][0]) if iv else 0.0
    ksum = sum(v[1] for v in per.values())
    print(f"{args.cfg}: loop={r.loop} m={r.m} wall {wall * 1e3:.1f} ms; kernel span {span / 1e3:.1f} ms, "
          f"busy {busy / 1e3:.1f} ms ({100 * busy / max(span, 1):.0f}%), sum of kernels {ksum / 1e3:.1f} ms, "
          f"{len(iv)} kernels, gaps {sum(gaps) / 1e3:.1f} ms (>20us: {sum(g for g in gaps if g > 20) / 1e3:.1f} ms)")
    for k, (c, t) in sorted(per.items(), key=lambda x: -x[1][1])[:22]:
        print(f"  {t / 1e3:9.3f} ms {100 * t / max(ksum, 1):5.1f}% {c:6d}  avg {t / c:8.1f} us  {k}")
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"wall_ms": wall * 1e3, "span_ms": span / 1e3, "busy_ms": busy / 1e3,
                       "kernels": {k: v for k, v in per.items()}}, f, indent=1)


if __name__ == "__main__":
    main()
