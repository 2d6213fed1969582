"""Full C4 (dfeast_sbgv N=1e6, kd=16, M0=96, Ne=8) on the GPU against the
reference-kernel golden (tests/golden/full_c4.npz): m, loop, eigenvalues,
residuals, wall time.  Usage: python tools/run_c4.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1203_4031_b200 as fb
from paper_1203_4031_b200 import workloads as W

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
t0 = time.perf_counter()
w = W.c4_sbgv()
print(f"workload built in {time.perf_counter() - t0:.1f}s", flush=True)
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                         "full_c4.npz"))
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = fb.feast_sb(w.a, w.kla, w.emin, w.emax, w.m0, b=w.b, klb=w.klb, uplo=w.uplo, fpm=w.fpm())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    m = res.m
    ref_e = g["e"][: int(g["scal"][0])]
    scale = max(abs(w.emin), abs(w.emax))
    de = np.abs(np.sort(res.e[:m]) - np.sort(ref_e)).max() / scale if m == len(ref_e) else float("nan")
    print(f"c4: info={res.info} m={m} (ref {int(g['scal'][0])}) loop={res.loop} (ref {int(g['scal'][1])}) "
          f"max|dl|/s={de:.2e} maxres={max(res.res[:m]):.2e} factorizations={res.factorizations} "
          f"{dt * 1e3:.1f} ms ({(res.loop + 1) / dt:.2f} it/s)", flush=True)
