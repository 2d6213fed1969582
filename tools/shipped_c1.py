"""BASELINE.md §4 "shipped reference path": feastlib.feast_sy exactly as
published (its own pure-Python LU and solves) on config 1 (dfeast_syev,
N = 2000, M0 = 150, Ne = 8), timed once on this host's cores, next to the
oracle path (feastlib's kernel + LAPACK) -- test/bench infrastructure, run by
hand: python tools/shipped_c1.py > profiles/rNN_shipped_c1.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
threads = len(os.sched_getaffinity(0))
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
import numpy as np  # noqa: E402

from oracle import ref  # noqa: E402
from paper_1203_4031_b200 import workloads as W  # noqa: E402

w = W.c1_syev()
out = {"workload": "c1_dfeast_syev N=2000 M0=150 Ne=8", "cores": threads}
t0 = time.perf_counter()
r = ref.reference_solve(w)
dt = time.perf_counter() - t0
out["oracle_path"] = {"seconds": dt, "iterations_per_s": (r.loop + 1) / dt, "info": int(r.info), "m": int(r.m),
                      "loops": int(r.loop), "max_res": float(np.max(r.res[:r.m]))}
t0 = time.perf_counter()
s = ref.shipped_solve(w)
dt = time.perf_counter() - t0
out["shipped_path"] = {"seconds": dt, "iterations_per_s": (s.loop + 1) / dt, "info": int(s.info), "m": int(s.m),
                       "loops": int(s.loop), "max_res": float(np.max(s.res[:s.m])),
                       "max_rel_dlambda_vs_oracle_path": float(np.abs(s.e[:s.m] - r.e[:r.m]).max() / 0.05)}
print(json.dumps(out))
