"""One full FEAST solve of a BASELINE config (default C2) for launch lists / timing.
Usage: python tools/prof_solve.py [c1|c2|c3|c4s|...] [warm]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1203_4031_b200 as fb
from paper_1203_4031_b200 import workloads as W

tag = sys.argv[1] if len(sys.argv) > 1 else "c2"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = {"c1": W.c1_syev, "c2": W.c2_sygv, "c3": W.c3_heev}.get(tag, lambda: W.scaled(tag))()
dev = torch.device("cuda", 0)
A = torch.from_numpy(w.a).to(dev)
B = None if w.b is None else torch.from_numpy(w.b).to(dev)
fn = fb.feast_he if w.hermitian else fb.feast_sy
for i in range(warm + 1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn(A, w.emin, w.emax, w.m0, b=B, fpm=w.fpm())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{tag}: info={r.info} m={r.m} loop={r.loop} m0={r.m0} {dt * 1e3:.1f} ms "
          f"({(r.loop + 1) / dt:.2f} it/s) maxres={max(r.res[:r.m]) if r.m else 0:.2e}", flush=True)
