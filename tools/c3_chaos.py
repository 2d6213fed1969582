"""Loop count of the full C3 solve under rounding-level perturbations of A
(A * (1 + k*2^-52)): shows how sensitive the M0-shrink dynamics are."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1203_4031_b200 as fb
from paper_1203_4031_b200 import workloads as W

tag = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = {"c1": W.c1_syev, "c2": W.c2_sygv, "c3": W.c3_heev}[tag]()
A0 = torch.from_numpy(w.a).cuda()
B = None if w.b is None else torch.from_numpy(w.b).cuda()
for k in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    A = A0 * (1.0 + k * 2.0 ** -52)
    r = (fb.feast_he if w.hermitian else fb.feast_sy)(A, w.emin, w.emax, w.m0, b=B, fpm=w.fpm())
    print(f"{tag} k={k}: info={r.info} loop={r.loop} m0={r.m0} m={r.m} maxres={max(r.res[:r.m]):.2e}", flush=True)
