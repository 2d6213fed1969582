"""The REFERENCE kernel (feastlib SymmetricRci/HermitianRci driven by the
LAPACK caller of tests/golden/make_golden.py) on a workload with A scaled by
(1 + k*2^-52): how far the reference's own loop count and M0 shrink move
under rounding-level perturbations.  Runs in the build container (needs
/root/reference).  Usage: python tools/ref_sensitivity.py c3s 0 1 2 3 4 5
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import make_golden as mg  # noqa: E402
from paper_1203_4031_b200 import workloads as W  # noqa: E402

tag = sys.argv[1]
ks = [int(v) for v in sys.argv[2:]] or [0, 1, 2]
w = W.scaled(tag) if tag.endswith("s") else {"c3": W.c3_heev}[tag]()
a0 = w.a.copy()
print(f"# reference kernel + LAPACK caller, {tag} (N={w.n} M0={w.m0} Ne={w.ne}), A <- A*(1+k*2^-52)", flush=True)
for k in ks:
    w.a = a0 * (1.0 + k * 2.0 ** -52)
    r, hist, wall, t = mg.run_kernel_lapack(w)
    print(f"ref {tag} k={k}: info={r.info} loop={r.loop} m0={r.m0} m={r.m} "
          f"maxres={np.max(r.res[:r.m]):.2e} wall={wall:.1f}s", flush=True)
