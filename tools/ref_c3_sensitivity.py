"""The REFERENCE kernel (feastlib SymmetricRci/HermitianRci, driven by the
LAPACK caller of tests/golden/make_golden.py) on config 3 with A scaled by
(1 + k*2^-52): shows that the reference's own loop count moves under
rounding-level perturbations (the M0 shrink at loop 0 is decided by rounding).
Runs in the build container (needs /root/reference).  Usage:
    python tools/ref_c3_sensitivity.py 1 2 > profiles/r01_c3_ref_sensitivity.txt
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import make_golden as mg  # noqa: E402
from paper_1203_4031_b200 import workloads as W  # noqa: E402

w = W.c3_heev()
a0 = w.a.copy()
print("# reference kernel + LAPACK caller, C3 (N=8192 M0=256 Ne=16 [-0.02,0.02]), A <- A*(1+k*2^-52)", flush=True)
for k in [int(v) for v in sys.argv[1:]] or [1, 2]:
    w.a = a0 * (1.0 + k * 2.0 ** -52)
    r, hist, wall, t = mg.run_kernel_lapack(w)
    print(f"ref c3 k={k}: info={r.info} loop={r.loop} m0={r.m0} m={r.m} "
          f"maxres={np.max(r.res[:r.m]):.2e} wall={wall:.0f}s", flush=True)
