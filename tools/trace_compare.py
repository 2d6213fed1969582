"""Per-loop (#eig, trace, epsout, max-res) of the GPU run vs the reference golden history."""
import contextlib
import io
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1203_4031_b200 as fb
from paper_1203_4031_b200 import workloads as W

tag = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = {"c1": W.c1_syev, "c2": W.c2_sygv, "c3": W.c3_heev}[tag]()
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", f"full_{tag}.npz"))
fpm = w.fpm()
fpm.set_slot(1, 1)
A = torch.from_numpy(w.a).cuda()
B = None if w.b is None else torch.from_numpy(w.b).cuda()
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    r = (fb.feast_he if w.hermitian else fb.feast_sy)(A, w.emin, w.emax, w.m0, b=B, fpm=fpm)
hist = [[float(v) for v in l.split()] for l in buf.getvalue().splitlines() if len(l.split()) == 5 and l.split()[0].isdigit()]
ref = g["history"]
print(f"{tag}: gpu loop={r.loop} m0={r.m0} m={r.m}; reference loop={int(g['scal'][1])} m0={int(g['scal'][3])}")
for i in range(max(len(hist), len(ref))):
    a = hist[i] if i < len(hist) else [np.nan] * 5
    b = ref[i] if i < len(ref) else [np.nan] * 5
    print(f"{i:3d} gpu #eig={a[1]:5.0f} trace={a[2]: .15e} eps={a[3]:.3e} res={a[4]:.2e} | "
          f"ref #eig={b[1]:5.0f} trace={b[2]: .15e} eps={b[3]:.3e} res={b[4]:.2e}")
