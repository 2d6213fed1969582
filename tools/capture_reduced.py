"""Capture the reduced problems (A_Q, B_Q) of a FEAST run and the GPU reduced
solver's answers (eps, Phi), for offline comparison with the reference's
generalized_eig on identical inputs.  Usage: capture_reduced.py c3 out.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1203_4031_b200 as fb  # noqa: E402
from paper_1203_4031_b200 import device as D  # noqa: E402
from paper_1203_4031_b200 import workloads as W  # noqa: E402

tag = sys.argv[1]
out = sys.argv[2]
w = {"c1": W.c1_syev, "c2": W.c2_sygv, "c3": W.c3_heev}[tag]()
calls = []
orig = D.Device.reduced_eig


def rec(self, Aq, Bq, m, eps_ptr, Phi):
    a = self.download(Aq.rows_view(0, m).cols_view(0, m))
    b = self.download(Bq.rows_view(0, m).cols_view(0, m))
    st = orig(self, Aq, Bq, m, eps_ptr, Phi)
    torch.cuda.synchronize()
    phi = self.download(Phi.rows_view(0, m).cols_view(0, m))
    calls.append((m, st, a, b, phi, eps_ptr))
    return st


D.Device.reduced_eig = rec
fn = fb.feast_he if w.hermitian else fb.feast_sy
r = fn(w.a, w.emin, w.emax, w.m0, b=w.b, fpm=w.fpm())
print("run", r.info, r.m0, r.loop, r.m, "maxres %.2e" % r.res[:r.m].max())
save = {}
for k, (m, st, a, b, phi, _) in enumerate(calls[-3:]):
    save[f"a{k}"], save[f"b{k}"], save[f"phi{k}"] = a, b, phi
    save[f"m{k}"] = np.array([m, st])
save["e_final"] = r.e
save["res_final"] = r.res
np.savez_compressed(out, **save)
print("calls", len(calls), [c[0] for c in calls])
