"""Forward error of the GPU shifted solve and dense multiply against LAPACK /
numpy, both measured against an iteratively refined solution whose residuals
are accumulated in extended precision (np.clongdouble).  C3-type pencil,
contour point nearest the real axis (the worst-conditioned shift).
Usage: python tools/accuracy.py [n] [nrhs]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.linalg as sl  # noqa: E402

from paper_1203_4031_b200.device import get_device  # noqa: E402
from paper_1203_4031_b200.quadrature import build_contour, gauss_legendre  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
m = int(sys.argv[2]) if len(sys.argv) > 2 else 32
rng = np.random.default_rng(3)
g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
a = (g + g.conj().T) / (2 * np.sqrt(n))
ct = build_contour(gauss_legendre(16), -0.02, 0.02)
dev = get_device()
_c = ctypes.c_void_p
P = ctypes.c_void_p
y = rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))
al = a.astype(np.clongdouble)


def refine(S, Sl, x0, lu):
    x = x0.copy()
    for _ in range(3):
        r = (y.astype(np.clongdouble) - Sl @ x.astype(np.clongdouble)).astype(np.complex128)
        x = x + sl.lu_solve(lu, r)
    return x


for k in (int(np.argmin(np.abs(ct.z.imag))), 0, len(ct.z) // 2):
    z = complex(ct.z[k])
    S = z * np.eye(n) - a
    Sl = z * np.eye(n, dtype=np.clongdouble) - al
    lu = sl.lu_factor(S)
    x_lap = sl.lu_solve(lu, y)
    x_true = refine(S, Sl, x_lap, lu)
    torch = dev.torch
    LU = dev.upload(S, cplx=True)
    piv = torch.empty(n, dtype=torch.int32, device=dev.tdev)
    dinv = torch.empty(int(dev.lib.fb_zgetrf_dinv_doubles(n)), dtype=torch.float64, device=dev.tdev)
    info = torch.empty(1, dtype=torch.int32, device=dev.tdev)
    dev.check(dev.lib.fb_zgetrf(dev.h, n, _c(LU.re), _c(LU.im), LU.ld, _c(piv.data_ptr()), _c(dinv.data_ptr()),
                                _c(info.data_ptr())), "zgetrf")
    W = dev.upload(y, cplx=True)
    dev.check(dev.lib.fb_zgetrs(dev.h, n, m, _c(LU.re), _c(LU.im), LU.ld, _c(piv.data_ptr()),
                                _c(dinv.data_ptr()), 0, _c(W.re), _c(W.im), W.ld), "zgetrs")
    x_gpu = dev.download(W)
    nrm = np.abs(x_true).max()
    # the GPU factor itself, used with LAPACK-style substitution (isolates factor vs sweep error)
    lu_g = dev.download(LU)
    pv = piv.cpu().numpy()
    x_gf = sl.lu_solve((lu_g, pv), y)
    e_lap = np.abs(x_lap - x_true).max() / nrm
    e_gpu = np.abs(x_gpu - x_true).max() / nrm
    e_gf = np.abs(x_gf - x_true).max() / nrm
    print(f"z[{k}]={z:.5f}: fwd err LAPACK {e_lap:.2e}  GPU {e_gpu:.2e}  (GPU factor + LAPACK trsm {e_gf:.2e})",
          flush=True)

# dense multiply A @ Q
q = rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))
ex = (al @ q.astype(np.clongdouble)).astype(np.complex128)
A = dev.upload(a, cplx=True)
Q = dev.upload(q, cplx=True)
C = dev.empty(n, m, True)
dev.gemm("N", "N", n, m, n, 1.0, A, Q, 0.0, C, cplx=True)
c_gpu = dev.download(C)
c_np = a @ q
nrm = np.abs(ex).max()
print(f"A@Q: max rel err numpy {np.abs(c_np - ex).max() / nrm:.2e}  GPU {np.abs(c_gpu - ex).max() / nrm:.2e}")
