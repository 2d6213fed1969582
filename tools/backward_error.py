"""Per-shift backward error of the GPU shifted LU + solve against LAPACK.

For S = z*B - A at the contour points of a C3/C5-type pencil:
    berr = max_j ||S x_j - y_j||_inf / (||S||_inf ||x_j||_inf + ||y_j||_inf)
for x from (i) LAPACK zgetrf/zgetrs, (ii) the GPU factor + GPU sweeps,
(iii) the GPU factor with LAPACK's substitution (isolates factor vs sweep).
Usage: python tools/backward_error.py [n] [nrhs] [ne] [gen]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.linalg as sl  # noqa: E402

from paper_1203_4031_b200.device import get_device  # noqa: E402
from paper_1203_4031_b200.quadrature import build_contour, gauss_legendre  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
m = int(sys.argv[2]) if len(sys.argv) > 2 else 64
ne = int(sys.argv[3]) if len(sys.argv) > 3 else 16
gen = len(sys.argv) > 4 and sys.argv[4] == "gen"
rng = np.random.default_rng(3)
g = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
a = (g + g.conj().T) / (2 * np.sqrt(n))
del g
if gen:
    h = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    b = np.eye(n) + 0.05 * (h @ h.conj().T) / n
    del h
    emin, emax = -0.0174, 0.0174
else:
    b = None
    emin, emax = -0.02, 0.02
ct = build_contour(gauss_legendre(ne), emin, emax)
dev = get_device()
torch = dev.torch
_c = ctypes.c_void_p
y = rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))


def berr(S, x, nS):
    r = S @ x - y
    num = np.abs(r).max(axis=0)   # inf-norm per column (approx: max modulus)
    den = nS * np.abs(x).max(axis=0) + np.abs(y).max(axis=0)
    return float((num / den).max())


def fwd(x, xr):
    return float((np.abs(x - xr).max(axis=0) / np.abs(xr).max(axis=0)).max())


print(f"n={n} nrhs={m} ne={ne} {'generalized' if gen else 'standard'}", flush=True)
order = np.argsort(np.abs(ct.z.imag))
for k in (int(order[0]), int(order[len(order) // 2]), int(order[-1])):
    z = complex(ct.z[k])
    S = z * (b if gen else np.eye(n)) - a
    nS = float(np.abs(S).sum(axis=1).max())
    t0 = time.time()
    lu = sl.lu_factor(S, check_finite=False)
    x_lap = sl.lu_solve(lu, y, check_finite=False)
    t_lap = time.time() - t0
    # one step of fp64 iterative refinement on the LAPACK solution: x_ref
    x_ref = x_lap + sl.lu_solve(lu, y - S @ x_lap, check_finite=False)
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
    lu_g = dev.download(LU)
    pv = piv.cpu().numpy().astype(np.int32)
    x_gf = sl.lu_solve((lu_g, pv), y, check_finite=False)
    # factor backward error ||P S - L U|| / ||S|| on a 256-column sample
    cols = np.arange(0, n, max(1, n // 256))
    L = np.tril(lu_g, -1) + np.eye(n)
    U = np.triu(lu_g)
    perm = np.arange(n)
    for i, p in enumerate(pv):
        perm[i], perm[p] = perm[p], perm[i]
    PS = S[perm][:, cols]
    fe_g = np.abs(PS - L @ U[:, cols]).max() / np.abs(S).max()
    Ll = np.tril(lu[0], -1) + np.eye(n)
    Ul = np.triu(lu[0])
    perm = np.arange(n)
    for i, p in enumerate(lu[1]):
        perm[i], perm[p] = perm[p], perm[i]
    fe_l = np.abs(S[perm][:, cols] - Ll @ Ul[:, cols]).max() / np.abs(S).max()
    print(f"z[{k}]={z:.6f} |Im z|={abs(z.imag):.2e}  LAPACK {t_lap:.1f}s", flush=True)
    print(f"   backward err: LAPACK {berr(S, x_lap, nS):.2e}  GPU {berr(S, x_gpu, nS):.2e}  "
          f"GPU-factor+LAPACK-trsm {berr(S, x_gf, nS):.2e}", flush=True)
    print(f"   forward err vs refined: LAPACK {fwd(x_lap, x_ref):.2e}  GPU {fwd(x_gpu, x_ref):.2e}  "
          f"GPU-factor+LAPACK-trsm {fwd(x_gf, x_ref):.2e}", flush=True)
    print(f"   factor err |PS-LU|max/|S|max: LAPACK {fe_l:.2e}  GPU {fe_g:.2e}   "
          f"max|L| LAPACK {np.abs(Ll).max():.2f} GPU {np.abs(L).max():.2f}", flush=True)
    del LU, W, lu_g, L, U, Ll, Ul, lu
