"""Full config 5 (zfeast_hegv, N = 32768, M0 = 512, Ne = 16) on one B200.

The CPU oracle cannot run this size (~30 h per pure-Python
LU; 16 LAPACK factors need 275 GB of host RAM), so parity is checked through
size-independent properties against independent computations on the same
pencil (cuSOLVER/cuBLAS through torch.linalg, test-only):
  * m = the Sylvester-inertia count in [Emin, Emax]: neg(A - Emax B) -
    neg(A - Emin B) from a block LDL^H (Haynsworth additivity; each pivot
    block's inertia from its eigenvalues) -- cuSOLVER's zheevd refuses
    N = 32768 (workspace overflow), so a full eigensolve is not available;
  * every residual <= 1e-10 (for a Hermitian-definite pencil the residual
    bounds the eigenvalue error: |lambda - lambda_true| <~ res * s * ||B||)
  * X is B-orthonormal: max |X^H B X - I| small.
Small n: the full eigenvalue list (torch.linalg.eigvalsh) is compared too.

Usage: python tools/c5_full.py [--n N] [--m0 M] [--emin E --emax E] [--no-inertia]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1203_4031_b200 as fb  # noqa: E402
from paper_1203_4031_b200 import workloads as W  # noqa: E402
from paper_1203_4031_b200.device import get_device  # noqa: E402

OUT = os.path.join(ROOT, "gpurun_out")


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


def independent_eigs(A, B):
    """Eigenvalues of the pencil (A, B): L = chol(B), C = L^-1 A L^-H, eigvalsh(C)."""
    t0 = time.perf_counter()
    L = torch.linalg.cholesky(torch.complex(B.plane(0), B.plane(1)))
    C = torch.complex(A.plane(0), A.plane(1))
    C = torch.linalg.solve_triangular(L, C, upper=False)
    C = torch.linalg.solve_triangular(L, C.conj().T, upper=False).conj().T
    del L
    C = 0.5 * (C + C.conj().T)
    ev = torch.linalg.eigvalsh(C).cpu().numpy()
    del C
    torch.cuda.empty_cache()
    log(f"independent eigvalsh done in {time.perf_counter() - t0:.1f}s")
    return ev


def inertia_neg(A, B, sigma, nb=2048):
    """Number of negative eigenvalues of H = A - sigma B (block LDL^H)."""
    t0 = time.perf_counter()
    n = A.rows
    H = torch.complex(A.plane(0), A.plane(1))
    H -= sigma * torch.complex(B.plane(0), B.plane(1))
    neg = 0
    for k in range(0, n, nb):
        e = min(n, k + nb)
        S = H[k:e, k:e]
        S = 0.5 * (S + S.conj().T)
        lam, V = torch.linalg.eigh(S)
        neg += int((lam < 0).sum().item())
        if e < n:
            # H22 -= H21 S^-1 H21^H with S^-1 = V diag(1/lam) V^H
            T = H[e:, k:e] @ V                      # (n-e, nb)
            H[e:, e:] -= (T / lam.unsqueeze(0)) @ T.conj().T
    del H
    torch.cuda.empty_cache()
    log(f"inertia at sigma={sigma!r}: neg={neg} ({time.perf_counter() - t0:.1f}s)")
    return neg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--m0", type=int, default=512)
    ap.add_argument("--emin", type=float, default=W.C5_INTERVAL[0])
    ap.add_argument("--emax", type=float, default=W.C5_INTERVAL[1])
    ap.add_argument("--no-inertia", action="store_true")
    ap.add_argument("--loops", type=int, default=None, help="cap fpm(4) (refinement passes)")
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    torch.cuda.set_device(0)
    dev = get_device()
    t0 = time.perf_counter()
    A, B = W.c5_device_planar(dev, n=args.n)
    torch.cuda.synchronize()
    log(f"pencil built on device in {time.perf_counter() - t0:.1f}s")
    report = {"n": args.n, "m0": args.m0}
    emin, emax = args.emin, args.emax
    ev = independent_eigs(A, B) if args.n <= 8192 else None
    if ev is not None:
        report["eigvalsh_count"] = int(((ev >= emin) & (ev <= emax)).sum())
    if not args.no_inertia:
        cnt = inertia_neg(A, B, emax) - inertia_neg(A, B, emin)
        report["inertia_count"] = cnt
        log(f"inertia count in [{emin}, {emax}]: {cnt}")
    fpm = fb.feastinit()
    fpm.set_slot(2, 16)
    if args.loops is not None:
        fpm.set_slot(4, args.loops)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fb.feast_he(A, emin, emax, args.m0, b=B, fpm=fpm)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    s = max(abs(emin), abs(emax))
    rep = {"info": int(r.info), "m": int(r.m), "m0_final": int(r.m0), "loop": int(r.loop), "seconds": dt,
           "it_per_s": (r.loop + 1) / dt, "factorizations": int(getattr(r, "factorizations", -1)),
           "max_res": float(np.max(r.res[:r.m])) if r.m else None, "epsout": float(r.epsout)}
    rep["history"] = [[float(v) for v in row] for row in getattr(r, "history", [])]
    rep["e_all"] = [float(v) for v in r.e[:r.m0]]
    rep["res_all"] = [float(v) for v in r.res[:r.m0]]
    if "inertia_count" in report:
        rep["count_inertia"] = report["inertia_count"]
    X = r.x[:, :r.m] if r.m else None
    if X is not None:
        Xd = torch.from_numpy(X).cuda()
        Bd = torch.complex(B.plane(0), B.plane(1))
        G = Xd.conj().T @ (Bd @ Xd)
        del Bd
        rep["b_orth_err"] = float((G - torch.eye(r.m, dtype=G.dtype, device=G.device)).abs().max())
        del Xd, G
    if ev is not None:
        inside = np.sort(ev[(ev >= emin) & (ev <= emax)])
        rep["count_independent"] = int(inside.size)
        if inside.size == r.m:
            rep["max_dl_over_s"] = float(np.abs(np.sort(r.e[:r.m]) - inside).max() / s)
    log(json.dumps(rep))
    report["feast"] = rep
    np.savez(os.path.join(OUT, f"c5_feast_n{args.n}.npz"), e=r.e, res=r.res,
             scal=np.array([r.m, r.loop, r.info, args.m0]))
    with open(os.path.join(OUT, f"c5_report_n{args.n}.json"), "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
