"""Rounding behaviour of the FP64 tensor-core GEMM (DMMA) against numpy/OpenBLAS.

C = A @ B with random A (m x k), B (k x n); the exact product is taken in
extended precision (np.longdouble).  Reports the RMS and the mean SIGNED error
(in units of |A||B| eps) for the GPU and for numpy at growing k: unbiased
round-to-nearest accumulation grows like sqrt(k) with mean ~0, a truncating
accumulator grows like k with a nonzero mean.
Usage: python tools/dmma_rounding.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1203_4031_b200.device import get_device  # noqa: E402

dev = get_device()
rng = np.random.default_rng(7)
m, n = 128, 64
eps = np.finfo(np.float64).eps
for k in (32, 256, 2048, 8192):
    a = rng.standard_normal((m, k))
    b = rng.standard_normal((k, n))
    ex = a.astype(np.longdouble) @ b.astype(np.longdouble)
    scale = (np.abs(a).astype(np.longdouble) @ np.abs(b).astype(np.longdouble)) * eps
    A = dev.upload(a, cplx=False)
    B = dev.upload(b, cplx=False)
    C = dev.empty(m, n, False)
    dev.gemm("N", "N", m, n, k, 1.0, A, B, 0.0, C)
    cg = dev.download(C)
    cn = a @ b
    for name, c in (("gpu", cg), ("numpy", cn)):
        e = ((c.astype(np.longdouble) - ex) / scale).astype(np.float64)
        print(f"k={k:5d} {name:6s} rms {np.sqrt(np.mean(e ** 2)):.3e}  mean {np.mean(e):+.3e}  "
              f"max {np.abs(e).max():.3e}", flush=True)
    # accumulate into C (beta = 1): the sweeps' X -= M X pattern, 64 rank-32 steps
    c0 = rng.standard_normal((m, n))
    C = dev.upload(c0, cplx=False)
    exs = c0.astype(np.longdouble)
    cn = c0.copy()
    for s in range(0, k, 32):
        As = dev.upload(np.ascontiguousarray(a[:, s:s + 32]), cplx=False)
        Bs = dev.upload(np.ascontiguousarray(b[s:s + 32]), cplx=False)
        dev.gemm("N", "N", m, n, 32, -1.0, As, Bs, 1.0, C)
        exs -= a[:, s:s + 32].astype(np.longdouble) @ b[s:s + 32].astype(np.longdouble)
        cn -= a[:, s:s + 32] @ b[s:s + 32]
    cg = dev.download(C)
    sc = scale + np.abs(c0) * eps
    for name, c in (("gpu-acc", cg), ("np-acc", cn)):
        e = ((c.astype(np.longdouble) - exs) / sc).astype(np.float64)
        print(f"k={k:5d} {name:7s} rms {np.sqrt(np.mean(e ** 2)):.3e}  mean {np.mean(e):+.3e}  "
              f"max {np.abs(e).max():.3e}", flush=True)
