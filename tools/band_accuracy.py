"""Backward error of the partitioned (SPIKE) band solve against LAPACK's
whole-band zgbsv on config-4's construction (N = 200000, kd = 16, shift 0 and
the shift nearest the real axis): ||S x - y||_inf / (||S||_inf ||x||_inf), for
P = 1 (one partition: the reference's whole-band LU on the GPU) and the
default partition size.  Usage: python tools/band_accuracy.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.linalg as sla  # noqa: E402
import torch  # noqa: E402

from paper_1203_4031_b200 import workloads as W  # noqa: E402
from paper_1203_4031_b200.banded import DeviceBandOps, expand_band, pad_band  # noqa: E402
from paper_1203_4031_b200.device import get_device  # noqa: E402
from paper_1203_4031_b200.quadrature import build_contour, gauss_legendre  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
dev = get_device()
w = W.c4_sbgv(n=n, interval=(-0.0008386 * 1e6 / n, 0.00089835 * 1e6 / n))
kl, m0 = w.kla, 24
fa = expand_band(w.a, w.kla, w.uplo, False)
fbm = pad_band(expand_band(w.b, w.klb, w.uplo, False), w.klb, kl)
ct = build_contour(gauss_legendre(8), w.emin, w.emax)
zs = [complex(ct.z[0]), complex(ct.z[3])]
rng = np.random.default_rng(1)
y = rng.standard_normal((n, m0))


def berr(z, x):
    s = z * fbm - fa                      # (2kl+1, n), row kl+d = d-th subdiagonal
    r = -y.astype(complex)
    for d in range(-kl, kl + 1):
        j0, j1 = max(0, -d), min(n, n - d)
        r[j0 + d:j1 + d] += s[kl + d, j0:j1, None] * x[j0:j1]
    snorm = np.abs(s).sum(0).max()
    return np.abs(r).max() / (snorm * np.abs(x).max()), np.abs(r).max() / np.abs(y).max()


for part in (10 ** 9, 4096, 1024):
    P = dev.lib.fb_debug_band_part_target(part, n, kl)
    ops = DeviceBandOps(dev, dev.upload(fa, cplx=False), dev.upload(fbm, cplx=False), kl, False)
    ops.prefactorize(zs)
    Y = dev.upload(y, cplx=False)
    ops.solve_pass(Y, False)
    for z in zs:
        x = dev.download(ops.pass_result(z, False))
        print(f"GPU P={P:4d} z={z:.3e}: backward error {berr(z, x)[0]:.2e}  |Sx-y|/|y| {berr(z, x)[1]:.2e}", flush=True)
dev.lib.fb_debug_band_part_target(0, n, kl)
for z in zs:
    s = z * fbm - fa
    ab = np.zeros((2 * kl + 1, n), dtype=complex)   # LAPACK band: ab[ku + i - j, j] = S(i, j); ours: s[kl + (i-j), j]
    ab[:] = s
    x = sla.solve_banded((kl, kl), ab, y.astype(complex))
    print(f"LAPACK zgbsv z={z:.3e}: backward error {berr(z, x)[0]:.2e}  |Sx-y|/|y| {berr(z, x)[1]:.2e}", flush=True)
