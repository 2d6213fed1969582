"""C4 band kernels in isolation: factor the Ne = 8 shifts of config 4
(N = 1e6, kd = 16) in one batched call, then time the batched solve of one
contour pass (M0 = 96 right-hand sides) and the band multiply with CUDA
events; print algorithmic GB/s and FP64 TFLOP/s against the roofline
counts of DESIGN.md.  Also a per-shift solve residual check.

Usage: python tools/prof_band.py [reps] [n] [partition rows]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1203_4031_b200 import workloads as W  # noqa: E402
from paper_1203_4031_b200.banded import DeviceBandOps, expand_band, pad_band  # noqa: E402
from paper_1203_4031_b200.device import get_device  # noqa: E402
from paper_1203_4031_b200.quadrature import build_contour, gauss_legendre  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
torch.cuda.set_device(0)
dev = get_device()
if len(sys.argv) > 3:   # partition-size target (rows), default 4096
    print("partitions:", dev.lib.fb_debug_band_part_target(int(sys.argv[3]), n, 16))
w = W.c4_sbgv() if n == 1_000_000 else W.c4_sbgv(n=n, interval=(-0.01, 0.01))
kl, m0 = w.kla, w.m0
fa = expand_band(w.a, w.kla, w.uplo, False)
fbm = pad_band(expand_band(w.b, w.klb, w.uplo, False), w.klb, kl)
FA, FB = dev.upload(fa, cplx=False), dev.upload(fbm, cplx=False)
ops = DeviceBandOps(dev, FA, FB, kl, False)
zs = list(build_contour(gauss_legendre(8), w.emin, w.emax).z)


def timed(fn, k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


fac = {}
t_f = timed(lambda: fac.update(DeviceBandOps(dev, FA, FB, kl, False).prefactorize(zs)), 1)
fac = ops.prefactorize(zs)
Y = dev.empty(n, m0, False)
Y.plane(0).copy_(torch.rand(n, m0, dtype=torch.float64, device=dev.tdev) - 0.5)
ops.solve_pass(Y, False)
t_s = timed(lambda: ops.solve_pass(Y, False), reps)
Xs0 = ops._pass[(id(ops._batches[0]), 0)][0][:, 0].clone()
X = dev.empty(n, m0, False)
t_m = timed(lambda: ops.multiply_a(Y, X), reps)
ct = build_contour(gauss_legendre(8), w.emin, w.emax)
Q = dev.zeros(n, m0, False)


def pass_acc():
    ops.solve_pass(Y, False)
    dev.accumulate_terms([(0, ct.weights[k], ct.theta[k], ops.pass_result(complex(ct.z[k]), False))
                          for k in range(len(zs))], ct.radius, Q)


t_sa = timed(pass_acc, reps)
Q_ref = dev.zeros(n, m0, False)
Q, Q_keep = Q_ref, Q
pass_acc()
Q = Q_keep
spec = [(complex(ct.z[k]), False, 0, ct.weights[k], ct.theta[k]) for k in range(len(zs))]
Q.zero_()
assert ops.solve_pass_accumulate(Y, spec, ct.radius, Q)
qd = float((Q.plane(0) - Q_ref.plane(0)).abs().max() / Q_ref.plane(0).abs().max())
t_fa = timed(lambda: ops.solve_pass_accumulate(Y, spec, ct.radius, Q), reps)

ne = len(zs)
solve_bytes = ne * ((3 * kl + 1) * n * 16 + 2 * n * m0 * 16)
solve_flops = ne * 8 * 3 * kl * n * m0
mv_bytes = (2 * kl + 1) * n * 8 + 2 * n * m0 * 8
print(f"n={n} kl={kl} m0={m0} Ne={ne}")
print(f"factor (8 shifts, incl. alloc): {t_f:.2f} ms")
print(f"solve pass (8 shifts): {t_s:.2f} ms  -> {solve_bytes / t_s / 1e6:.0f} GB/s algorithmic, "
      f"{solve_flops / t_s / 1e9:.2f} TFLOP/s")
print(f"solve pass + quadrature sum (accumulate_terms): {t_sa:.2f} ms")
print(f"fused pass (sweeps + interface + correction/accumulation kernel): {t_fa:.2f} ms -> "
      f"{solve_bytes / t_fa / 1e6:.0f} GB/s algorithmic, {solve_flops / t_fa / 1e9:.2f} TFLOP/s; "
      f"max |Q_fused - Q_unfused| / max|Q| = {qd:.2e}")
print(f"band matvec A*Y: {t_m:.3f} ms -> {mv_bytes / t_m / 1e6:.0f} GB/s")
if w.klb < kl:
    FBc = dev.upload(expand_band(w.b, w.klb, w.uplo, False), cplx=False)
    ops_c = DeviceBandOps(dev, FA, FB, kl, False, mv_b=(FBc, w.klb))
    t_mb = timed(lambda: ops_c.multiply_b(Y, X), reps)
    t_mb0 = timed(lambda: ops.multiply_b(Y, X), reps)
    bb = (2 * w.klb + 1) * n * 8 + 2 * n * m0 * 8
    print(f"band matvec B*Y: padded kl={kl} {t_mb0:.3f} ms; own klb={w.klb} {t_mb:.3f} ms -> {bb / t_mb / 1e6:.0f} GB/s")

# residual check of shift 0's solve: || S x - y || / ||y|| through a band multiply
x0 = torch.complex(Xs0[0], Xs0[1])
z = complex(zs[0])
fa_t = torch.from_numpy(fa).to(dev.tdev)
fb_t = torch.from_numpy(fbm).to(dev.tdev)
y0 = Y.plane(0)
r = torch.zeros_like(x0)
for s in range(-kl, kl + 1):
    j0, j1 = max(0, -s), min(n, n - s)
    d = z * fb_t[kl + s, j0:j1] - fa_t[kl + s, j0:j1]
    r[j0 + s:j1 + s] += d[:, None] * x0[j0:j1]
rel = float((r - y0).abs().max() / y0.abs().max())
print(f"shift 0 solve residual max|Sx - y| / max|y| = {rel:.2e}")
