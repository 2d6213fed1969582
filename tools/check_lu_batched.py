"""Batched shifted LU + direct and adjoint solves against numpy: max residual |S x - y| / (|S| |x| n) per shift.
Usage: python tools/check_lu_batched.py [n] [count] [nrhs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1203_4031_b200.dense import DeviceDenseOps  # noqa: E402
from paper_1203_4031_b200.device import get_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 640
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 3
nrhs = int(sys.argv[3]) if len(sys.argv) > 3 else 24
dev = get_device()
rng = np.random.default_rng(n)
a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
a = (a + a.conj().T) / 2
ops = DeviceDenseOps(dev, dev.upload(a, cplx=True), None, True)
zs = [complex(0.3 * k, 0.5 + 0.1 * k) for k in range(cnt)]
ops.prefactorize(zs)
y = rng.standard_normal((n, nrhs)) + 1j * rng.standard_normal((n, nrhs))
worst = 0.0
for adj in (False, True):
    ops.solve_pass(dev.upload(y, cplx=True), adj)
    for z in zs:
        x = dev.download(ops.pass_result(z, adj))
        s = z * np.eye(n) - a
        if adj:
            s = s.conj().T
        r = np.abs(s @ x - y).max() / (np.abs(s).max() * np.abs(x).max() * n)
        worst = max(worst, r)
        print(f"n={n} z={z} adjoint={adj}: residual {r:.2e}")
print("OK" if worst < 1e-13 else "BROKEN")
