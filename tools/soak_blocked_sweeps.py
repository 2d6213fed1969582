"""Soak test of the blocked direct sweeps (trsm.cu: 256-row dataflow sweep + one TMA-fed ZGEMM
per outer block, n >= 6144): repeated solve passes must be bit-identical to the first one (a
stale tile in any launch would break that) and the first must satisfy (zB - A) x = y.
Usage: python tools/soak_blocked_sweeps.py [n] [count] [nrhs] [passes]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1203_4031_b200.dense import DeviceDenseOps  # noqa: E402
from paper_1203_4031_b200.device import get_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 6144
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 4
nrhs = int(sys.argv[3]) if len(sys.argv) > 3 else 256
passes = int(sys.argv[4]) if len(sys.argv) > 4 else 12
dev = get_device()
rng = np.random.default_rng(n)
a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
a = (a + a.conj().T) / 2
ops = DeviceDenseOps(dev, dev.upload(a, cplx=True), None, True)
zs = [complex(0.3 * k, 0.5 + 0.1 * k) for k in range(cnt)]
ops.prefactorize(zs)
y = rng.standard_normal((n, nrhs)) + 1j * rng.standard_normal((n, nrhs))
Y = dev.upload(y, cplx=True)
first, differ, worst = None, 0, 0.0
for p in range(passes):
    ops.solve_pass(Y, True)
    got = [np.stack([dev.download(ops.pass_result(z, adj)) for adj in (False, True)]) for z in zs]
    if first is None:
        first = got
        for z, x in zip(zs, got):
            s = z * np.eye(n) - a
            for adj, sm in ((0, s), (1, s.conj().T)):
                worst = max(worst, np.abs(sm @ x[adj] - y).max() / (np.abs(sm).max() * np.abs(x[adj]).max() * n))
    else:
        differ += sum(int(not np.array_equal(g, f)) for g, f in zip(got, first))
print(f"n={n} shifts={cnt} columns={nrhs}: first pass residual {worst:.2e}; "
      f"{passes - 1} repeat passes, {differ} results not bit-identical to the first")
print("OK" if worst < 1e-13 and differ == 0 else "BROKEN")
