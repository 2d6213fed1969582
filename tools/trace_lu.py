"""Timeline of one batched shifted LU (C2 size) under torch.profiler: kernel
totals per name, GPU busy time, and how much of the LU wall time only the
latency-bound panel work (panel/swap kernels) was running -- the part of the
critical path the trailing GEMMs do not hide.  Usage: trace_lu.py [n] [count]"""
import collections
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1203_4031_b200.device import get_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
count = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = get_device()
P = ctypes.c_void_p
rng = np.random.default_rng(0)
a = torch.from_numpy(rng.standard_normal((n, n)) / np.sqrt(n)).cuda()
zs = [complex(0.1 * np.cos(t), 0.05 * np.sin(t)) for t in np.linspace(0.2, 2.9, count)]
zr = (ctypes.c_double * count)(*[z.real for z in zs])
zi = (ctypes.c_double * count)(*[z.imag for z in zs])
lu = torch.empty((2, count, n, n), dtype=torch.float64, device="cuda")
piv = torch.empty((count, n), dtype=torch.int32, device="cuda")
dd = int(dev.lib.fb_zgetrf_dinv_doubles(n))
dinv = torch.empty((count, dd), dtype=torch.float64, device="cuda")
info = torch.empty(count, dtype=torch.int32, device="cuda")
lib, h = dev.lib, dev.h


def run():
    lib.fb_dense_shift_batched(h, count, n, zr, zi, P(a.data_ptr()), None, n, None, None, n,
                               P(lu[0].data_ptr()), P(lu[1].data_ptr()), n, n * n)
    lib.fb_zgetrf_batched(h, count, n, P(lu[0].data_ptr()), P(lu[1].data_ptr()), n, n * n,
                          P(piv.data_ptr()), n, P(dinv.data_ptr()), dd, P(info.data_ptr()))


for _ in range(2):
    run()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name.replace("(anonymous namespace)::", "")
             .replace("void ", "").split("(")[0][:50]) for e in evs)
t0, t1 = iv[0][0], max(e for _, e, _ in iv)
per = collections.defaultdict(lambda: [0, 0.0])
for s, e, nm in iv:
    per[nm][0] += 1
    per[nm][1] += e - s
# sweep: at each instant, which classes are active
pts = []
for s, e, nm in iv:
    cls = "gemm" if "gemm" in nm else "panel"
    pts.append((s, 1, cls))
    pts.append((e, -1, cls))
pts.sort()
act = {"gemm": 0, "panel": 0}
last = t0
only = collections.defaultdict(float)
for t, d, c in pts:
    dt = t - last
    key = ("gemm" if act["gemm"] else "") + ("+panel" if act["panel"] else "")
    only[key or "idle"] += dt
    act[c] += d
    last = t
print(f"n={n} count={count}: LU span {(t1 - t0) / 1e3:.2f} ms, {len(iv)} kernels")
for k, v in sorted(only.items(), key=lambda x: -x[1]):
    print(f"  {k:12s} {v / 1e3:8.2f} ms")
for k, (c, t) in sorted(per.items(), key=lambda x: -x[1][1])[:12]:
    print(f"  {t / 1e3:8.2f} ms {c:5d}  avg {t / c:8.1f} us  {k}")
