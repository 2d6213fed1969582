"""Batched shifted LU (fb_zgetrf_batched) of config-2 size: count shifts of an
N x N real matrix, timed with CUDA events.  Usage: prof_lub.py [n] [count] [reps]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1203_4031_b200.device import get_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
count = int(sys.argv[2]) if len(sys.argv) > 2 else 8
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
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
for r in range(reps):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    rc = lib.fb_dense_shift_batched(h, count, n, zr, zi, P(a.data_ptr()), None, n, None, None, n,
                                    P(lu[0].data_ptr()), P(lu[1].data_ptr()), n, n * n)
    assert rc == 0, rc
    e1.record()
    rc = lib.fb_zgetrf_batched(h, count, n, P(lu[0].data_ptr()), P(lu[1].data_ptr()), n, n * n,
                               P(piv.data_ptr()), n, P(dinv.data_ptr()), dd, P(info.data_ptr()))
    assert rc == 0, rc
    e2.record()
    torch.cuda.synchronize()
    ms = e1.elapsed_time(e2)
    print(f"n={n} count={count}: shift {e0.elapsed_time(e1):.2f} ms, zgetrf {ms:.2f} ms "
          f"({count * 8 / 3 * n ** 3 / ms / 1e9:.2f} TF/s)", flush=True)
