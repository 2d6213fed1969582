"""One shifted LU + one solve of config 2 (N=4096), for ncu launch lists and
CUDA-event breakdowns.  Usage: python tools/prof_lu.py [n] [nrhs]"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1203_4031_b200.device import get_device

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 160
reps = int(os.environ.get("REPS", "3"))
dev = get_device()
P = ctypes.c_void_p
rng = np.random.default_rng(0)
a = rng.standard_normal((n, n)) / np.sqrt(n)
A = dev.upload(a, cplx=False)
lu = dev.empty(n, n, True)
piv = torch.empty(n, dtype=torch.int32, device=dev.tdev)
dinv = torch.empty(int(dev.lib.fb_zgetrf_dinv_doubles(n)), dtype=torch.float64, device=dev.tdev)
info = torch.empty(1, dtype=torch.int32, device=dev.tdev)
W = dev.upload(rng.standard_normal((n, nrhs)) + 0j, cplx=True)
for r in range(reps):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    e[0].record()
    dev.check(dev.lib.fb_dense_shift(dev.h, n, 0.01, 0.02, P(A.re), None, A.ld, None, None, 0,
                                     P(lu.re), P(lu.im), lu.ld), "shift")
    e[1].record()
    t0 = time.perf_counter()
    dev.check(dev.lib.fb_zgetrf(dev.h, n, P(lu.re), P(lu.im), lu.ld, P(piv.data_ptr()),
                                P(dinv.data_ptr()), P(info.data_ptr())), "zgetrf")
    t1 = time.perf_counter()
    e[2].record()
    dev.check(dev.lib.fb_zgetrs(dev.h, n, nrhs, P(lu.re), P(lu.im), lu.ld, P(piv.data_ptr()),
                                P(dinv.data_ptr()), 0, P(W.re), P(W.im), W.ld), "zgetrs")
    e[3].record()
    dev.check(dev.lib.fb_zgetrs(dev.h, n, nrhs, P(lu.re), P(lu.im), lu.ld, P(piv.data_ptr()),
                                P(dinv.data_ptr()), 1, P(W.re), P(W.im), W.ld), "zgetrs")
    e[4].record()
    torch.cuda.synchronize()
    lu_ms = e[1].elapsed_time(e[2])
    print(f"rep {r}: shift {e[0].elapsed_time(e[1]):.3f} ms, zgetrf {lu_ms:.3f} ms "
          f"({8 / 3 * n**3 / lu_ms / 1e9:.2f} TF, host issue {1e3 * (t1 - t0):.1f} ms), "
          f"zgetrs {e[2].elapsed_time(e[3]):.3f} ms ({8 * n * n * nrhs / e[2].elapsed_time(e[3]) / 1e9:.2f} TF), "
          f"adjoint {e[3].elapsed_time(e[4]):.3f} ms, launches {dev.launches()}", flush=True)
if os.environ.get("PANEL_PROF"):
    buf = (ctypes.c_ulonglong * 8)()
    dev.lib.fb_debug_panel_profile(buf)   # reset
    dev.check(dev.lib.fb_dense_shift(dev.h, n, 0.01, 0.02, P(A.re), None, A.ld, None, None, 0,
                                     P(lu.re), P(lu.im), lu.ld), "shift")
    dev.check(dev.lib.fb_zgetrf(dev.h, n, P(lu.re), P(lu.im), lu.ld, P(piv.data_ptr()),
                                P(dinv.data_ptr()), P(info.data_ptr())), "zgetrf")
    torch.cuda.synchronize()
    dev.lib.fb_debug_panel_profile(buf)
    names = ["argmax", "publish", "barrier", "winner", "swap+scale", "update"]
    cols = n
    print("panel phase cycles per column:", {k: round(buf[i] / cols) for i, k in enumerate(names)})
    npan = (n + 31) // 32
    print("panel prologue / epilogue cycles per panel:", round(buf[6] / npan), round(buf[7] / npan))
