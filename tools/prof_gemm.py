"""ZGEMM / DGEMM throughput of fb_gemm for the shapes the FEAST path issues."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1203_4031_b200.device import get_device

dev = get_device()
rng = np.random.default_rng(0)


def bench(cplx, opa, opb, m, n, k, reps=10):
    ar = (m, k) if opa == "N" else (k, m)
    br = (k, n) if opb == "N" else (n, k)
    A = dev.empty(*ar, cplx)
    B = dev.empty(*br, cplx)
    C = dev.empty(m, n, cplx)
    for t in (A, B, C):
        t.t.normal_()
    for _ in range(2):
        dev.gemm(opa, opb, m, n, k, -1.0, A, B, 1.0, C, cplx=cplx)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dev.gemm(opa, opb, m, n, k, -1.0, A, B, 1.0, C, cplx=cplx)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = (8 if cplx else 2) * m * n * k
    print(f"{'Z' if cplx else 'D'}GEMM {opa}{opb} m={m} n={n} k={k}: {ms:.3f} ms  {flops / ms / 1e9:.2f} TF/s")


for args in [(True, "N", "N", 4096, 4096, 128), (True, "N", "N", 8192, 8192, 128), (True, "N", "N", 4096, 4096, 1024),
             (True, "N", "N", 4096, 128, 32), (True, "N", "N", 4096, 3968, 32),
             (False, "N", "N", 4096, 160, 4096), (True, "N", "N", 8192, 256, 8192),
             (False, "C", "N", 160, 160, 4096), (True, "C", "N", 256, 256, 8192),
             (False, "N", "N", 4096, 160, 160)]:
    bench(*args)
