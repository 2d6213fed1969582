"""Time fb_chol_check / fb_reduced_eig at the BASELINE M0 sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1203_4031_b200.device import get_device

dev = get_device()
rng = np.random.default_rng(0)
for m, cplx in ((150, False), (160, False), (256, True), (512, True)):
    g = rng.standard_normal((m, m)) + (1j * rng.standard_normal((m, m)) if cplx else 0)
    a = (g + g.conj().T) / 2
    h = rng.standard_normal((m, m)) + (1j * rng.standard_normal((m, m)) if cplx else 0)
    b = h @ h.conj().T + m * np.eye(m)
    A, B = dev.upload(a, cplx=cplx), dev.upload(b, cplx=cplx)
    PHI = dev.empty(m, m, cplx)
    eps = torch.empty(m, dtype=torch.float64, device=dev.tdev)
    import ctypes
    buf = (ctypes.c_ulonglong * 8)()
    for rep in range(3):
        dev.lib.fb_debug_reduced_profile(buf)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        f = dev.chol_check(B, m)
        e[1].record()
        st = dev.reduced_eig(A, B, m, eps.data_ptr(), PHI)
        e[2].record()
        torch.cuda.synchronize()
    import scipy.linalg as sla
    ref = sla.eigh(a, b, eigvals_only=True)
    err = np.abs(eps.cpu().numpy() - ref).max()
    print(f"m={m} cplx={cplx}: chol {e[0].elapsed_time(e[1]):.3f} ms, eig {e[1].elapsed_time(e[2]):.3f} ms, "
          f"status={st} fail={f} max|d eps|={err:.2e}", flush=True)
    dev.lib.fb_debug_reduced_profile(buf)
    print("   cycles: " + ", ".join(f"{k} {v}" for k, v in zip(
        ("chol(2 launches)", "C", "householder", "fold|bisect", "QL|invit", "backsolve|backtransform", "-|backsolve"),
        buf[:7])))
