"""cuBLAS (torch) complex/real FP64 GEMM throughput on the LU / projection
shapes, as a calibration point for fb_gemm (library code, measurement only)."""
import torch


def t(fn, reps=10):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dev = "cuda"
for (b, m, n, k) in [(8, 3968, 3968, 128), (1, 4096, 4096, 128), (1, 8192, 8192, 128), (1, 4096, 4096, 1024),
                     (1, 8192, 8192, 256), (8, 3968, 3968, 256)]:
    for dt, fl in ((torch.complex128, 8), (torch.float64, 2)):
        A = torch.randn(b, m, k, dtype=dt, device=dev)
        B = torch.randn(b, k, n, dtype=dt, device=dev)
        C = torch.randn(b, m, n, dtype=dt, device=dev)
        ms = t(lambda: C.baddbmm_(A, B, alpha=-1))
        print(f"cuBLAS {'Z' if dt.is_complex else 'D'}GEMM batch={b} {m}x{n}x{k}: {ms:.3f} ms "
              f"{b * fl * m * n * k / ms / 1e9:.2f} TF/s", flush=True)
        del A, B, C
