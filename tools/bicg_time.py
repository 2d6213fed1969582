"""Wall time of the GPU BiCGStab inner solver (feast_scsr solver='iterative')
on the golden CSR pencils (tests/golden/sparse.npz, lowest 8 eigenvalues,
iter_tol 1e-10).  Run twice, with FB_BICG_GRAPH=0 and unset, to compare
eager launches with the CUDA-graph replay of the iteration chunks."""

import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")


def main():
    import torch
    import paper_1203_4031_b200 as fb
    from test_sparse_cpu import _case
    g = np.load("tests/golden/sparse.npz")
    for name in ("lap2d", "fem1d_gv"):
        a, b, meta, herm = _case(g, name)
        opts = fb.SolverOptions(solver="iterative", iter_tol=1e-10)
        fb.feast_scsr(a, meta[6], meta[7], 16, b=b, options=opts)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fb.feast_scsr(a, meta[6], meta[7], 16, b=b, options=opts)
        torch.cuda.synchronize()
        print(f"{name} graph={os.environ.get('FB_BICG_GRAPH', '1')} info={r.info} m={r.m} loop={r.loop} "
              f"wall={time.perf_counter() - t0:.3f}s")


if __name__ == "__main__":
    main()
