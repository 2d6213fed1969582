"""CSR backend timings on one GPU (feast_scsr, sparse.py:503-511).

Cases (seeded, synthetic):
  system  -- the reference's "system-shaped" generalized pencil stand-in
             (test_sparse.py:176-220: N=1671, NNZ=11435, kl=3, shared pattern)
  fem1d   -- 1-D FEM-like pentadiagonal pencil, N=1e6, nodes shuffled (the
             reorder must recover the band), B = mass matrix; ~64 eigenvalues
  strip2d -- 5-point Laplacian on a 16 x 60000 strip (N=960000), shuffled
Each line: wall time of one warm solve, loops, m, the reordered bandwidth and
backend, plus CUDA-event times of the CSR SpMM (multiply_a) and the row
gather at the solve width, with their algorithmic HBM bytes.
"""

import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")


def _sym_coo(n, offs, rng, diag):
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [diag]
    for d, s in offs:
        r = np.arange(n - d)
        v = s * (1 + 0.2 * rng.standard_normal(n - d))
        rows += [r + d, r]
        cols += [r, r + d]
        vals += [v, v]
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def case(name, rng, shuffle=True):
    from paper_1203_4031_b200.sparse import CsrMatrix
    if name == "fem1d":
        n = 1_000_000
        r, c, v = _sym_coo(n, [(1, -0.7), (2, 0.2)], rng, 2.0 * (1 + 0.2 * rng.standard_normal(n)))
        br, bc, bv = _sym_coo(n, [(1, 1 / 6)], np.random.default_rng(0), np.full(n, 4 / 6))
        bv[bv != 4 / 6] = 1 / 6
    elif name == "strip2d":
        gx, gy = 16, 60000
        n = gx * gy
        idx = np.arange(n).reshape(gy, gx)
        pairs = [(idx[:, :-1].ravel(), idx[:, 1:].ravel()), (idx[:-1, :].ravel(), idx[1:, :].ravel())]
        r = np.concatenate([np.arange(n)] + [p[0] for p in pairs] + [p[1] for p in pairs])
        c = np.concatenate([np.arange(n)] + [p[1] for p in pairs] + [p[0] for p in pairs])
        v = np.concatenate([4.0 + 0.3 * rng.random(n)] + [-np.ones(p[0].size) for p in pairs] * 2)
        br = bc = bv = None
    else:
        raise ValueError(name)
    p = rng.permutation(n)
    if not shuffle:
        p = np.arange(n)
    ip = np.empty_like(p)
    ip[p] = np.arange(n)
    a = CsrMatrix.from_coo(n, ip[r] + 1, ip[c] + 1, v)
    b = None if br is None else CsrMatrix.from_coo(n, ip[br] + 1, ip[bc] + 1, bv)
    return a, b


def interval(name):
    # 64 eigenvalues each, by Sylvester inertia counts (band LDL^T) of the
    # unshuffled pencils in the build container
    return {"fem1d": (0.5, 0.5004219), "strip2d": (0.5, 0.5007823)}[name]


def main():
    import torch
    import paper_1203_4031_b200 as fb
    from paper_1203_4031_b200.sparse import DeviceCsrOps
    rng = np.random.default_rng(7)
    names = sys.argv[1:] or ["fem1d", "strip2d"]
    for name in names:
        a, b = case(name, rng)
        emin, emax = interval(name)
        m0 = 96
        fb.feast_scsr(a, emin, emax, m0, b=b)                 # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fb.feast_scsr(a, emin, emax, m0, b=b)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        from paper_1203_4031_b200.device import get_device
        dev = get_device(None)
        af = a.expand_full()
        t1 = time.perf_counter()
        ops = DeviceCsrOps(dev, af, None if b is None else b.expand_full(), False)
        torch.cuda.synchronize()
        setup = time.perf_counter() - t1
        X = dev.empty(a.n, m0, False)
        X.t.normal_()
        Y = dev.empty(a.n, m0, False)
        W = dev.empty(a.n, m0, True, ld=m0)
        W.t.normal_()
        T = dev.empty(a.n, m0, True, ld=m0)
        st = torch.cuda.current_stream()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        for _ in range(3):
            ops.multiply_a(X, Y)
        e[0].record(st)
        for _ in range(20):
            ops.multiply_a(X, Y)
        e[1].record(st)
        for _ in range(20):
            ops._permute(ops.perm, W, T) if ops.mode == "band" else None
        e[2].record(st)
        torch.cuda.synchronize()
        spmm_ms = e[0].elapsed_time(e[1]) / 20
        gather_ms = e[1].elapsed_time(e[2]) / 20
        nnz = af.nnz
        spmm_bytes = nnz * 16 + (a.n + 1) * 8 + 2 * a.n * m0 * 8     # index+value stream, X once, Y once
        gather_bytes = 2 * a.n * m0 * 16 + a.n * 8
        print(json.dumps({
            "case": name, "n": a.n, "nnz": nnz, "mode": ops.mode, "kl": getattr(ops, "kl", None),
            "m0": m0, "info": r.info, "m": r.m, "loop": r.loop, "wall_s": round(wall, 4), "host_setup_s": round(setup, 3), "inertia_count": 64,
            "iterations_per_s": round((r.loop + 1) / wall, 3),
            "max_res": float(np.max(r.res[:r.m])) if r.m else None,
            "spmm_ms": round(spmm_ms, 4), "spmm_GBps": round(spmm_bytes / spmm_ms / 1e6, 1),
            "gather_ms": round(gather_ms, 4), "gather_GBps": round(gather_bytes / gather_ms / 1e6, 1)
            if gather_ms > 0 else None}), flush=True)


if __name__ == "__main__":
    main()
