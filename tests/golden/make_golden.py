"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
(`feastlib` 0.1.0, /root/reference/pkg/src) in the build container.

The reference cannot travel to the GPU box, so its outputs are frozen here as
small .npz files.  Re-run with:

    python tests/golden/make_golden.py unit small          # seconds
    python tests/golden/make_golden.py scaled              # ~1 min
    python tests/golden/make_golden.py c1 c2 c3            # minutes (LAPACK caller)

`unit`/`small` call the reference's own functions and drivers unmodified.
`scaled`/`cN` drive the reference's own SymmetricRci/HermitianRci kernel with
a LAPACK-backed caller (zgetrf/zgetrs, zgbtrf/zgbtrs), the oracle SURVEY.md
§8(c) specifies for sizes where the pure-Python LU is infeasible.
"""

from __future__ import annotations

import os
import sys
import time

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
import scipy.linalg as sla  # noqa: E402
from scipy.linalg import lapack  # noqa: E402

import feastlib as fl  # noqa: E402
from feastlib import banded as fband  # noqa: E402
from feastlib import dense as fdense  # noqa: E402
from feastlib import kernel as fkernel  # noqa: E402
from feastlib import reduced as freduced  # noqa: E402


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, os.path.getsize(path), "bytes")


def _band_F(a, kl):
    n = a.shape[0]
    ab = np.zeros((2 * kl + 1, n), dtype=a.dtype)
    for s in range(-kl, kl + 1):
        for j in range(max(0, -s), min(n, n - s)):
            ab[kl + s, j] = a[j + s, j]
    return ab


def _rand_band(n, kl, rng, cplx=False):
    a = rng.normal(size=(n, n))
    if cplx:
        a = a + 1j * rng.normal(size=(n, n))
    a = (a + a.conj().T) / 2
    mask = np.abs(np.subtract.outer(np.arange(n), np.arange(n))) <= kl
    return np.where(mask, a, 0)


def make_unit():
    out = {}
    for seed, off, cnt in ((42, 0, 64), (7, 4, 6), (11, 0, 4), (2**63 + 5, 100, 33)):
        out[f"rng_{seed}_{off}_{cnt}"] = fkernel.random_uniform(seed, off, cnt)
    for ne in fl.params.ALLOWED_CONTOUR_POINTS:
        r = fl.gauss_legendre(ne)
        out[f"gl_nodes_{ne}"] = r.nodes
        out[f"gl_weights_{ne}"] = r.weights
        c = fl.build_contour(r, -0.7, 1.3)
        out[f"contour_z_{ne}"] = c.z
        out[f"contour_theta_{ne}"] = c.theta
    rng = np.random.default_rng(20261020)
    # accumulation (kernel.py:108-124)
    q0 = rng.normal(size=(9, 4))
    w2 = rng.normal(size=(9, 4)) + 1j * rng.normal(size=(9, 4))
    q = q0.copy()
    fkernel.accumulate_subspace(q, w2, 0.3, 1.7, 0.9, "symmetric")
    out.update(acc_q0=q0, acc_w2=w2, acc_sym=q)
    qc0 = q0 + 1j * rng.normal(size=(9, 4))
    qd = qc0.copy()
    fkernel.accumulate_subspace(qd, w2, 0.3, 1.7, 0.9, "hermitian-direct")
    qa = qc0.copy()
    fkernel.accumulate_subspace(qa, w2, 0.3, 1.7, 0.9, "hermitian-adjoint")
    out.update(acc_qc0=qc0, acc_hd=qd, acc_ha=qa)
    # dense LU (dense.py:30-88)
    for n in (1, 2, 5, 20, 64, 97):
        a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
        bm = rng.normal(size=(n, 3)) + 1j * rng.normal(size=(n, 3))
        lu, piv = fdense.lu_factor(a)
        out[f"lu_a_{n}"] = a
        out[f"lu_b_{n}"] = bm
        out[f"lu_lu_{n}"] = lu
        out[f"lu_piv_{n}"] = piv
        out[f"lu_x_{n}"] = fdense.lu_solve((lu, piv), bm)
        out[f"lu_xa_{n}"] = fdense.lu_solve((lu, piv), bm, adjoint=True)
    # band LU (banded.py:68-146), matvec (50-65), expand (21-47)
    for n, kl in ((6, 1), (12, 3), (9, 0), (40, 4), (130, 16)):
        a = _rand_band(n, kl, rng, cplx=True) + 3j * np.eye(n)
        fb = fband.expand_band(_band_F(a, kl), kl, "F", True)
        ab, ipiv, _ = fband.band_lu_factor(fb, kl)
        bm = rng.normal(size=(n, 3)) + 1j * rng.normal(size=(n, 3))
        out[f"blu_a_{n}_{kl}"] = a
        out[f"blu_fb_{n}_{kl}"] = fb
        out[f"blu_ab_{n}_{kl}"] = ab
        out[f"blu_ipiv_{n}_{kl}"] = ipiv
        out[f"blu_b_{n}_{kl}"] = bm
        out[f"blu_x_{n}_{kl}"] = fband.band_lu_solve((ab, ipiv, kl), bm)
        out[f"blu_xa_{n}_{kl}"] = fband.band_lu_solve((ab, ipiv, kl), bm, adjoint=True)
        x = rng.normal(size=(n, 4))
        out[f"bmv_x_{n}_{kl}"] = x
        out[f"bmv_y_{n}_{kl}"] = fband.band_matvec(fb, x)
        for uplo in ("F", "L", "U"):
            ar = _rand_band(n, kl, rng, cplx=True)
            if uplo == "F":
                st = _band_F(ar, kl)
            elif uplo == "L":
                st = np.zeros((kl + 1, n), dtype=complex)
                for d in range(kl + 1):
                    st[d, : n - d] = np.diagonal(ar, -d)
            else:
                st = np.zeros((kl + 1, n), dtype=complex)
                for d in range(kl + 1):
                    st[kl - d, d:] = np.diagonal(ar, d)
            out[f"xb_in_{uplo}_{n}_{kl}"] = st
            out[f"xb_out_{uplo}_{n}_{kl}"] = fband.expand_band(st, kl, uplo, True)
    # reduced eigensolver (reduced.py)
    for n, cplx in ((2, False), (8, False), (7, True), (40, False), (33, True)):
        if cplx:
            g = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
            h = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
        else:
            g = rng.normal(size=(n, n))
            h = rng.normal(size=(n, n))
        aq = (g + g.conj().T) / 2
        bq = h @ h.conj().T + n * np.eye(n)
        eps, phi = freduced.generalized_eig(aq, bq)
        out[f"red_aq_{n}"] = aq
        out[f"red_bq_{n}"] = bq
        out[f"red_eps_{n}"] = eps
        out[f"red_phi_{n}"] = phi
    for name, mat in (("neg2", np.diag([1.0, -1.0])), ("neg1", np.diag([-1.0, 2.0])),
                      ("sing", np.array([[1.0, 1.0, 0], [1.0, 1.0, 0], [0, 0, 1.0]]))):
        _, fail = freduced.spd_factor(mat)
        out[f"spd_{name}_in"] = mat
        out[f"spd_{name}_fail"] = np.array(fail)
    _save("unit.npz", **out)


def _pack(prefix, r, out):
    out[prefix + "e"] = r.e
    out[prefix + "x"] = r.x
    out[prefix + "res"] = r.res
    out[prefix + "scal"] = np.array([r.m, r.loop, r.info, r.m0], dtype=np.int64)
    out[prefix + "epsout"] = np.array(r.epsout)


def make_small():
    """Driver runs (pure reference path) on small pencils incl. edge cases."""
    out = {}
    rng = np.random.default_rng(777)
    cases = []
    hello = np.array([[2.0, -1.0], [-1.0, 2.0]])
    cases.append(("hello", "sy", dict(a=hello, emin=-5.0, emax=5.0, m0=2)))
    f = fl.feastinit(); f.set_slot(14, 1)
    cases.append(("hello_fpm14", "sy", dict(a=hello, emin=-5.0, emax=5.0, m0=2, fpm=f)))
    f = fl.feastinit(); f.set_slot(6, 1)
    cases.append(("hello_res", "sy", dict(a=hello, emin=-5.0, emax=5.0, m0=2, fpm=f)))
    cases.append(("hello_none", "sy", dict(a=hello, emin=10.0, emax=20.0, m0=2)))
    f = fl.feastinit(); f.set_slot(4, 0)
    cases.append(("hello_budget", "sy", dict(a=hello, emin=-5.0, emax=5.0, m0=2, fpm=f)))
    cases.append(("diag_m0small", "sy", dict(a=np.diag([1.0, 2.0, 3.0, 4.0]), emin=0.5, emax=3.5, m0=2)))
    cases.append(("eye4", "sy", dict(a=np.eye(4), emin=0.0, emax=2.0, m0=4)))
    a = np.diag([1.0, 2.0, 3.0, -0.05, -0.1, 4.05, 4.1, 4.15])
    f = fl.feastinit(); f.set_slot(2, 3); f.set_slot(3, 6); f.set_slot(4, 30)
    cases.append(("leaked_spurious", "sy", dict(a=a, emin=0.0, emax=4.0, m0=6, fpm=f)))
    for tag, n, m_lo, m_hi, m0, gen in (("sy60", 60, 20, 31, 18, False), ("sy97", 97, 40, 52, 20, False)):
        a = rng.normal(size=(n, n)); a = (a + a.T) / 2
        ev = np.linalg.eigvalsh(a)
        emin, emax = 0.5 * (ev[m_lo - 1] + ev[m_lo]), 0.5 * (ev[m_hi] + ev[m_hi + 1])
        cases.append((tag, "sy", dict(a=a, emin=emin, emax=emax, m0=m0)))
    n = 50
    a = rng.normal(size=(n, n)); a = (a + a.T) / 2
    g = rng.normal(size=(n, n)); b = g @ g.T + n * np.eye(n)
    ev = sla.eigh(a, b, eigvals_only=True)
    cases.append(("sygv50", "sy", dict(a=a, b=b, emin=0.5 * (ev[14] + ev[15]),
                                        emax=0.5 * (ev[25] + ev[26]), m0=16)))
    f = fl.feastinit(); f.set_slot(2, 16); f.set_slot(6, 1); f.set_slot(3, 10)
    cases.append(("sygv50_ne16_res", "sy", dict(a=a, b=b, emin=0.5 * (ev[14] + ev[15]),
                                                 emax=0.5 * (ev[25] + ev[26]), m0=16, fpm=f)))
    for uplo in ("L", "U"):
        cases.append((f"sygv50_{uplo}", "sy", dict(a=a, b=b, uplo=uplo, emin=0.5 * (ev[14] + ev[15]),
                                                     emax=0.5 * (ev[25] + ev[26]), m0=16)))
    n = 40
    a = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)); a = (a + a.conj().T) / 2
    ev = np.linalg.eigvalsh(a)
    cases.append(("heev40", "he", dict(a=a, emin=0.5 * (ev[9] + ev[10]), emax=0.5 * (ev[19] + ev[20]), m0=15)))
    g = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)); b = g @ g.conj().T + n * np.eye(n)
    ev = sla.eigh(a, b, eigvals_only=True)
    cases.append(("hegv40", "he", dict(a=a, b=b, emin=0.5 * (ev[4] + ev[5]), emax=0.5 * (ev[14] + ev[15]), m0=15)))
    cases.append(("hegv40_L", "he", dict(a=a, b=b, uplo="L", emin=0.5 * (ev[4] + ev[5]),
                                         emax=0.5 * (ev[14] + ev[15]), m0=15)))
    # banded
    n, kl = 200, 3
    a = _rand_band(n, kl, rng)
    bmat = (4 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)) / 6
    ev = sla.eigh(a, bmat, eigvals_only=True)
    sbcase = dict(ab=_band_F(a, kl), kla=kl, b=_band_F(bmat, 1), klb=1,
                  emin=0.5 * (ev[89] + ev[90]), emax=0.5 * (ev[104] + ev[105]), m0=24)
    cases.append(("sbgv200", "sb", sbcase))
    ab_l = np.zeros((kl + 1, n))
    for d in range(kl + 1):
        ab_l[d, : n - d] = np.diagonal(a, -d)
    cases.append(("sbev200_L", "sb", dict(ab=ab_l, kla=kl, uplo="L", emin=-0.5, emax=0.5, m0=40)))
    n, kl = 60, 2
    a = _rand_band(n, kl, rng, cplx=True)
    ev = np.linalg.eigvalsh(a)
    cases.append(("hbev60", "hb", dict(ab=_band_F(a, kl), kla=kl, emin=0.5 * (ev[19] + ev[20]),
                                        emax=0.5 * (ev[29] + ev[30]), m0=16)))
    lap = 2000
    ab3 = np.zeros((3, lap)); ab3[0, 1:] = -1.0; ab3[1] = 2.0; ab3[2, :-1] = -1.0
    lam = 2.0 - 2.0 * np.cos(np.arange(1, lap + 1) * np.pi / (lap + 1))
    for ne in (4, 8, 16):
        f = fl.feastinit(); f.set_slot(2, ne); f.set_slot(6, 1); f.set_slot(3, 10)
        cases.append((f"lap2000_ne{ne}", "sb", dict(ab=ab3, kla=1, emin=0.0,
                                                     emax=0.5 * (lam[49] + lam[50]), m0=75, fpm=f)))
    names = []
    for name, kind, kw in cases:
        t0 = time.time()
        kw = dict(kw)
        fpm = kw.pop("fpm", None)
        if kind in ("sy", "he"):
            fn = fl.feast_sy if kind == "sy" else fl.feast_he
            r = fn(kw["a"], kw["emin"], kw["emax"], kw["m0"], b=kw.get("b"), uplo=kw.get("uplo", "F"), fpm=fpm)
            out[f"{name}__a"] = kw["a"]
            if kw.get("b") is not None:
                out[f"{name}__b"] = kw["b"]
        else:
            fn = fl.feast_sb if kind == "sb" else fl.feast_hb
            r = fn(kw["ab"], kw["kla"], kw["emin"], kw["emax"], kw["m0"], b=kw.get("b"),
                   klb=kw.get("klb"), uplo=kw.get("uplo", "F"), fpm=fpm)
            out[f"{name}__a"] = kw["ab"]
            if kw.get("b") is not None:
                out[f"{name}__b"] = kw["b"]
        fp = np.array([(fpm or fl.feastinit()).slot(i) for i in range(1, 65)])
        out[f"{name}__cfg"] = np.array([kw["emin"], kw["emax"], kw["m0"], kw.get("kla", 0),
                                        kw.get("klb", 0)], dtype=np.float64)
        out[f"{name}__uplo"] = np.array(kw.get("uplo", "F"))
        out[f"{name}__kind"] = np.array(kind)
        out[f"{name}__fpm"] = fp
        _pack(f"{name}__", r, out)
        names.append(name)
        print(f"{name:18s} info={r.info} m={r.m} loop={r.loop} {time.time() - t0:.1f}s")
    out["names"] = np.array(names)
    _save("small.npz", **out)


class LapackCaller:
    """Answers the reference kernel's tasks with LAPACK."""

    def __init__(self, kernel, a=None, b=None, band=None):
        self.k, self.a, self.b, self.band = kernel, a, b, band
        self.factors = {}
        self.t = dict(factor=0.0, solve=0.0, mult=0.0)

    def _factor(self, z):
        if self.band is None:
            s = -self.a.astype(np.complex128)
            if self.b is None:
                s[np.diag_indices(s.shape[0])] += z
            else:
                s += z * self.b
            return ("d", sla.lu_factor(s, overwrite_a=True, check_finite=False))
        fa, fb, kl = self.band
        s = -fa.astype(np.complex128)
        if fb is None:
            s[kl] += z
        else:
            s += z * fb
        ab = np.zeros((3 * kl + 1, s.shape[1]), dtype=np.complex128, order="F")
        ab[kl:] = s
        lu, piv, info = lapack.zgbtrf(ab, kl, kl, overwrite_ab=1)
        assert info == 0
        return ("b", (lu, piv, kl))

    def _solve(self, f, rhs, trans):
        if f[0] == "d":
            return sla.lu_solve(f[1], rhs, trans=trans, check_finite=False)
        lu, piv, kl = f[1]
        x, info = lapack.zgbtrs(lu, kl, kl, np.asarray(rhs, dtype=np.complex128), piv, trans=trans)
        return x

    def _mult(self, mat, x):
        if self.band is None:
            return mat @ x
        return fband.band_matvec(mat, x)

    def run(self):
        k = self.k
        f = None
        task = k.step()
        while task != fl.RciTask.DONE:
            t0 = time.time()
            if task == fl.RciTask.FACTORIZE:
                z = complex(k.ze)
                if z not in self.factors:
                    self.factors[z] = self._factor(z)
                f = self.factors[z]
                self.t["factor"] += time.time() - t0
            elif task == fl.RciTask.SOLVE:
                k.work2[:, :k.m0] = self._solve(f, k.work2[:, :k.m0], 0)
                self.t["solve"] += time.time() - t0
            elif task == fl.RciTask.SOLVE_ADJOINT:
                k.work2[:, :k.m0] = self._solve(f, k.work2[:, :k.m0], 2)
                self.t["solve"] += time.time() - t0
            elif task in (fl.RciTask.MULTIPLY_A, fl.RciTask.MULTIPLY_B):
                s = k.multiply_columns
                if task == fl.RciTask.MULTIPLY_A:
                    k.work1[:, s] = self._mult(self.a if self.band is None else self.band[0], k.x[:, s])
                else:
                    mat = self.b if self.band is None else self.band[1]
                    k.work1[:, s] = k.x[:, s] if mat is None else self._mult(mat, k.x[:, s])
                self.t["mult"] += time.time() - t0
            task = k.step()
        return k.result


def run_kernel_lapack(w, verbose_trace=True):
    """Drive the reference kernel for a workloads.Workload with LAPACK."""
    import contextlib
    import io
    cls = fl.HermitianRci if w.hermitian else fl.SymmetricRci
    fpm = fl.feastinit()
    fpm.set_slot(2, w.ne)
    fpm.set_slot(1, 1)                       # runtime report: per-loop trace lines
    k = cls(w.n, w.m0, w.emin, w.emax, fpm)
    if w.kind == "dense":
        caller = LapackCaller(k, a=w.a, b=w.b)
    else:
        kl = max(w.kla, w.klb)
        fa = fband._pad_band(fband.expand_band(w.a, w.kla, w.uplo, w.hermitian), w.kla, kl)
        fb = fband._pad_band(fband.expand_band(w.b, w.klb, w.uplo, w.hermitian), w.klb, kl)
        caller = LapackCaller(k, band=(fa, fb, kl))
    buf = io.StringIO()
    t0 = time.time()
    with contextlib.redirect_stdout(buf):
        r = caller.run()
    wall = time.time() - t0
    hist = []
    for line in buf.getvalue().splitlines():
        p = line.split()
        if len(p) == 5 and p[0].isdigit():
            hist.append([float(v) for v in p])
    return r, np.array(hist), wall, caller.t


def make_config(tag, w):
    r, hist, wall, t = run_kernel_lapack(w)
    out = {}
    _pack("", r, out)
    out["x"] = r.x[:, : r.m] if w.n * r.m <= 250_000 else np.zeros((0, 0))
    out["history"] = hist
    out["meta"] = np.array([w.n, w.m0, w.emin, w.emax, wall, t["factor"], t["solve"], t["mult"]])
    a_sum = np.array([np.sum(w.a), np.sum(np.abs(w.a))])
    out["a_checksum"] = a_sum
    _save(f"{tag}.npz", **out)
    print(f"{tag}: info={r.info} m={r.m} loop={r.loop} maxres={np.max(r.res[: r.m]) if r.m else 0:.2e} "
          f"wall={wall:.1f}s {t}")


def _sparse_cases():
    """Seeded CSR pencils for the sparse golden: (name, kind, a, b, uplo, m0,
    solver, iter_tol, fpm slots).  Node numbering is shuffled so the matrices
    are NOT banded in the given order (the GPU reorders them)."""
    from paper_1203_4031_b200.sparse import CsrMatrix as C
    rng = np.random.default_rng(1203)
    cases = []
    # 2-D 5-point Laplacian on a 12 x 15 grid + random diagonal, shuffled
    gx, gy = 12, 15
    n = gx * gy
    lap = np.zeros((n, n))
    for i in range(gx):
        for j in range(gy):
            k = i * gy + j
            lap[k, k] = 4.0 + 0.3 * rng.random()
            for di, dj in ((1, 0), (0, 1)):
                if i + di < gx and j + dj < gy:
                    l = (i + di) * gy + j + dj
                    lap[k, l] = lap[l, k] = -1.0
    p = rng.permutation(n)
    lap = lap[np.ix_(p, p)]
    cases.append(("lap2d", lap, None, "F", False))
    # 1-D FEM stiffness with random coefficients (pentadiagonal) / mass, lower storage, shuffled
    n = 250
    a = np.zeros((n, n))
    for d, s in ((0, 2.0), (1, -0.7), (2, 0.2)):
        v = s * (1 + 0.2 * rng.standard_normal(n - d))
        a += np.diag(v, -d) + (np.diag(v, d) if d else 0)
    b = (4 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1)) / 6
    p = rng.permutation(n)
    cases.append(("fem1d_gv", a[np.ix_(p, p)], b[np.ix_(p, p)], "L", False))
    # complex Hermitian random sparse pattern (~6 per row), upper storage
    n = 200
    h = np.zeros((n, n), dtype=complex)
    for _ in range(3 * n):
        i, j = rng.integers(0, n, 2)
        if i != j:
            v = rng.standard_normal() + 1j * rng.standard_normal()
            h[i, j] += v
            h[j, i] += np.conj(v)
    h += np.diag(rng.uniform(-3, 3, n))
    cases.append(("herm_rand", h, None, "U", True))
    # Hermitian generalized on the Laplacian's pattern, B = mass-like SPD with a different pattern
    n = 180
    hb = lap.astype(complex)
    iu = np.triu_indices(n, 1)
    nz = np.abs(hb[iu]) > 0
    ph = np.exp(1j * rng.uniform(0, 2 * np.pi, nz.sum()))
    vals = hb[iu].copy()
    vals[nz] = vals[nz] * ph
    hb[iu] = vals
    hb[(iu[1], iu[0])] = np.conj(vals)
    bb = np.eye(n) * 1.2 + 0.05 * (np.eye(n, k=1) + np.eye(n, k=-1))
    cases.append(("herm_gv", hb, bb.astype(complex), "F", True))
    return cases


def make_sparse():
    """feast_scsr / feast_hcsr golden runs of the reference (direct and
    iterative inner solver) on the seeded pencils of _sparse_cases()."""
    import scipy.linalg as sla
    out = {}

    def gap(ev, lo, hi):
        return 0.5 * (ev[lo - 1] + ev[lo]) if lo > 0 else ev[0] - 0.1, 0.5 * (ev[hi] + ev[hi + 1])

    for name, a, b, uplo, herm in _sparse_cases():
        ev = sla.eigh(a, b, eigvals_only=True)
        mid = int(np.argmin(np.abs(ev - np.median(ev))))
        emin, emax = gap(ev, mid - 4, mid + 5)        # interior: 10 eigenvalues
        lmin, lmax = gap(ev, 0, 7)                    # lowest 8 eigenvalues
        ca = fl.CsrMatrix.from_dense(a, uplo)
        cb = None if b is None else fl.CsrMatrix.from_dense(b, uplo)
        out[name + "_ia"], out[name + "_ja"], out[name + "_v"] = ca.ia, ca.ja, ca.values
        if cb is not None:
            out[name + "_bia"], out[name + "_bja"], out[name + "_bv"] = cb.ia, cb.ja, cb.values
        out[name + "_meta"] = np.array([a.shape[0], emin, emax, 16, int(herm), "FLU".index(uplo), lmin, lmax])
        fn = fl.feast_hcsr if herm else fl.feast_scsr
        runs = [("direct", 1e-3, emin, emax, "")]
        if name in ("lap2d", "fem1d_gv"):
            runs += [("iterative", 1e-10, lmin, lmax, "_low"), ("iterative", 1e-3, lmin, lmax, "_low")]
        if name == "lap2d":
            runs += [("iterative", 1e-10, emin, emax, "")]   # reference ends with info -2 (no convergence)
        for solver, tol, e0, e1, where in runs:
            tag = f"{name}_{solver}{'' if solver == 'direct' else '_%g' % tol}{where}"
            t0 = time.time()
            r = fn(ca, e0, e1, 16, b=cb, options=fl.SolverOptions(solver=solver, iter_tol=tol))
            _pack(tag + "_", r, out)
            print(f"{tag}: info={r.info} m={r.m} loop={r.loop} "
                  f"maxres={np.max(r.res[:r.m]) if r.m else 0:.2e} {time.time() - t0:.1f}s")
    _save("sparse.npz", **out)


def make_c3_trajectories(ks):
    """Config 3 under 1-ulp perturbations A*(1 + k*2^-52): the reference
    kernel's trajectory (final M0 after the loop-0 shrink, loop count, info,
    per-loop history) for each k, so the GPU run can be compared with the
    reference trajectory that has the same post-shrink M0 (the shrink index is
    decided at rounding level, kernel.py:385-400;
    profiles/r01_c3_ref_sensitivity.txt)."""
    from paper_1203_4031_b200 import workloads as W
    w = W.c3_heev()
    a0 = w.a.copy()
    out = {}
    path = os.path.join(HERE, "c3_trajectories.npz")
    if os.path.exists(path):
        out = dict(np.load(path))
    for k in ks:
        w.a = a0 * (1.0 + k * 2.0 ** -52)
        r, hist, wall, _ = run_kernel_lapack(w)
        m = int(r.m)
        out[f"k{k}_scal"] = np.array([k, r.m0, r.loop, r.info, m], dtype=np.int64)
        out[f"k{k}_e"] = r.e[:m]
        out[f"k{k}_res"] = r.res[:m]
        out[f"k{k}_history"] = hist
        print(f"c3 k={k}: m0={r.m0} loop={r.loop} info={r.info} m={m} "
              f"maxres={np.max(r.res[:m]):.2e} wall={wall:.0f}s", flush=True)
        _save("c3_trajectories.npz", **out)


if __name__ == "__main__":
    from paper_1203_4031_b200 import workloads as W
    what = sys.argv[1:] or ["unit", "small"]
    if "unit" in what:
        make_unit()
    if "small" in what:
        make_small()
    if "sparse" in what:
        make_sparse()
    if "c3traj" in what:
        make_c3_trajectories([int(v) for v in os.environ.get("C3_KS", "0 1 2 3 4 5").split()])
    if "scaled" in what:
        for tag in ("c1s", "c2s", "c3s", "c5s", "c4s"):
            make_config(f"scaled_{tag}", W.scaled(tag))
    if "c5m" in what:
        # mid-size config-5 pencil: place the interval mid-gap around the 150
        # eigenvalues nearest 0 (independent LAPACK zhegvx), then the reference
        # kernel + LAPACK caller
        w = W.c5m_hegv(interval=(-1.0, 1.0))
        if W.C5M_INTERVAL is None:
            t0 = time.time()
            ev = sla.eigh(w.a, w.b, eigvals_only=True, subset_by_value=(-0.03, 0.03), driver="gvx")
            i0 = int(np.searchsorted(ev, 0.0))
            lo, hi = i0 - 75, i0 + 75
            w.emin, w.emax = 0.5 * (ev[lo - 1] + ev[lo]), 0.5 * (ev[hi - 1] + ev[hi])
            w.expect_m = 150
            print(f"C5M_INTERVAL = ({w.emin!r}, {w.emax!r})  count 150  gaps "
                  f"{ev[lo] - ev[lo - 1]:.2e} {ev[hi] - ev[hi - 1]:.2e}  ({time.time() - t0:.0f}s)", flush=True)
        else:
            (w.emin, w.emax), w.expect_m = W.C5M_INTERVAL, W.C5M_COUNT
        make_config("mid_c5m", w)
    for tag, fn in (("c1", W.c1_syev), ("c2", W.c2_sygv), ("c3", W.c3_heev), ("c4", W.c4_sbgv)):
        if tag in what:
            make_config(f"full_{tag}", fn())
