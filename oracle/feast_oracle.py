"""numpy restatement of the reference FEAST hot path — TEST INFRASTRUCTURE ONLY.

Every function cites the reference location it restates (paths relative to
``/root/reference/pkg/src/feastlib``).  The restatement is written as plain
loops over numpy primitives so it can be checked line by line against the
reference; the ``Lapack*Ops`` classes answer the same tasks with LAPACK
(scipy) so that the BASELINE configurations finish in minutes, exactly as the
survey's "reference kernel + LAPACK caller" oracle.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "ALLOWED_NE", "splitmix_uniform", "start_block", "default_fpm", "gl_rule", "half_circle", "accumulate",
    "expand_uplo", "lu_factor_ref", "lu_solve_ref", "expand_band", "pad_band",
    "band_matvec", "band_lu_factor_ref", "band_lu_solve_ref", "cholesky_lower",
    "reduced_eig", "column_residuals", "finalize_order", "OracleResult",
    "oracle_feast", "RefDenseOps", "RefBandOps", "LapackDenseOps",
    "LapackBandOps", "oracle_feast_sy", "oracle_feast_he", "oracle_feast_sb",
    "CsrDirectOps", "CsrIterativeOps", "oracle_feast_csr",
]

# params.py:11 — supported Gauss-Legendre orders
ALLOWED_NE = (3, 4, 5, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48)
# params.py:18 — defaults of the 64-slot control vector (1-based slot: value)
DEFAULT_FPM = {1: 0, 2: 8, 3: 12, 4: 20, 5: 0, 6: 0, 7: 5, 14: 0}


def default_fpm():
    v = [0] * 65                       # index 0 unused: v[i] == fpm(i)
    for k, val in DEFAULT_FPM.items():
        v[k] = val
    return v


# --------------------------------------------------------------------------
# kernel.py:84-102 — counter-based SplitMix64 stream mapped to [-1, 1)
# --------------------------------------------------------------------------
_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix_uniform(seed: int, offset: int, count: int) -> np.ndarray:
    ctr = np.arange(offset + 1, offset + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        s = np.uint64(seed % (1 << 64)) + ctr * _G
        s = (s ^ (s >> np.uint64(30))) * _M1
        s = (s ^ (s >> np.uint64(27))) * _M2
    s ^= s >> np.uint64(31)
    return (s >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0


def start_block(seed, n, m0, hermitian):
    """kernel.py:496-498 (real) and 521-525 (complex: reals then imags)."""
    if hermitian:
        raw = splitmix_uniform(seed, 0, 2 * n * m0)
        v = raw[: n * m0] + 1j * raw[n * m0:]
    else:
        v = splitmix_uniform(seed, 0, n * m0)
    return v.reshape((n, m0), order="F")


# --------------------------------------------------------------------------
# quadrature.py:41-95 — Gauss-Legendre by Newton from Chebyshev-angle guesses
# --------------------------------------------------------------------------
def _legendre(n, x):
    p0 = np.ones_like(x)
    p1 = x.copy()
    for j in range(2, n + 1):
        p0, p1 = p1, ((2 * j - 1) * x * p1 - (j - 1) * p0) / j
    return p1, n * (x * p1 - p0) / (x * x - 1.0)


def gl_rule(ne: int):
    """Return (nodes ascending, weights); paired nodes are exact negations."""
    if ne not in ALLOWED_NE:
        raise ValueError(f"unsupported order {ne}")
    k = np.arange(1, ne // 2 + 1)
    x = np.cos(math.pi * (k - 0.25) / (ne + 0.5))
    for _ in range(100):
        p, dp = _legendre(ne, x)
        dx = p / dp
        x = x - dx
        if np.max(np.abs(dx)) < 1e-16:
            break
    _, dp = _legendre(ne, x)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    xp, wp = x[::-1], w[::-1]                     # ascending positive half
    if ne % 2:
        _, d0 = _legendre(ne, np.array([0.0]))
        nodes = np.concatenate([-xp[::-1], [0.0], xp])
        weights = np.concatenate([wp[::-1], 2.0 / (d0 * d0), wp])
    else:
        nodes = np.concatenate([-xp[::-1], xp])
        weights = np.concatenate([wp[::-1], wp])
    return nodes, weights


def half_circle(nodes, weights, emin, emax):
    """quadrature.py:87-95: theta = -(pi/2)(x-1), z = c + r e^{i theta}."""
    if not emin < emax:
        raise ValueError("emin >= emax")
    r = (emax - emin) / 2.0
    c = (emax + emin) / 2.0
    theta = -(np.pi / 2.0) * (nodes - 1.0)
    z = c + r * np.exp(1j * theta)
    return theta, z, weights.copy(), r, c


# --------------------------------------------------------------------------
# kernel.py:108-124 — quadrature accumulation
# --------------------------------------------------------------------------
def accumulate(q, x, w, r, theta, variant):
    if q.shape != x.shape:
        raise ValueError("shape mismatch")
    if variant == "symmetric":
        q -= (w / 2.0) * (r * np.exp(1j * theta) * x).real
    elif variant == "hermitian-direct":
        q -= (w / 4.0) * r * np.exp(1j * theta) * x
    elif variant == "hermitian-adjoint":
        q -= (w / 4.0) * r * np.exp(-1j * theta) * x
    else:
        raise ValueError(variant)


# --------------------------------------------------------------------------
# dense.py:15-88 — UPLO expansion and the unblocked partial-pivoting LU
# --------------------------------------------------------------------------
def expand_uplo(a, uplo, hermitian):
    uplo = uplo.upper()
    if uplo == "F":
        return np.asarray(a)
    t = np.tril(a) if uplo == "L" else np.triu(a)
    strict = t - np.diag(np.diag(t))
    return t + (strict.conj().T if hermitian else strict.T)


class SingularPivot(Exception):
    pass


def lu_factor_ref(a):
    """dense.py:30-50: right-looking LU, argmax |.| pivot, full-row swaps."""
    lu = np.array(a, dtype=np.complex128, copy=True)
    n = lu.shape[0]
    piv = np.arange(n)
    for k in range(n):
        p = k + int(np.argmax(np.abs(lu[k:, k])))
        if lu[p, k] == 0:
            raise SingularPivot(k)
        piv[k] = p
        if p != k:
            lu[[k, p]] = lu[[p, k]]
        if k + 1 < n:
            lu[k + 1:, k] /= lu[k, k]
            lu[k + 1:, k + 1:] -= np.outer(lu[k + 1:, k], lu[k, k + 1:])
    return lu, piv


def lu_solve_ref(factor, b, adjoint=False):
    """dense.py:53-88: pivots up front, unit-L forward, U backward; the
    adjoint goes U^H forward, L^H backward, then pivots in reverse."""
    lu, piv = factor
    n = lu.shape[0]
    x = np.array(b, dtype=np.complex128, copy=True)
    vec = x.ndim == 1
    if vec:
        x = x[:, None]
    if not adjoint:
        for k in range(n):
            if piv[k] != k:
                x[[k, piv[k]]] = x[[piv[k], k]]
        for k in range(n - 1):
            x[k + 1:] -= np.outer(lu[k + 1:, k], x[k])
        for k in range(n - 1, -1, -1):
            x[k] /= lu[k, k]
            if k:
                x[:k] -= np.outer(lu[:k, k], x[k])
    else:
        for k in range(n):
            if k:
                x[k] -= lu[:k, k].conj() @ x[:k]
            x[k] /= np.conj(lu[k, k])
        for k in range(n - 1, -1, -1):
            if k + 1 < n:
                x[k] -= lu[k + 1:, k].conj() @ x[k + 1:]
        for k in range(n - 1, -1, -1):
            if piv[k] != k:
                x[[k, piv[k]]] = x[[piv[k], k]]
    return x[:, 0] if vec else x


# --------------------------------------------------------------------------
# banded.py:16-146 — band storage, band matvec, band LU and solves
# --------------------------------------------------------------------------
def band_rows_needed(kl, uplo):
    """banded.py:16-18."""
    return 2 * kl + 1 if uplo.upper() == "F" else kl + 1


def expand_band(ab, kl, uplo, hermitian):
    """banded.py:21-47: to the full-band layout, row kl+s = s-th subdiagonal
    (entry A[j+s, j] at [kl+s, j]); out-of-pattern slots are never read."""
    ab = np.asarray(ab)
    n = ab.shape[1]
    uplo = uplo.upper()
    fb = np.zeros((2 * kl + 1, n), dtype=ab.dtype)
    if uplo == "F":
        fb[kl] = ab[kl]
        for d in range(1, kl + 1):
            fb[kl - d, d:] = ab[kl - d, d:]
            fb[kl + d, :n - d] = ab[kl + d, :n - d]
    elif uplo == "L":
        fb[kl] = ab[0]
        for d in range(1, kl + 1):
            s = ab[d, :n - d]
            fb[kl + d, :n - d] = s
            fb[kl - d, d:] = np.conj(s) if hermitian else s
    else:
        fb[kl] = ab[kl]
        for d in range(1, kl + 1):
            s = ab[kl - d, d:]
            fb[kl - d, d:] = s
            fb[kl + d, :n - d] = np.conj(s) if hermitian else s
    return fb


def pad_band(fb, kl_from, kl_to):
    """banded.py:181-187."""
    if kl_from == kl_to:
        return fb
    out = np.zeros((2 * kl_to + 1, fb.shape[1]), dtype=fb.dtype)
    out[kl_to - kl_from:kl_to + kl_from + 1] = fb
    return out


def band_matvec(fb, x):
    """banded.py:50-65: y[j+s] += fb[kl+s, j] x[j] for every diagonal s."""
    n = fb.shape[1]
    kl = (fb.shape[0] - 1) // 2
    y = np.zeros((n,) + x.shape[1:], dtype=np.result_type(fb.dtype, x.dtype))
    for s in range(-kl, kl + 1):
        j0, j1 = max(0, -s), min(n, n - s)
        if j1 <= j0:
            continue
        d = fb[kl + s, j0:j1]
        y[j0 + s:j1 + s] += (d[:, None] if x.ndim > 1 else d) * x[j0:j1]
    return y


def band_lu_factor_ref(fb, kl):
    """banded.py:68-103: dgbtf2-style band LU, kv = 2 kl working rows above
    the diagonal, argmax pivot over <= kl+1 rows."""
    n = fb.shape[1]
    kv = 2 * kl
    ab = np.zeros((3 * kl + 1, n), dtype=np.complex128)
    ab[kl:] = fb
    ipiv = np.arange(n)
    ju = 0
    for j in range(n):
        km = min(kl, n - 1 - j)
        jp = int(np.argmax(np.abs(ab[kv:kv + km + 1, j])))
        if ab[kv + jp, j] == 0:
            raise SingularPivot(j)
        ipiv[j] = j + jp
        ju = max(ju, min(j + kl + jp, n - 1))
        if jp:
            cols = np.arange(j, ju + 1)
            hi = kv + jp + j - cols
            lo = kv + j - cols
            t = ab[hi, cols].copy()
            ab[hi, cols] = ab[lo, cols]
            ab[lo, cols] = t
        if km > 0:
            ab[kv + 1:kv + 1 + km, j] /= ab[kv, j]
            l = ab[kv + 1:kv + 1 + km, j]
            for c in range(j + 1, ju + 1):
                u = ab[kv + j - c, c]
                if u != 0:
                    ab[kv + j - c + 1:kv + j - c + 1 + km, c] -= l * u
    return ab, ipiv, kl


def band_lu_solve_ref(factor, b, adjoint=False):
    """banded.py:106-146."""
    ab, ipiv, kl = factor
    n = ab.shape[1]
    kv = 2 * kl
    x = np.array(b, dtype=np.complex128, copy=True)
    vec = x.ndim == 1
    if vec:
        x = x[:, None]
    if not adjoint:
        if kl > 0:
            for j in range(n - 1):
                p = ipiv[j]
                if p != j:
                    x[[j, p]] = x[[p, j]]
                km = min(kl, n - 1 - j)
                if km:
                    x[j + 1:j + 1 + km] -= ab[kv + 1:kv + 1 + km, j][:, None] * x[j]
        for j in range(n - 1, -1, -1):
            x[j] /= ab[kv, j]
            lm = min(kv, j)
            if lm:
                x[j - lm:j] -= ab[kv - lm:kv, j][:, None] * x[j]
    else:
        for j in range(n):
            lm = min(kv, j)
            if lm:
                x[j] -= ab[kv - lm:kv, j].conj() @ x[j - lm:j]
            x[j] /= np.conj(ab[kv, j])
        if kl > 0:
            for j in range(n - 2, -1, -1):
                km = min(kl, n - 1 - j)
                if km:
                    x[j] -= ab[kv + 1:kv + 1 + km, j].conj() @ x[j + 1:j + 1 + km]
                p = ipiv[j]
                if p != j:
                    x[[j, p]] = x[[p, j]]
    return x[:, 0] if vec else x


# --------------------------------------------------------------------------
# reduced.py:22-218 — Cholesky, Householder tridiagonalisation, implicit QL
# --------------------------------------------------------------------------
class ReducedFailure(Exception):
    pass


def cholesky_lower(b):
    """reduced.py:22-40: (L, None) or (None, 1-based failing pivot)."""
    b = np.asarray(b)
    n = b.shape[0]
    L = np.zeros_like(b)
    for j in range(n):
        d = (b[j, j] - L[j, :j] @ L[j, :j].conj()).real
        if not (d > 0.0) or not np.isfinite(d):
            return None, j + 1
        L[j, j] = np.sqrt(d)
        if j + 1 < n:
            L[j + 1:, j] = (b[j + 1:, j] - L[j + 1:, :j] @ L[j, :j].conj()) / L[j, j]
    return L, None


def _fwd(L, rhs):
    x = np.array(rhs, copy=True)
    for i in range(L.shape[0]):
        if i:
            x[i] -= L[i, :i] @ x[:i]
        x[i] /= L[i, i]
    return x


def _bwd_adj(L, rhs):
    x = np.array(rhs, copy=True)
    n = L.shape[0]
    for i in range(n - 1, -1, -1):
        if i + 1 < n:
            x[i] -= L[i + 1:, i].conj() @ x[i + 1:]
        x[i] /= np.conj(L[i, i])
    return x


def _householder_tridiag(a):
    """reduced.py:65-114."""
    a = np.array(a, copy=True)
    n = a.shape[0]
    cplx = np.iscomplexobj(a)
    v = np.eye(n, dtype=a.dtype)
    for k in range(n - 2):
        x = a[k + 1:, k].copy()
        nx = np.linalg.norm(x)
        if nx == 0.0:
            continue
        ph = x[0] / abs(x[0]) if x[0] != 0 else 1.0
        alpha = -ph * nx
        u = x.copy()
        u[0] -= alpha
        nu = np.linalg.norm(u)
        if nu == 0.0:
            continue
        u /= nu
        s = a[k + 1:, k + 1:]
        p = 2.0 * (s @ u)
        kap = (u.conj() @ p).real
        s -= np.outer(p, u.conj())
        s -= np.outer(u, p.conj())
        s += (2.0 * kap) * np.outer(u, u.conj())
        a[k + 1, k] = alpha
        a[k + 2:, k] = 0.0
        a[k, k + 1:] = a[k + 1:, k].conj()
        v[:, k + 1:] -= 2.0 * np.outer(v[:, k + 1:] @ u, u.conj())
    d = a.diagonal().real.astype(np.float64).copy()
    e = np.zeros(max(n - 1, 0))
    if n > 1:
        sub = np.diagonal(a, -1).copy()
        if cplx:
            ph = np.ones(n, dtype=a.dtype)
            for j in range(n - 1):
                mag = abs(sub[j])
                ph[j + 1] = ph[j] * (sub[j] / mag) if mag != 0 else ph[j]
                e[j] = mag
            v = v * ph[None, :]
        else:
            e[:] = sub.real
    return d, e, v


def _implicit_ql(d, e, z, max_sweeps=30):
    """reduced.py:117-172 (Wilkinson shift, <= 30 sweeps per eigenvalue)."""
    n = d.shape[0]
    eps = np.finfo(np.float64).eps
    if n == 1:
        return
    ee = np.zeros(n)
    ee[:n - 1] = e
    for l in range(n):
        sweeps = 0
        while True:
            m = l
            while m < n - 1:
                if abs(ee[m]) <= eps * (abs(d[m]) + abs(d[m + 1])):
                    break
                m += 1
            if m == l:
                break
            sweeps += 1
            if sweeps > max_sweeps:
                raise ReducedFailure(l)
            g = (d[l + 1] - d[l]) / (2.0 * ee[l])
            r = math.hypot(g, 1.0)
            g = d[m] - d[l] + ee[l] / (g + (r if g >= 0 else -r))
            s = c = 1.0
            p = 0.0
            broke = False
            for i in range(m - 1, l - 1, -1):
                f = s * ee[i]
                b = c * ee[i]
                r = math.hypot(f, g)
                ee[i + 1] = r
                if r == 0.0:
                    d[i + 1] -= p
                    ee[m] = 0.0
                    broke = True
                    break
                s = f / r
                c = g / r
                g = d[i + 1] - p
                r = (d[i] - g) * s + 2.0 * c * b
                p = s * r
                d[i + 1] = g + p
                g = c * r - b
                zi = z[:, i].copy()
                z[:, i] = c * zi - s * z[:, i + 1]
                z[:, i + 1] = s * zi + c * z[:, i + 1]
            if not broke:
                d[l] -= p
                ee[l] = g
                ee[m] = 0.0


def reduced_eig(aq, bq, method="restated"):
    """reduced.py:188-218: eigenpairs of aq phi = eps bq phi, ascending,
    phi^H bq phi = I.  ``method='lapack'`` swaps the restated tridiagonal QL
    for LAPACK (only used to keep the large-M0 oracle runs fast)."""
    aq = np.asarray(aq)
    bq = np.asarray(bq)
    n = aq.shape[0]
    if not (np.all(np.isfinite(aq)) and np.all(np.isfinite(bq))):
        raise ReducedFailure("non-finite")
    if n == 1:
        b00 = bq[0, 0].real
        if b00 <= 0:
            raise ReducedFailure("b00")
        return (np.array([aq[0, 0].real / b00]),
                np.full((1, 1), 1.0 / np.sqrt(b00), dtype=aq.dtype))
    if method == "lapack":
        import scipy.linalg as sla
        try:
            return sla.eigh(aq, bq)
        except np.linalg.LinAlgError as exc:  # pragma: no cover
            raise ReducedFailure(str(exc))
    L, fail = cholesky_lower(bq)
    if fail is not None:
        raise ReducedFailure(fail)
    c = _fwd(L, aq)
    c = _fwd(L, c.conj().T).conj().T
    c = 0.5 * (c + c.conj().T)
    d, e, v = _householder_tridiag(c)
    _implicit_ql(d, e, v)
    order = np.argsort(d, kind="stable")
    return d[order], _bwd_adj(L, v[:, order])


# --------------------------------------------------------------------------
# kernel.py:147-177, 446-466 — residuals, spurious flagging, output order
# --------------------------------------------------------------------------
def column_residuals(ax, bx, lam, scale):
    num = np.abs(ax - lam[None, :] * bx).sum(axis=0)
    den = np.abs(scale * bx).sum(axis=0)
    out = np.full(lam.shape, np.inf)
    ok = den > 0.0
    out[ok] = num[ok] / den[ok]
    return out


def finalize_order(e, x, res, emin, emax, tol):
    """kernel.py:446-466 + 156-177, in place; returns m."""
    m0 = e.shape[0]
    ins = (e >= emin) & (e <= emax) & np.isfinite(res) & (res >= 0)
    if ins.any():
        thr = max(100.0 * float(np.median(res[ins])), tol * 1.0e4)
        res[ins & (res > thr)] = -1.0
    spur = (res < 0) | ~np.isfinite(res)
    inside = (e >= emin) & (e <= emax) & ~spur
    outside = ~inside & ~spur
    idx = np.nonzero(inside)[0]
    idx = idx[np.argsort(e[idx], kind="stable")]
    order = np.concatenate([idx, np.nonzero(outside)[0], np.nonzero(spur)[0]])
    e[:] = e[order]
    x[:, :m0] = x[:, order]
    res[:] = res[order]
    if spur.any():
        res[m0 - int(spur.sum()):] = -1.0
    return len(idx)


# --------------------------------------------------------------------------
# kernel.py:328-444 — the refinement loop, written as a straight function
# --------------------------------------------------------------------------
@dataclass
class OracleResult:
    e: np.ndarray
    x: np.ndarray
    m: int
    res: np.ndarray
    epsout: float
    loop: int
    info: int
    m0: int
    history: list = field(default_factory=list)   # per loop (m, trace, epsout, maxres)


def _validate(n, m0, emin, emax, fpm):
    """params.py:88-123 precedence: 202, 201, 200, then 100+i."""
    if n <= 0:
        return 202
    if m0 > n or m0 <= 0:
        return 201
    if emin >= emax:
        return 200
    checks = ((1, lambda v: v in (0, 1)), (2, lambda v: v in ALLOWED_NE),
              (3, lambda v: v >= 1), (4, lambda v: v >= 0),
              (5, lambda v: v in (0, 1)), (6, lambda v: v in (0, 1)),
              (7, lambda v: v >= 1), (14, lambda v: v in (0, 1)))
    for i, ok in checks:
        if not ok(fpm[i]):
            return 100 + i
    return 0


def oracle_feast(ops, n, m0, emin, emax, *, hermitian, fpm=None, seed=42,
                 x0=None, reduced="restated"):
    """Run one FEAST solve against an ops object (factorize(z) / solve /
    solve_adjoint / multiply_a / multiply_b), following kernel.py:328-444.
    Factorizations are cached per shift as in _driver.py:45,66-70."""
    fpm = default_fpm() if fpm is None else list(fpm)
    wdt = np.complex128 if hermitian else np.float64
    m0_alloc = m0
    info = _validate(n, m0, emin, emax, fpm)
    e = np.zeros(max(m0, 0))
    res = np.zeros(max(m0, 0))
    x = np.zeros((max(n, 0), max(m0, 0)), dtype=wdt)
    if info:
        return OracleResult(e, x, 0, res, 1.0, 0, info, m0)
    tol = 10.0 ** -min(fpm[3], 16)
    nodes, weights = gl_rule(fpm[2])
    theta, zs, ws, r, _ = half_circle(nodes, weights, emin, emax)
    scale = max(abs(emin), abs(emax))
    hist = []
    factors = {}
    if fpm[5] == 1:
        x[:, :] = np.asarray(x0)[:, :m0]
        y = np.asarray(ops.multiply_b(x[:, :m0]), dtype=wdt).copy()
    else:
        y = start_block(seed, n, m0_alloc, hermitian).astype(wdt)
    trace_prev = None
    loop = 0
    while True:
        q = np.zeros((n, m0), dtype=wdt)
        for k in range(len(zs)):
            z = complex(zs[k])
            if z not in factors:
                factors[z] = ops.factorize(z)
            f = factors[z]
            xk = ops.solve(f, y[:, :m0].astype(np.complex128))
            accumulate(q, xk, ws[k], r, theta[k],
                       "hermitian-direct" if hermitian else "symmetric")
            if hermitian:
                xk = ops.solve_adjoint(f, y[:, :m0].astype(np.complex128))
                accumulate(q, xk, ws[k], r, theta[k], "hermitian-adjoint")
        if fpm[14] == 1:
            x[:, :m0] = q
            return OracleResult(e, x, 0, res, 1.0, loop, 4, m0, hist)
        aq_full = np.asarray(ops.multiply_a(q))
        bq_full = np.asarray(ops.multiply_b(q))
        qh = q.conj().T
        aq = qh @ aq_full
        bq = qh @ bq_full
        aq = 0.5 * (aq + aq.conj().T)
        bq = 0.5 * (bq + bq.conj().T)
        while m0 > 0:
            _, fail = cholesky_lower(bq[:m0, :m0])
            if fail is None:
                break
            m0 = fail - 1
        if m0 == 0:
            return OracleResult(e, x, 0, res, 1.0, loop, -3, 0, hist)
        if m0 < q.shape[1]:
            x[:, m0:] = 0
            e[m0:] = 0
            res[m0:] = 0
        try:
            lam, phi = reduced_eig(aq[:m0, :m0], bq[:m0, :m0], method=reduced)
        except ReducedFailure:
            return OracleResult(e, x, 0, res, 1.0, loop, -3, m0, hist)
        e[:m0] = lam
        x[:, :m0] = q[:, :m0] @ phi
        r_ = column_residuals(aq_full[:, :m0] @ phi, bq_full[:, :m0] @ phi, lam, scale)
        res[:m0] = r_
        inside = (lam >= emin) & (lam <= emax)
        m = int(inside.sum())
        tr = float(lam[inside].sum())
        epsout = 1.0 if trace_prev is None else abs(tr - trace_prev) / scale
        maxres = float(r_[inside].max()) if m else 0.0
        hist.append((m, tr, epsout, maxres))
        if m == 0:
            code = 1
        elif (epsout < tol) if fpm[6] == 0 else (maxres < tol):
            code = 3 if (m == m0 and m0 < n) else 0
        elif loop >= fpm[4]:
            code = 3 if (m == m0 and m0 < n) else 2
        else:
            trace_prev = tr
            loop += 1
            y = np.zeros((n, m0_alloc), dtype=wdt)
            y[:, :m0] = ops.multiply_b(x[:, :m0])
            continue
        mm = finalize_order(e[:m0], x[:, :m0], res[:m0], emin, emax, tol)
        return OracleResult(e, x, mm, res, epsout, loop, code, m0, hist)


# --------------------------------------------------------------------------
# Ops objects (the _DenseOps / _BandedOps protocol, dense.py:91-117,
# banded.py:149-178): restated pure-numpy kernels and LAPACK-backed ones.
# --------------------------------------------------------------------------
class RefDenseOps:
    """dense.py:91-117 with the restated unblocked LU (small N only)."""

    def __init__(self, a, b=None):
        self.a, self.b = a, b

    def factorize(self, z):
        n = self.a.shape[0]
        s = (z * np.eye(n) if self.b is None else z * self.b) - self.a
        return lu_factor_ref(s)

    def solve(self, f, rhs):
        return lu_solve_ref(f, rhs)

    def solve_adjoint(self, f, rhs):
        return lu_solve_ref(f, rhs, adjoint=True)

    def multiply_a(self, x):
        return self.a @ x

    def multiply_b(self, x):
        return x.copy() if self.b is None else self.b @ x


class LapackDenseOps(RefDenseOps):
    """Same tasks answered by zgetrf/zgetrs (scipy)."""

    def factorize(self, z):
        import scipy.linalg as sla
        n = self.a.shape[0]
        s = -self.a.astype(np.complex128)
        if self.b is None:
            s[np.diag_indices(n)] += z
        else:
            s += z * self.b
        return sla.lu_factor(s, overwrite_a=True, check_finite=False)

    def solve(self, f, rhs):
        import scipy.linalg as sla
        return sla.lu_solve(f, rhs, trans=0, check_finite=False)

    def solve_adjoint(self, f, rhs):
        import scipy.linalg as sla
        return sla.lu_solve(f, rhs, trans=2, check_finite=False)


class RefBandOps:
    """banded.py:149-178 with the restated band LU (small N only)."""

    def __init__(self, fa, fb, kl):
        self.fa, self.fb, self.kl = fa, fb, kl

    def _shift(self, z):
        s = -self.fa.astype(np.complex128)
        if self.fb is None:
            s[self.kl] += z
        else:
            s += z * self.fb
        return s

    def factorize(self, z):
        return band_lu_factor_ref(self._shift(z), self.kl)

    def solve(self, f, rhs):
        return band_lu_solve_ref(f, rhs)

    def solve_adjoint(self, f, rhs):
        return band_lu_solve_ref(f, rhs, adjoint=True)

    def multiply_a(self, x):
        return band_matvec(self.fa, x)

    def multiply_b(self, x):
        return x.copy() if self.fb is None else band_matvec(self.fb, x)


class LapackBandOps(RefBandOps):
    """Same tasks answered by zgbtrf/zgbtrs (scipy.linalg.lapack)."""

    def factorize(self, z):
        from scipy.linalg import lapack
        kl = self.kl
        s = self._shift(z)                           # (2kl+1, n), row kl+s = sub s
        n = s.shape[1]
        # LAPACK gbtrf storage: ab[kl + ku + i - j, j] = A[i, j], ku = kl,
        # with kl extra rows on top for fill-in.  Our row kl+s holds A[j+s, j]
        # so it maps to LAPACK row 2kl + s.
        ab = np.zeros((3 * kl + 1, n), dtype=np.complex128, order="F")
        ab[kl:, :] = s
        lu, piv, info = lapack.zgbtrf(ab, kl, kl, overwrite_ab=1)
        if info > 0:
            raise SingularPivot(info - 1)
        return lu, piv

    def solve(self, f, rhs):
        from scipy.linalg import lapack
        lu, piv = f
        x, info = lapack.zgbtrs(lu, self.kl, self.kl, np.asarray(rhs, dtype=np.complex128), piv, trans=0)
        return x

    def solve_adjoint(self, f, rhs):
        from scipy.linalg import lapack
        lu, piv = f
        x, info = lapack.zgbtrs(lu, self.kl, self.kl, np.asarray(rhs, dtype=np.complex128), piv, trans=2)
        return x


# --------------------------------------------------------------------------
# driver-shaped conveniences (dense.py:120-183, banded.py:190-258)
# --------------------------------------------------------------------------
def oracle_feast_sy(a, emin, emax, m0, *, b=None, uplo="F", fpm=None, seed=42,
                    x0=None, lapack=True, reduced="restated"):
    a = expand_uplo(np.asarray(a, dtype=np.float64), uplo, False)
    b = None if b is None else expand_uplo(np.asarray(b, dtype=np.float64), uplo, False)
    ops = (LapackDenseOps if lapack else RefDenseOps)(a, b)
    return oracle_feast(ops, a.shape[0], m0, emin, emax, hermitian=False, fpm=fpm,
                        seed=seed, x0=x0, reduced=reduced)


def oracle_feast_he(a, emin, emax, m0, *, b=None, uplo="F", fpm=None, seed=42,
                    x0=None, lapack=True, reduced="restated"):
    a = expand_uplo(np.asarray(a, dtype=np.complex128), uplo, True)
    b = None if b is None else expand_uplo(np.asarray(b, dtype=np.complex128), uplo, True)
    ops = (LapackDenseOps if lapack else RefDenseOps)(a, b)
    return oracle_feast(ops, a.shape[0], m0, emin, emax, hermitian=True, fpm=fpm,
                        seed=seed, x0=x0, reduced=reduced)


def oracle_feast_sb(ab, kla, emin, emax, m0, *, b=None, klb=None, uplo="F",
                    fpm=None, seed=42, x0=None, lapack=True, hermitian=False,
                    reduced="restated"):
    dt = np.complex128 if hermitian else np.float64
    kl = max(kla, klb if b is not None else 0)
    fa = pad_band(expand_band(np.asarray(ab, dtype=dt), kla, uplo, hermitian), kla, kl)
    fb = None
    if b is not None:
        fb = pad_band(expand_band(np.asarray(b, dtype=dt), klb, uplo, hermitian), klb, kl)
    ops = (LapackBandOps if lapack else RefBandOps)(fa, fb, kl)
    return oracle_feast(ops, fa.shape[1], m0, emin, emax, hermitian=hermitian,
                        fpm=fpm, seed=seed, x0=x0, reduced=reduced)


# --------------------------------------------------------------------------
# CSR backend (sparse.py:316-462)
# --------------------------------------------------------------------------

class CsrDirectOps(LapackDenseOps):
    """_SparseOps(solver='direct') (sparse.py:430-462).  The reference's sparse
    LU (minimum-degree order, no pivoting, sparse.py:172-313) is an exact
    factorization of z*B - A, so its solves are answered here by zgetrf/zgetrs
    on the dense shifted matrix; A*x / B*x are the same products."""


class CsrIterativeOps(RefDenseOps):
    """_SparseOps(solver='iterative'): union pattern of A and B (B = I when
    absent) with aligned data (sparse.py:316-351), shifted data per z and
    conj(z) (sparse.py:394-409), and the diagonal-preconditioned BiCGStab of
    sparse.py:354-391 per right-hand-side column (sparse.py:411-427)."""

    def __init__(self, a, b=None, tol=1e-3):
        super().__init__(a, b)
        n = a.shape[0]
        mask = a != 0
        mask |= (np.eye(n, dtype=bool) if b is None else b != 0)
        self.rows, self.cols = np.nonzero(mask)          # row-major = sorted keys
        self.indptr = np.concatenate([[0], np.cumsum(np.bincount(self.rows, minlength=n))])
        self.a_data = a[self.rows, self.cols].astype(np.complex128)
        bd = np.eye(n) if b is None else b
        self.b_data = bd[self.rows, self.cols].astype(np.complex128)
        self.tol = tol

    def _matvec(self, data, x):
        y = np.zeros(len(self.indptr) - 1, dtype=np.complex128)
        contrib = data * x[self.cols]
        nz = np.flatnonzero(np.diff(self.indptr) > 0)
        y[nz] = np.add.reduceat(contrib, self.indptr[nz])
        return y

    def _operator(self, z):
        data = z * self.b_data - self.a_data
        diag = np.zeros(len(self.indptr) - 1, dtype=np.complex128)
        on = self.rows == self.cols
        diag[self.rows[on]] = data[on]
        diag[diag == 0] = 1.0
        return data, diag

    def factorize(self, z):
        return self._operator(z), self._operator(complex(z).conjugate())

    def _bicgstab(self, data, diag, b):
        """sparse.py:354-391, one column."""
        maxiter = max(8 * len(diag), 200)
        x = np.zeros_like(b)
        r = b.copy()
        bnorm = np.linalg.norm(b)
        if bnorm == 0:
            return x
        rhat = r.copy()
        rho = alpha = omega = 1.0 + 0j
        v = np.zeros_like(b)
        p = np.zeros_like(b)
        for _ in range(maxiter):
            rho1 = np.vdot(rhat, r)
            if rho1 == 0:
                raise SingularPivot(-1)
            beta = (rho1 / rho) * (alpha / omega)
            p = r + beta * (p - omega * v)
            phat = p / diag
            v = self._matvec(data, phat)
            denom = np.vdot(rhat, v)
            if denom == 0:
                raise SingularPivot(-1)
            alpha = rho1 / denom
            s = r - alpha * v
            if np.linalg.norm(s) <= self.tol * bnorm:
                return x + alpha * phat
            shat = s / diag
            t = self._matvec(data, shat)
            tt = np.vdot(t, t)
            if tt == 0:
                raise SingularPivot(-1)
            omega = np.vdot(t, s) / tt
            x = x + alpha * phat + omega * shat
            r = s - omega * t
            if np.linalg.norm(r) <= self.tol * bnorm:
                return x
            rho = rho1
        raise SingularPivot(-1)

    def _solve(self, op, rhs):
        data, diag = op
        rhs = np.asarray(rhs, dtype=np.complex128)
        out = np.empty_like(rhs)
        for k in range(rhs.shape[1]):
            out[:, k] = self._bicgstab(data, diag, rhs[:, k].copy())
        return out

    def solve(self, f, rhs):
        return self._solve(f[0], rhs)

    def solve_adjoint(self, f, rhs):
        return self._solve(f[1], rhs)


def oracle_feast_csr(a, emin, emax, m0, *, b=None, hermitian=False, solver="direct", iter_tol=1e-3,
                     fpm=None, seed=42):
    """feast_scsr / feast_hcsr (sparse.py:465-517) on full dense copies a, b of
    the expanded CSR matrices."""
    dt = np.complex128 if hermitian else np.float64
    a = np.asarray(a, dtype=dt)
    b = None if b is None else np.asarray(b, dtype=dt)
    ops = CsrDirectOps(a, b) if solver == "direct" else CsrIterativeOps(a, b, iter_tol)
    try:
        return oracle_feast(ops, a.shape[0], m0, emin, emax, hermitian=hermitian, fpm=fpm, seed=seed)
    except SingularPivot:        # _driver.py:88-91: inner-solver failure -> info -2
        n = a.shape[0]
        return OracleResult(np.zeros(m0), np.zeros((n, m0), dtype=dt), 0, np.zeros(m0), 1.0, 0, -2, m0)
