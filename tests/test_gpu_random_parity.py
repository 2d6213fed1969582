"""Randomised parity sweep: seeded dense and banded pencils of assorted sizes,
intervals placed mid-gap, GPU drivers vs the CPU oracle (reference kernel
restated + LAPACK caller).  Bar (BASELINE north_star): same m, eigenvalues
within 1e-10 * max(|Emin|, |Emax|), every residual <= 1e-10, loop within +-1."""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def _interval(ev, lo_idx, count):
    return 0.5 * (ev[lo_idx - 1] + ev[lo_idx]), 0.5 * (ev[lo_idx + count - 1] + ev[lo_idx + count])


def _check(r, o, emin, emax):
    s = max(abs(emin), abs(emax))
    assert r.info == o.info, (r.info, o.info)   # incl. both running out of loops (info 2)
    assert r.m == o.m
    assert abs(r.loop - o.loop) <= 1, (r.loop, o.loop)
    if o.info == 0:
        assert np.abs(np.sort(r.e[:r.m]) - np.sort(o.e[:o.m])).max() <= 1e-10 * s
        assert r.res[:r.m].max() <= 1e-10


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("kind", ["sy", "sygv", "he", "hegv"])
def test_dense_random_pencils(seed, kind):
    import paper_1203_4031_b200 as fb
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(60, 420))
    herm = kind.startswith("he")
    g = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if herm else 0)
    a = (g + g.conj().T) / (2 * np.sqrt(n))
    b = None
    if kind.endswith("gv"):
        h = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if herm else 0)
        b = np.eye(n) + 0.1 * (h @ h.conj().T) / n
    ev = np.sort(np.linalg.eigvals(a if b is None else np.linalg.solve(b, a)).real)
    count = int(rng.integers(4, 24))
    lo = int(rng.integers(1, n - count - 1))
    emin, emax = _interval(ev, lo, count)
    m0 = int(1.6 * count) + 4
    r = (fb.feast_he if herm else fb.feast_sy)(a, emin, emax, m0, b=b)
    o = (O.oracle_feast_he if herm else O.oracle_feast_sy)(a, emin, emax, m0, b=b)
    _check(r, o, emin, emax)
    if o.info == 0:
        assert r.m == count


@pytest.mark.parametrize("seed", range(4))
def test_banded_random_pencils(seed):
    import paper_1203_4031_b200 as fb
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(300, 1500))
    kd = int(rng.integers(1, 9))
    ab = np.zeros((kd + 1, n))
    ab[0] = rng.standard_normal(n) + 4.0 * (np.arange(n) / n - 0.5)
    for d in range(1, kd + 1):
        ab[d, :n - d] = rng.standard_normal(n - d)
    bb = np.zeros((2, n))
    bb[0] = 4.0 / 6.0
    bb[1, :n - 1] = 1.0 / 6.0
    full_a = O.expand_band(ab, kd, "L", False)
    full_b = O.expand_band(bb, 1, "L", False)
    A = np.zeros((n, n))
    B = np.zeros((n, n))
    for s_ in range(-kd, kd + 1):
        j0, j1 = max(0, -s_), min(n, n - s_)
        A[np.arange(j0, j1) + s_, np.arange(j0, j1)] = full_a[kd + s_, j0:j1]
    for s_ in (-1, 0, 1):
        j0, j1 = max(0, -s_), min(n, n - s_)
        B[np.arange(j0, j1) + s_, np.arange(j0, j1)] = full_b[1 + s_, j0:j1]
    ev = np.sort(np.linalg.eigvals(np.linalg.solve(B, A)).real)
    count = int(rng.integers(4, 16))
    lo = int(np.searchsorted(ev, 0.0)) - count // 2
    emin, emax = _interval(ev, lo, count)
    m0 = int(1.6 * count) + 4
    r = fb.feast_sb(ab, kd, emin, emax, m0, b=bb, klb=1, uplo="L")
    o = O.oracle_feast_sb(ab, kd, emin, emax, m0, b=bb, klb=1, uplo="L")
    assert r.m == count
    _check(r, o, emin, emax)
