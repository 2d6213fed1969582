"""Place the frozen search intervals of workloads.py (run once in the build
container; prints the constants).  Dense: scipy eigh; band: Sylvester inertia."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.linalg as sla
from paper_1203_4031_b200 import workloads as W
from oracle.inertia import count_below


def midgap_nearest(ev, k, center=0.0):
    ev = np.sort(ev)
    i0 = int(np.searchsorted(ev, center))
    lo = max(i0 - k // 2, 1)
    hi = lo + k - 1
    return 0.5 * (ev[lo - 1] + ev[lo]), 0.5 * (ev[hi] + ev[hi + 1]), k


def band_eig_k(ab, bb, k, lo=-50.0, hi=50.0):
    """k-th smallest eigenvalue (0-based) by bisection on the inertia count."""
    for _ in range(100):
        mid = 0.5 * (lo + hi)
        if count_below(ab, bb, mid) > k:
            hi = mid
        else:
            lo = mid
        if hi - lo < 1e-13 * max(1.0, abs(mid)):
            break
    return 0.5 * (lo + hi)


def band_interval(n, kd, seed, k=64):
    ab, bb = W.c4_band_matrices(n, kd, seed)
    i0 = count_below(ab, bb, 0.0)
    lo = i0 - k // 2
    hi = lo + k - 1
    a = band_eig_k(ab, bb, lo - 1, -1.0, 1.0); b = band_eig_k(ab, bb, lo, -1.0, 1.0)
    c = band_eig_k(ab, bb, hi, -1.0, 1.0); d = band_eig_k(ab, bb, hi + 1, -1.0, 1.0)
    emin, emax = 0.5 * (a + b), 0.5 * (c + d)
    m = count_below(ab, bb, emax) - count_below(ab, bb, emin)
    return (emin, emax), m, (b - a, d - c)


out = {}
which = sys.argv[1:] or ["scaled", "c1", "c2", "c3", "c4"]
if "scaled" in which:
    w = W.c1_syev(n=400, m0=40, seed=11, interval=(-1, 1))
    out["c1s"] = midgap_nearest(np.linalg.eigvalsh(w.a), 20)
    w = W.c2_sygv(n=512, m0=40, seed=12, interval=(-1, 1))
    out["c2s"] = midgap_nearest(sla.eigh(w.a, w.b, eigvals_only=True), 20)
    w = W.c3_heev(n=384, m0=40, seed=13, interval=(-1, 1))
    out["c3s"] = midgap_nearest(np.linalg.eigvalsh(w.a), 20)
    w = W.c5_hegv(n=320, m0=48, seed=15, interval=(-1, 1))
    out["c5s"] = midgap_nearest(sla.eigh(w.a, w.b, eigvals_only=True), 24)
    iv, m, gaps = band_interval(20000, 16, 14)
    out["c4s"] = (iv[0], iv[1], m)
    print("gaps c4s", gaps)
if "c1" in which:
    w = W.c1_syev(interval=(-1, 1))
    ev = np.linalg.eigvalsh(w.a)
    out["c1"] = (-0.05, 0.05, int(((ev >= -0.05) & (ev <= 0.05)).sum()),
                 float(np.min(np.abs(np.abs(ev) - 0.05))))
if "c2" in which:
    w = W.c2_sygv(interval=(-1, 1))
    out["c2"] = midgap_nearest(sla.eigh(w.a, w.b, eigvals_only=True), 100)
if "c3" in which:
    w = W.c3_heev(interval=(-1, 1))
    ev = np.linalg.eigvalsh(w.a)
    out["c3"] = (-0.02, 0.02, int(((ev >= -0.02) & (ev <= 0.02)).sum()),
                 float(np.min(np.abs(np.abs(ev) - 0.02))))
if "c4" in which:
    iv, m, gaps = band_interval(1_000_000, 16, 4)
    out["c4"] = (iv[0], iv[1], m)
    print("gaps c4", gaps)
for k, v in out.items():
    print(k, repr(tuple(float(x) if not isinstance(x, int) else x for x in v)))


def band_interval_wide(n, kd, seed, k=64, search=5):
    """Like band_interval but moves each endpoint to the widest nearby gap."""
    ab, bb = W.c4_band_matrices(n, kd, seed)
    i0 = count_below(ab, bb, 0.0)
    lo0 = i0 - k // 2
    hi0 = lo0 + k - 1
    ev = {}
    def lam(i):
        if i not in ev:
            ev[i] = band_eig_k(ab, bb, i, -1.0, 1.0)
        return ev[i]
    best_lo = max(range(lo0 - search, lo0 + search + 1), key=lambda i: lam(i) - lam(i - 1))
    best_hi = max(range(hi0 - search, hi0 + search + 1), key=lambda i: lam(i + 1) - lam(i))
    emin = 0.5 * (lam(best_lo - 1) + lam(best_lo))
    emax = 0.5 * (lam(best_hi) + lam(best_hi + 1))
    m = count_below(ab, bb, emax) - count_below(ab, bb, emin)
    spacing = (lam(hi0) - lam(lo0)) / (k - 1)
    return (emin, emax), m, ((lam(best_lo) - lam(best_lo - 1)) / spacing,
                             (lam(best_hi + 1) - lam(best_hi)) / spacing)


if "wide" in which:
    for tag, n, seed in (("c4s", 20000, 14), ("c4", 1_000_000, 4)):
        iv, m, gaps = band_interval_wide(n, 16, seed)
        print(tag, repr((float(iv[0]), float(iv[1]), m)), "gap/spacing", gaps, flush=True)
