"""Partitioned (SPIKE) band LU / solve through the C ABI (fb_band_factor_batched,
fb_band_solve_batched) against dense numpy solves of the same shifted band
matrices z*B - A (banded.py:156-170), with the partition count forced up so
the interface system is exercised at small N.  P = 1 must reproduce the
reference's whole-band LU (banded.py:68-103) exactly as the sequential path."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    from paper_1203_4031_b200.device import get_device
    return get_device()


def _c(x):
    return ctypes.c_void_p(x)


def _band(n, kl, rng, cplx, spd=False):
    """Full-band layout (2kl+1, n): row kl+s holds the s-th subdiagonal."""
    fb = np.zeros((2 * kl + 1, n), dtype=np.complex128 if cplx else np.float64)
    for s in range(-kl, kl + 1):
        if s >= 0:
            v = rng.standard_normal(n - s) + (1j * rng.standard_normal(n - s) if cplx else 0)
            fb[kl + s, : n - s] = v
            fb[kl - s, s:] = np.conj(v) if cplx else v  # Hermitian / symmetric pattern
    if spd:
        fb *= 0.05
        fb[kl] = 1.0 + 0.0j if cplx else 1.0
    else:
        fb[kl] = fb[kl].real
    return fb


def _dense(fb, kl):
    n = fb.shape[1]
    a = np.zeros((n, n), dtype=fb.dtype)
    for s in range(-kl, kl + 1):
        for j in range(max(0, -s), min(n, n - s)):
            a[j + s, j] = fb[kl + s, j]
    return a


def _spike(dev, fa, fbm, kl, zs, rhs, part):
    torch = dev.torch
    n = fa.shape[1]
    cnt = len(zs)
    P = dev.lib.fb_debug_band_part_target(part, n, kl)
    try:
        cplx = np.iscomplexobj(fa)
        FA = dev.upload(fa, cplx=cplx)
        FB = None if fbm is None else dev.upload(fbm, cplx=cplx)
        auxd = int(dev.lib.fb_band_aux_doubles(n, kl))
        lw = (3 * kl + 1) * n
        fact = torch.empty((2, cnt, lw), dtype=torch.float64, device=dev.tdev)
        ipiv = torch.empty((cnt, n), dtype=torch.int32, device=dev.tdev)
        aux = torch.empty((cnt, auxd), dtype=torch.float64, device=dev.tdev)
        info = torch.empty(cnt, dtype=torch.int32, device=dev.tdev)
        zr = (ctypes.c_double * cnt)(*[z.real for z in zs])
        zi = (ctypes.c_double * cnt)(*[z.imag for z in zs])
        dev.check(dev.lib.fb_band_factor_batched(
            dev.h, cnt, n, kl, zr, zi, _c(FA.re), _c(FA.im) if FA.im else None,
            _c(FB.re) if FB else None, _c(FB.im) if (FB and FB.im) else None, FA.ld,
            _c(fact[0].data_ptr()), _c(fact[1].data_ptr()), lw, _c(ipiv.data_ptr()), n,
            _c(aux.data_ptr()), auxd, _c(info.data_ptr())), "band_factor_batched")
        bad = (ctypes.c_int * cnt)()
        dev.lib.fb_read_info_batched(dev.h, cnt, _c(info.data_ptr()), bad)
        assert list(bad) == [-1] * cnt
        m = rhs.shape[1]
        X = torch.empty((2, cnt, n, m), dtype=torch.float64, device=dev.tdev)
        X[0].copy_(torch.from_numpy(np.ascontiguousarray(rhs.real)).to(dev.tdev).expand(cnt, n, m))
        X[1].copy_(torch.from_numpy(np.ascontiguousarray(rhs.imag)).to(dev.tdev).expand(cnt, n, m))
        dev.check(dev.lib.fb_band_solve_batched(
            dev.h, cnt, n, kl, m, _c(fact[0].data_ptr()), _c(fact[1].data_ptr()), lw, _c(ipiv.data_ptr()), n,
            _c(aux.data_ptr()), auxd, _c(X[0].data_ptr()), _c(X[1].data_ptr()), m, n * m),
            "band_solve_batched")
        torch.cuda.synchronize()
        x = X[0].cpu().numpy() + 1j * X[1].cpu().numpy()
        return P, fact, ipiv, x
    finally:
        dev.lib.fb_debug_band_part_target(0, n, kl)


@pytest.mark.parametrize("n,kl,part,cplx,gen", [
    (300, 1, 40, False, False), (300, 3, 40, False, True), (1000, 5, 64, False, True),
    (1000, 16, 64, False, True), (777, 16, 100, True, True), (2000, 7, 128, True, False),
    (4096, 16, 256, False, True), (515, 2, 33, False, True),
])
def test_spike_solve_matches_dense(dev, n, kl, part, cplx, gen):
    rng = np.random.default_rng(n * 31 + kl)
    fa = _band(n, kl, rng, cplx) * 0.3
    fbm = _band(n, kl, rng, cplx, spd=True) if gen else None
    zs = [complex(0.1 * np.cos(t), 0.3 * np.sin(t) + 0.02) for t in (0.3, 1.2, 2.5)]
    rhs = rng.standard_normal((n, 37)) + 1j * rng.standard_normal((n, 37))
    P, _, _, x = _spike(dev, fa, fbm, kl, zs, rhs, part)
    assert P > 1
    A = _dense(fa, kl)
    B = np.eye(n) if fbm is None else _dense(fbm, kl)
    for i, z in enumerate(zs):
        S = z * B - A
        ref = np.linalg.solve(S, rhs)
        err = np.abs(x[i] - ref).max() / np.abs(ref).max()
        assert err <= 1e-11, (i, err)


@pytest.mark.parametrize("n,kl", [(130, 16), (40, 4)])
def test_spike_single_partition_is_reference_lu(dev, unit_golden, n, kl):
    """P = 1: the partitioned factor equals the reference band LU (same pivots,
    same working array) and the solve matches the reference solve."""
    g = unit_golden
    tag = f"{n}_{kl}"
    fbm = g[f"blu_fb_{tag}"]
    P, fact, ipiv, x = _spike(dev, -fbm, None, kl, [0j], g[f"blu_b_{tag}"], 10 ** 9)
    assert P == 1
    assert np.array_equal(ipiv[0].cpu().numpy(), g[f"blu_ipiv_{tag}"])
    lw = 3 * kl + 1
    ab = (fact[0, 0].cpu().numpy() + 1j * fact[1, 0].cpu().numpy()).reshape(n, lw).T
    ref = g[f"blu_ab_{tag}"]
    assert np.abs(ab - ref).max() <= 1e-12 * max(1, np.abs(ref).max())
    assert np.abs(x[0] - g[f"blu_x_{tag}"]).max() <= 1e-10 * max(1, np.abs(x[0]).max())


@pytest.mark.parametrize("n,kl,klb,part,herm,m", [
    (1500, 16, 1, 300, False, 96), (900, 5, 5, 128, False, 37), (777, 16, 16, 100, True, 50),
    (640, 3, 0, 10 ** 9, False, 20), (1200, 2, 2, 64, True, 7),
])
def test_fused_pass_matches_dense_quadrature(dev, n, kl, klb, part, herm, m):
    """fb_band_solve_accumulate (sweeps + interface + correction/accumulation
    kernel) through DeviceBandOps.solve_pass_accumulate: Q against the dense
    numpy evaluation of kernel.py:350-364 (solve every shift, accumulate with
    kernel.py:108-124), and against the unfused solve_pass + accumulate_terms."""
    from paper_1203_4031_b200.banded import DeviceBandOps, pad_band
    from paper_1203_4031_b200.quadrature import build_contour, gauss_legendre
    rng = np.random.default_rng(n + 7 * kl + (1 if herm else 0))
    fa = _band(n, kl, rng, herm) * 0.3
    fbm = pad_band(_band(n, klb, rng, herm, spd=True), klb, kl)
    ct = build_contour(gauss_legendre(8), -0.25, 0.2)
    zs = [complex(z) for z in ct.z]
    P = dev.lib.fb_debug_band_part_target(part, n, kl)
    try:
        assert (P > 1) == (part < n)
        FA, FB = dev.upload(fa, cplx=herm), dev.upload(fbm, cplx=herm)
        ops = DeviceBandOps(dev, FA, FB, kl, herm)
        ops.prefactorize(zs)
        y = rng.standard_normal((n, m)) + (1j * rng.standard_normal((n, m)) if herm else 0)
        Y = dev.upload(y, cplx=herm)
        spec = []
        for k, z in enumerate(zs):
            for adj in ((False, True) if herm else (False,)):
                spec.append((z, adj, (2 if adj else 1) if herm else 0, ct.weights[k], ct.theta[k]))
        Q = dev.zeros(n, m, herm)
        assert ops.solve_pass_accumulate(Y, spec, ct.radius, Q)
        q = dev.download(Q)
        # unfused path
        Q2 = dev.zeros(n, m, herm)
        ops.solve_pass(Y, herm)
        dev.accumulate_terms([(v, w, th, ops.pass_result(z, adj)) for z, adj, v, w, th in spec], ct.radius, Q2)
        q2 = dev.download(Q2)
    finally:
        dev.lib.fb_debug_band_part_target(0, n, kl)
    A, B = _dense(fa, kl), _dense(fbm, kl)
    ref = np.zeros_like(q)
    for z, adj, v, w, th in spec:
        S = z * B - A
        x = np.linalg.solve(S.conj().T if adj else S, y)
        if v == 0:
            ref -= (w / 2.0) * (ct.radius * np.exp(1j * th) * x).real
        else:
            ref -= ((w / 4.0) * ct.radius) * np.exp((1j if v == 1 else -1j) * th) * x
    scale = np.abs(ref).max()
    assert np.abs(q2 - ref).max() <= 1e-10 * scale
    assert np.abs(q - ref).max() <= 1e-10 * scale
    assert np.abs(q - q2).max() <= 1e-12 * scale
