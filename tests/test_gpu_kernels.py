"""Kernel-level parity of libfeastb200.so against the CPU oracle and the
reference's golden vectors.  Every call goes through the C ABI."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    from paper_1203_4031_b200.device import get_device
    return get_device()


def _c(x):
    return ctypes.c_void_p(x)


def test_splitmix_bitexact(dev, unit_golden):
    for key in unit_golden.files:
        if not key.startswith("rng_"):
            continue
        _, seed, off, cnt = key.split("_")
        cnt = int(cnt)
        out = dev.empty(cnt, 1, False)
        dev.splitmix(int(seed), int(off), 0, out)
        got = dev.download(out)[:, 0]
        assert got.tobytes() == unit_golden[key].tobytes(), key


@pytest.mark.parametrize("herm", [False, True])
def test_start_block_bitexact(dev, herm):
    from paper_1203_4031_b200.kernel import HermitianRci, SymmetricRci
    n, m0 = 37, 11
    cls = HermitianRci if herm else SymmetricRci
    k = cls(n, m0, -1.0, 1.0, seed=99, host_mirror=False)
    k._fill_random_y()
    got = dev.download(k.Y)
    ref = O.start_block(99, n, m0, herm)
    assert got.tobytes() == ref.astype(got.dtype).tobytes()


@pytest.mark.parametrize("variant", ["symmetric", "hermitian-direct", "hermitian-adjoint"])
def test_accumulate_matches_reference(dev, unit_golden, variant):
    g = unit_golden
    q0 = g["acc_q0"] if variant == "symmetric" else g["acc_qc0"]
    ref = {"symmetric": g["acc_sym"], "hermitian-direct": g["acc_hd"],
           "hermitian-adjoint": g["acc_ha"]}[variant]
    Q = dev.upload(q0, cplx=np.iscomplexobj(q0))
    X = dev.upload(g["acc_w2"], cplx=True)
    dev.accumulate({"symmetric": 0, "hermitian-direct": 1, "hermitian-adjoint": 2}[variant],
                   X, Q, 0.3, 1.7, 0.9)
    got = dev.download(Q)
    assert np.abs(got - ref).max() <= 4e-16 * np.abs(ref).max()


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("ops", ["NN", "CN", "NT", "TN", "NC"])
@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 5, 3), (64, 64, 64), (131, 70, 45), (40, 37, 3000)])
def test_gemm_vs_numpy(dev, cplx, ops, shape):
    rng = np.random.default_rng(hash((cplx, ops, shape)) % 2**32)
    m, n, k = shape

    def mk(r, c):
        x = rng.standard_normal((r, c))
        if cplx:
            x = x + 1j * rng.standard_normal((r, c))
        return x

    a = mk(m, k) if ops[0] == "N" else mk(k, m)
    b = mk(k, n) if ops[1] == "N" else mk(n, k)
    c0 = mk(m, n)
    alpha, beta = (1.5 - 0.5j, 0.25 + 1j) if cplx else (1.5, 0.25)

    def op(x, o):
        return x if o == "N" else (x.T if o == "T" else x.conj().T)

    ref = alpha * op(a, ops[0]) @ op(b, ops[1]) + beta * c0
    A, B, C = dev.upload(a, cplx=cplx), dev.upload(b, cplx=cplx), dev.upload(c0, cplx=cplx)
    dev.gemm(ops[0], ops[1], m, n, k, alpha, A, B, beta, C, cplx=cplx)
    got = dev.download(C)
    tol = 1e-13 * max(1.0, np.sqrt(k)) * (np.abs(a).max() * np.abs(b).max() * k + np.abs(c0).max())
    assert np.abs(got - ref).max() <= tol


def _lu(dev, a):
    n = a.shape[0]
    torch = dev.torch
    LU = dev.upload(a, cplx=True)
    piv = torch.empty(n, dtype=torch.int32, device=dev.tdev)
    dinv = torch.empty(int(dev.lib.fb_zgetrf_dinv_doubles(n)), dtype=torch.float64, device=dev.tdev)
    info = torch.empty(1, dtype=torch.int32, device=dev.tdev)
    dev.check(dev.lib.fb_zgetrf(dev.h, n, _c(LU.re), _c(LU.im), LU.ld, _c(piv.data_ptr()),
                                _c(dinv.data_ptr()), _c(info.data_ptr())), "zgetrf")
    bad = dev.read_info(info.data_ptr())
    return LU, piv, dinv, bad


def _solve(dev, n, LU, piv, dinv, b, adjoint):
    W = dev.upload(b, cplx=True)
    dev.check(dev.lib.fb_zgetrs(dev.h, n, W.cols, _c(LU.re), _c(LU.im), LU.ld, _c(piv.data_ptr()),
                                _c(dinv.data_ptr()), 1 if adjoint else 0, _c(W.re), _c(W.im), W.ld),
              "zgetrs")
    return dev.download(W)


@pytest.mark.parametrize("n", [1, 2, 5, 20, 64, 97])
def test_zgetrf_matches_reference_factor(dev, unit_golden, n):
    g = unit_golden
    LU, piv, dinv, bad = _lu(dev, g[f"lu_a_{n}"])
    assert bad == -1
    assert np.array_equal(piv.cpu().numpy(), g[f"lu_piv_{n}"])
    lu = dev.download(LU)
    assert np.abs(lu - g[f"lu_lu_{n}"]).max() <= 1e-12 * max(1, np.abs(lu).max())
    x = _solve(dev, n, LU, piv, dinv, g[f"lu_b_{n}"], False)
    xa = _solve(dev, n, LU, piv, dinv, g[f"lu_b_{n}"], True)
    assert np.abs(x - g[f"lu_x_{n}"]).max() <= 1e-10 * max(1, np.abs(x).max())
    assert np.abs(xa - g[f"lu_xa_{n}"]).max() <= 1e-10 * max(1, np.abs(xa).max())


@pytest.mark.parametrize("n", [31, 33, 127, 128, 129, 300, 1000, 2049])
def test_zgetrf_random_residual(dev, n):
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    LU, piv, dinv, bad = _lu(dev, a)
    assert bad == -1
    b = rng.standard_normal((n, 17)) + 1j * rng.standard_normal((n, 17))
    x = _solve(dev, n, LU, piv, dinv, b, False)
    xa = _solve(dev, n, LU, piv, dinv, b, True)
    scale = np.abs(a).max() * np.abs(x).max() * n
    assert np.abs(a @ x - b).max() <= 1e-13 * scale
    assert np.abs(a.conj().T @ xa - b).max() <= 1e-13 * np.abs(a).max() * np.abs(xa).max() * n
    if n <= 300:   # identical pivot sequence to the restated reference LU
        _, piv_ref = O.lu_factor_ref(a)
        assert np.array_equal(piv.cpu().numpy(), piv_ref)


def test_zgetrf_zero_pivot_reports_column(dev):
    a = np.zeros((40, 40), dtype=complex)
    a[np.arange(40), np.arange(40)] = 1.0
    a[17, 17] = 0.0
    _, _, _, bad = _lu(dev, a)
    assert bad == 17


@pytest.mark.parametrize("n", [2, 8, 7, 40, 33])
def test_reduced_eig_matches_reference(dev, unit_golden, n):
    g = unit_golden
    aq, bq = g[f"red_aq_{n}"], g[f"red_bq_{n}"]
    cplx = np.iscomplexobj(aq)
    A, B = dev.upload(aq, cplx=cplx), dev.upload(bq, cplx=cplx)
    PHI = dev.empty(n, n, cplx)
    eps = dev.torch.empty(n, dtype=dev.torch.float64, device=dev.tdev)
    st = dev.reduced_eig(A, B, n, eps.data_ptr(), PHI)
    assert st == 0
    e = eps.cpu().numpy()
    assert np.abs(e - g[f"red_eps_{n}"]).max() <= 1e-12 * max(1, np.abs(e).max())
    phi = dev.download(PHI)
    ref = g[f"red_phi_{n}"]
    for j in range(n):
        k = int(np.argmax(np.abs(ref[:, j])))
        ph = phi[k, j] / ref[k, j]
        assert abs(abs(ph) - 1) <= 1e-9
        assert np.abs(phi[:, j] - ph * ref[:, j]).max() <= 1e-9


def test_chol_check_failure_index(dev, unit_golden):
    g = unit_golden
    for name in ("neg2", "neg1", "sing"):
        mat = g[f"spd_{name}_in"]
        B = dev.upload(mat, cplx=False)
        fail = dev.chol_check(B, mat.shape[0])
        assert fail == int(g[f"spd_{name}_fail"])


def test_reduced_eig_reports_cholesky_pivot(dev, unit_golden):
    """The reduced solve's status is the same 1-based failing pivot as
    spd_factor (reduced.py:22-40); kernel.py's M0 shrink relies on it."""
    g = unit_golden
    for name in ("neg2", "neg1", "sing"):
        mat = g[f"spd_{name}_in"]
        n = mat.shape[0]
        A, B = dev.upload(np.eye(n), cplx=False), dev.upload(mat, cplx=False)
        PHI = dev.empty(n, n, False)
        eps = dev.torch.empty(n, dtype=dev.torch.float64, device=dev.tdev)
        assert dev.reduced_eig(A, B, n, eps.data_ptr(), PHI) == int(g[f"spd_{name}_fail"])


@pytest.mark.parametrize("cplx", [False, True])
def test_reduced_eig_nonfinite_is_solver_error(dev, cplx):
    rng = np.random.default_rng(11)
    n = 24
    a = rng.standard_normal((n, n))
    a = a + a.T
    a[3, 5] = a[5, 3] = np.nan
    b = np.eye(n)
    A, B = dev.upload(a, cplx=cplx), dev.upload(b, cplx=cplx)
    PHI = dev.empty(n, n, cplx)
    eps = dev.torch.empty(n, dtype=dev.torch.float64, device=dev.tdev)
    assert dev.reduced_eig(A, B, n, eps.data_ptr(), PHI) == -2


@pytest.mark.parametrize("n,cplx", [(1, False), (3, True), (64, False), (150, False), (152, True),
                                    (160, False), (256, True), (257, False), (300, True)])
def test_reduced_eig_sizes(dev, n, cplx):
    """Cluster path (M0 <= 256) and single-CTA path (larger) against LAPACK:
    eigenvalues, A Phi = B Phi diag(eps) and Phi^H B Phi = I."""
    import scipy.linalg as sla
    rng = np.random.default_rng(n)
    g = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)
    a = (g + g.conj().T) / 2
    h = rng.standard_normal((n, n)) + (1j * rng.standard_normal((n, n)) if cplx else 0)
    b = np.eye(n) + 0.1 * h @ h.conj().T / n
    A, B = dev.upload(a, cplx=cplx), dev.upload(b, cplx=cplx)
    PHI = dev.empty(n, n, cplx)
    eps = dev.torch.empty(n, dtype=dev.torch.float64, device=dev.tdev)
    assert dev.reduced_eig(A, B, n, eps.data_ptr(), PHI) == 0
    e = eps.cpu().numpy()
    ref = sla.eigh(a, b, eigvals_only=True)
    scale = max(1.0, np.abs(ref).max())
    assert np.abs(e - ref).max() <= 1e-12 * scale
    phi = dev.download(PHI)
    assert np.abs(a @ phi - b @ phi * e[None, :]).max() <= 1e-10 * scale
    assert np.abs(phi.conj().T @ b @ phi - np.eye(n)).max() <= 1e-10


def test_residuals_match_oracle(dev):
    rng = np.random.default_rng(5)
    n, m = 1500, 23
    ax = rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))
    bx = rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))
    bx[:, 4] = 0
    lam = rng.standard_normal(m)
    AX, BX = dev.upload(ax), dev.upload(bx)
    lt = dev.torch.tensor(lam, device=dev.tdev)
    rt = dev.torch.empty(m, dtype=dev.torch.float64, device=dev.tdev)
    dev.residuals(AX, BX, lt.data_ptr(), 0.7, rt.data_ptr())
    got = rt.cpu().numpy()
    ref = O.column_residuals(ax, bx, lam, 0.7)
    assert np.isinf(got[4]) and np.isinf(ref[4])
    ok = np.isfinite(ref)
    assert np.abs(got[ok] - ref[ok]).max() <= 1e-13 * np.abs(ref[ok]).max()


@pytest.mark.parametrize("cplx", [False, True])
def test_residual_sums_over_row_blocks(dev, cplx):
    """fb_residual_sums (multi-GPU row sharding): the per-block numerator /
    denominator sums add up to _column_residuals (kernel.py:147-153)."""
    rng = np.random.default_rng(55)
    n, m = 1100, 17
    ax = rng.standard_normal((n, m)) + (1j * rng.standard_normal((n, m)) if cplx else 0)
    bx = rng.standard_normal((n, m)) + (1j * rng.standard_normal((n, m)) if cplx else 0)
    lam = rng.standard_normal(m)
    AX, BX = dev.upload(ax, cplx=cplx), dev.upload(bx, cplx=cplx)
    lt = dev.torch.tensor(lam, device=dev.tdev)
    tot = np.zeros(2 * m)
    for r0, r1 in ((0, 367), (367, 733), (733, n)):
        st = dev.torch.empty(2 * m, dtype=dev.torch.float64, device=dev.tdev)
        dev.residual_sums(AX.rows_view(r0, r1), BX.rows_view(r0, r1), lt.data_ptr(), 0.7, st.data_ptr())
        tot += st.cpu().numpy()
    ref = O.column_residuals(ax, bx, lam, 0.7)
    got = tot[0::2] / tot[1::2]
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    assert np.allclose(tot[1::2], np.abs(0.7 * bx).sum(0), rtol=1e-13)


def test_symmetrize(dev):
    rng = np.random.default_rng(6)
    a = rng.standard_normal((19, 19)) + 1j * rng.standard_normal((19, 19))
    A = dev.upload(a)
    dev.symmetrize(A)
    assert dev.download(A).tobytes() == (0.5 * (a + a.conj().T)).tobytes()


def _band_call(dev, fb, kl, z, fbm=None):
    n = fb.shape[1]
    torch = dev.torch
    FA = dev.upload(fb, cplx=np.iscomplexobj(fb))
    FB = None if fbm is None else dev.upload(fbm, cplx=np.iscomplexobj(fbm))
    w = dev.empty(n, 3 * kl + 1, True)
    ipiv = torch.empty(n, dtype=torch.int32, device=dev.tdev)
    info = torch.empty(1, dtype=torch.int32, device=dev.tdev)
    dev.check(dev.lib.fb_band_factor(dev.h, n, kl, z.real, z.imag, _c(FA.re), _c(FA.im),
                                     _c(FB.re) if FB else None, _c(FB.im) if FB else None, FA.ld,
                                     _c(w.re), _c(w.im), _c(ipiv.data_ptr()), _c(info.data_ptr())),
              "band_factor")
    return w, ipiv, dev.read_info(info.data_ptr())


@pytest.mark.parametrize("n,kl", [(6, 1), (12, 3), (9, 0), (40, 4), (130, 16)])
def test_band_lu_matches_reference(dev, unit_golden, n, kl):
    g = unit_golden
    tag = f"{n}_{kl}"
    fb = g[f"blu_fb_{tag}"]
    # factorize z*I - (-fb) = fb  (shift with z = 0 of FA = -fb)
    w, ipiv, bad = _band_call(dev, -fb, kl, 0j)
    assert bad == -1
    assert np.array_equal(ipiv.cpu().numpy(), g[f"blu_ipiv_{tag}"])
    ab = dev.download(w).T              # column-major working array -> (3kl+1, n)
    ref = g[f"blu_ab_{tag}"]
    assert np.abs(ab - ref).max() <= 1e-12 * max(1, np.abs(ref).max())
    for adj, key in ((0, "blu_x"), (1, "blu_xa")):
        W = dev.upload(g[f"blu_b_{tag}"], cplx=True)
        dev.check(dev.lib.fb_band_solve(dev.h, n, kl, W.cols, _c(w.re), _c(w.im), _c(ipiv.data_ptr()),
                                        adj, _c(W.re), _c(W.im), W.ld), "band_solve")
        x = dev.download(W)
        assert np.abs(x - g[f"{key}_{tag}"]).max() <= 1e-10 * max(1, np.abs(x).max())


@pytest.mark.parametrize("n,kl", [(6, 1), (12, 3), (40, 4), (130, 16)])
def test_band_matvec(dev, unit_golden, n, kl):
    g = unit_golden
    tag = f"{n}_{kl}"
    fb = g[f"blu_fb_{tag}"]
    x = g[f"bmv_x_{tag}"]
    FB = dev.upload(fb)
    X = dev.upload(x, cplx=True)
    Y = dev.empty(n, x.shape[1], True)
    dev.check(dev.lib.fb_band_matvec(dev.h, n, kl, x.shape[1], _c(FB.re), _c(FB.im), FB.ld, _c(X.re),
                                     _c(X.im), X.ld, _c(Y.re), _c(Y.im), Y.ld), "band_matvec")
    assert np.abs(dev.download(Y) - g[f"bmv_y_{tag}"]).max() <= 1e-13 * n


@pytest.mark.parametrize("uplo", ["F", "L", "U"])
@pytest.mark.parametrize("herm", [False, True])
@pytest.mark.parametrize("kl,kl_to", [(1, 1), (3, 3), (1, 4), (4, 6)])
def test_expand_band_device_bitexact(dev, uplo, herm, kl, kl_to):
    """Device band expansion == host expand_band + pad_band bit for bit, with
    the out-of-pattern slots of the LAPACK band poisoned by NaN (never read,
    banded.py:21-47; test_banded.py:145-164)."""
    from paper_1203_4031_b200.banded import band_required_rows, expand_band, expand_band_device, pad_band
    rng = np.random.default_rng(kl * 10 + kl_to + (7 if herm else 0))
    n = 23
    rows = band_required_rows(kl, uplo)
    ab = rng.standard_normal((rows, n)) + (1j * rng.standard_normal((rows, n)) if herm else 0)
    for d in range(1, kl + 1):   # poison the slots outside the band pattern
        if uplo == "F":
            ab[kl - d, :d] = np.nan
            ab[kl + d, n - d:] = np.nan
        elif uplo == "L":
            ab[d, n - d:] = np.nan
        else:
            ab[kl - d, :d] = np.nan
    want = pad_band(expand_band(ab, kl, uplo, herm), kl, kl_to)
    got = expand_band_device(dev, ab, kl, uplo, herm, kl_to)
    g = got.plane(0).cpu().numpy() + (1j * got.plane(1).cpu().numpy() if herm else 0)
    assert np.array_equal(g, want)


@pytest.mark.parametrize("n,count", [(1792, 4), (1100, 8)])
def test_batched_lu_tma_trailing_update_with_lookahead(dev, n, count):
    """Batched shifted LU large enough for the TMA-fed trailing update to run
    concurrently with the look-ahead panels of the next block (gemm_tma.cu):
    every shift's solve against numpy.  (The swizzled tiles must be aligned at
    run time: a CTA's dynamic shared memory is not 1024-byte aligned when the
    SM is shared with other kernels' CTAs -- n = 1792 x 4 shifts caught it.)"""
    from paper_1203_4031_b200.dense import DeviceDenseOps
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    a = (a + a.conj().T) / 2
    ops = DeviceDenseOps(dev, dev.upload(a, cplx=True), None, True)
    zs = [complex(0.3 * k, 0.5 + 0.1 * k) for k in range(count)]
    ops.prefactorize(zs)
    y = rng.standard_normal((n, 12)) + 1j * rng.standard_normal((n, 12))
    ops.solve_pass(dev.upload(y, cplx=True), False)
    for z in zs:
        x = dev.download(ops.pass_result(z, False))
        s = z * np.eye(n) - a
        assert np.abs(s @ x - y).max() <= 1e-13 * np.abs(s).max() * np.abs(x).max() * n


@pytest.mark.parametrize("n,count,nrhs", [(6144, 2, 160), (6300, 1, 152), (6144, 1, 24)])
def test_blocked_sweeps_large_n(dev, n, count, nrhs):
    """Sweeps at n >= 6144 run blocked (trsm.cu: a single-CTA solve of each
    256-row diagonal block + one TMA-fed ZGEMM over the pending rows, M^H tiles
    for the adjoint sweeps): (zB - A) x = y and (zB - A)^H x = y against numpy,
    ragged n, column counts that are not a tile multiple (the 32-column tail
    form of the update kernel, alone for 24 columns) included.  Repeated
    passes must be bit-identical: before the stage release of the TMA kernel was
    ordered after the fragment loads' completion (gemm_tma.cu), about one pass
    in three of the (6144, 2, 160) case returned a wrong 16-column sub-tile."""
    from paper_1203_4031_b200.dense import DeviceDenseOps
    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    a = (a + a.conj().T) / 2
    ops = DeviceDenseOps(dev, dev.upload(a, cplx=True), None, True)
    zs = [complex(0.3 * k, 0.5 + 0.1 * k) for k in range(count)]
    ops.prefactorize(zs)
    y = rng.standard_normal((n, nrhs)) + 1j * rng.standard_normal((n, nrhs))
    Y = dev.upload(y, cplx=True)
    ops.solve_pass(Y, True)
    first = {(z, adj): dev.download(ops.pass_result(z, adj)).copy() for z in zs for adj in (False, True)}
    for (z, adj), x in first.items():
        s = z * np.eye(n) - a
        if adj:
            s = s.conj().T
        assert np.abs(s @ x - y).max() <= 1e-13 * np.abs(s).max() * np.abs(x).max() * n
    for _ in range(4):
        ops.solve_pass(Y, True)
        for (z, adj), x in first.items():
            assert np.array_equal(dev.download(ops.pass_result(z, adj)), x)
