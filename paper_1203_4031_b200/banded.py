"""Banded drivers feast_sb / feast_hb on the GPU (mirrors banded.py:1-258).

LAPACK-style band storage is normalised on the host exactly as the reference
does (expand_band / _pad_band, banded.py:21-47, 181-187) and uploaded once;
the shifted band LU, the band solves and the band multiplies run on the
device through libfeastb200.so.
"""

from __future__ import annotations

import ctypes

import threading

import numpy as np

from . import _lib
from ._driver import SolverOptions, run_rci
from ._errors import SingularMatrixError
from .device import Planar, get_device
from .kernel import HermitianRci, SymmetricRci
from .params import feastinit, FeastParams


def _is_torch(x):
    return type(x).__module__.startswith("torch")

_UPLOS = ("F", "L", "U")


def band_required_rows(kl: int, uplo: str) -> int:
    """banded.py:16-18."""
    return 2 * kl + 1 if uplo.upper() == "F" else kl + 1


def expand_band(ab, kl: int, uplo: str, hermitian: bool) -> np.ndarray:
    """Full-band layout: row kl+s holds the s-th subdiagonal, A[j+s, j] at
    [kl+s, j]; only in-pattern slots of ``ab`` are read (banded.py:21-47)."""
    ab = np.asarray(ab)
    n = ab.shape[1]
    uplo = uplo.upper()
    out = np.zeros((2 * kl + 1, n), dtype=ab.dtype)
    if uplo == "F":
        out[kl] = ab[kl]
        for d in range(1, kl + 1):
            out[kl - d, d:] = ab[kl - d, d:]
            out[kl + d, :n - d] = ab[kl + d, :n - d]
        return out
    if uplo == "L":
        out[kl] = ab[0]
        for d in range(1, kl + 1):
            low = ab[d, :n - d]
            out[kl + d, :n - d] = low
            out[kl - d, d:] = np.conj(low) if hermitian else low
        return out
    out[kl] = ab[kl]
    for d in range(1, kl + 1):
        up = ab[kl - d, d:]
        out[kl - d, d:] = up
        out[kl + d, :n - d] = np.conj(up) if hermitian else up
    return out


def expand_band_device(dev, ab, kl: int, uplo: str, hermitian: bool, kl_to: int) -> Planar:
    """expand_band + pad_band on the device: only the in-pattern rows of the
    LAPACK band ``ab`` cross PCIe (kl+1 rows for 'L'/'U'), the full-band
    (2*kl_to+1) x n layout is assembled by device copies (the mirrored
    triangle conjugated for Hermitian input) -- the same values as the host
    functions, bit for bit (banded.py:21-47, 181-187)."""
    torch = dev.torch
    on_dev = isinstance(ab, torch.Tensor)   # a band array already resident on the device
    if not on_dev:
        ab = np.asarray(ab)
    n = ab.shape[1]
    uplo = uplo.upper()
    off = kl_to - kl
    out = dev.zeros(2 * kl_to + 1, n, hermitian)
    planes = [out.plane(0)] + ([out.plane(1)] if hermitian else [])
    # LAPACK band rows: 'F' 2kl+1 rows (diagonal in row kl); 'L' diagonal in
    # row 0, subdiagonals below; 'U' superdiagonals above the diagonal in row kl
    rows = list(range(2 * kl + 1)) if uplo == "F" else list(range(kl + 1))
    if on_dev:
        st = ab[rows[0]:rows[-1] + 1].to(dev.tdev)
        if hermitian:
            st = st.to(torch.complex128)
            sp = [st.real, st.imag]
        else:
            sp = [(st.real if st.is_complex() else st).to(torch.float64)]
    elif hermitian:
        src = np.ascontiguousarray(ab[rows[0]:rows[-1] + 1])
        st = torch.from_numpy(src.astype(np.complex128, copy=False)).to(dev.tdev)
        sp = [st.real, st.imag]
    else:
        src = np.ascontiguousarray(ab[rows[0]:rows[-1] + 1])
        st = torch.from_numpy(np.ascontiguousarray(src.real if np.iscomplexobj(src) else src,
                                                   dtype=np.float64)).to(dev.tdev)
        sp = [st]
    r0 = rows[0]

    def row(k, p):
        return sp[p][k - r0]

    for p, P in enumerate(planes):
        sign = -1.0 if (hermitian and p == 1) else 1.0
        if uplo == "F":
            P[off + kl].copy_(row(kl, p))
            for d in range(1, kl + 1):
                P[off + kl - d, d:].copy_(row(kl - d, p)[d:])
                P[off + kl + d, :n - d].copy_(row(kl + d, p)[:n - d])
        elif uplo == "L":
            P[off + kl].copy_(row(0, p))
            for d in range(1, kl + 1):
                low = row(d, p)[:n - d]
                P[off + kl + d, :n - d].copy_(low)
                P[off + kl - d, d:].copy_(low if sign > 0 else -low)
        else:
            P[off + kl].copy_(row(kl, p))
            for d in range(1, kl + 1):
                up = row(kl - d, p)[d:]
                P[off + kl - d, d:].copy_(up)
                P[off + kl + d, :n - d].copy_(up if sign > 0 else -up)
    return out


def pad_band(fb, kl_from: int, kl_to: int):
    if kl_from == kl_to:
        return fb
    out = np.zeros((2 * kl_to + 1, fb.shape[1]), dtype=fb.dtype)
    out[kl_to - kl_from:kl_to + kl_from + 1] = fb
    return out


class _BandFactor:
    """A factored shift.  Sequential path: (w, ipiv) own arrays.  Partitioned
    path: (batch, idx) into a _BandBatch; ``adj`` is the factor of conj(z)
    that serves A^H solves of Hermitian pencils (S(z)^H = S(conj z))."""

    __slots__ = ("z", "w", "ipiv", "info", "batch", "idx", "adj")

    def __init__(self, z, w=None, ipiv=None, info=None, batch=None, idx=0, adj=None):
        self.z, self.w, self.ipiv, self.info = z, w, ipiv, info
        self.batch, self.idx, self.adj = batch, idx, adj


class _BandBatch:
    """count partitioned (SPIKE) factors: fact (2, count, (3kl+1) n),
    ipiv (count, n), aux (count, fb_band_aux_doubles(n, kl)), info (count)."""

    def __init__(self, dev, n, kl, count):
        t = dev.torch
        self.count, self.n, self.kl = count, n, kl
        self.lw = (3 * kl + 1) * n
        self.auxd = int(dev.lib.fb_band_aux_doubles(n, kl))
        self.fact = t.empty((2, count, self.lw), dtype=t.float64, device=dev.tdev)
        self.ipiv = t.empty((count, max(n, 1)), dtype=t.int32, device=dev.tdev)
        self.aux = t.empty((count, self.auxd), dtype=t.float64, device=dev.tdev)
        self.info = t.empty(count, dtype=t.int32, device=dev.tdev)
        self.zs = [None] * count

    def args(self, i0=0):
        return (self.fact[0, i0].data_ptr(), self.fact[1, i0].data_ptr(), self.lw,
                self.ipiv[i0].data_ptr(), self.ipiv.shape[1], self.aux[i0].data_ptr(), self.auxd)

    @staticmethod
    def nbytes(dev, n, kl, count):
        return count * (8 * (2 * (3 * kl + 1) * n + int(dev.lib.fb_band_aux_doubles(n, kl))) + 4 * n)


class DeviceBandOps:
    """Device backend for the banded drivers (banded.py:149-178).

    For 1 <= kl <= 16 the shifts are factored together by the partitioned
    band LU (fb_band_factor_batched) and each contour pass solves every
    resident shift in one batched call (fb_band_solve_batched); larger
    bandwidths use the sequential per-shift kernels."""

    on_device = True
    # bench.py instrumentation: when a list, (start, end, count) CUDA events recorded
    # on the context stream around every batched factorization are appended to it.
    factor_event_sink = None

    def __init__(self, dev, FA: Planar, FB: Planar | None, kl: int, hermitian: bool, cache_bytes=None,
                 mv_a=None, mv_b=None):
        self.dev, self.FA, self.FB, self.kl, self.hermitian = dev, FA, FB, kl, hermitian
        # (band, kl) the matvecs stream: a matrix narrower than the common
        # factorization bandwidth kl = max(kla, klb) keeps its own compact copy
        # (the C4 mass matrix has 3 diagonals, its padded copy 33)
        self._mv_a = mv_a or (FA, kl)
        self._mv_b = mv_b or (FB, kl)
        self.n = FA.cols
        self.factorizations = 0
        self.partitioned = int(dev.lib.fb_band_aux_doubles(self.n, kl)) > 0 if self.n > 0 else False
        if cache_bytes is None:
            free, _ = dev.torch.cuda.mem_get_info(dev.tdev)
            cache_bytes = int(0.85 * free)
        self.cache_left = cache_bytes
        self._batches = []
        self._pass = {}
        self._xbuf = {}
        self._zmap = {}          # z -> (batch, idx) of every factored shift

    # -- factorization ---------------------------------------------------------------
    def _factor_batch(self, bb, zs):
        dev, n, kl = self.dev, self.n, self.kl
        cnt = len(zs)
        zr = (ctypes.c_double * cnt)(*[z.real for z in zs])
        zi = (ctypes.c_double * cnt)(*[z.imag for z in zs])
        FA, FB = self.FA, self.FB
        fr, fi, fs, piv, ps, aux, as_ = bb.args()
        sink = DeviceBandOps.factor_event_sink
        if sink is not None:
            ev = (dev.torch.cuda.Event(enable_timing=True), dev.torch.cuda.Event(enable_timing=True))
            ev[0].record()
        dev.check(dev.lib.fb_band_factor_batched(
            dev.h, cnt, n, kl, zr, zi, FA.re, FA.im, FB.re if FB is not None else None,
            FB.im if FB is not None else None, FA.ld, fr, fi, fs, piv, ps, aux, as_,
            bb.info.data_ptr()), "band_factor_batched")
        if sink is not None:
            ev[1].record()
            sink.append((ev[0], ev[1], cnt))
        self.factorizations += cnt
        bad = (ctypes.c_int * cnt)()
        rc = dev.lib.fb_read_info_batched(dev.h, cnt, bb.info.data_ptr(), bad)
        if rc not in (0, _lib.FB_ERR_SINGULAR):
            dev.check(rc, "read_info")
        for i, z in enumerate(zs):
            if bad[i] >= 0:
                raise SingularMatrixError(f"zero pivot at band column {bad[i]} (shift {z})")
            bb.zs[i] = z

    def prefactorize(self, zs):
        """All shifts (and conj shifts for Hermitian pencils) in batched calls."""
        zs = [complex(z) for z in zs]
        if not self.partitioned:
            return {z: self.factorize(z) for z in zs}
        want = list(zs)
        if self.hermitian:
            want += [z.conjugate() for z in zs]
        per = _BandBatch.nbytes(self.dev, self.n, self.kl, 1)
        if per * len(want) > self.cache_left:
            raise MemoryError("band factors exceed the device cache")
        self.cache_left -= per * len(want)
        made = {}
        for c0 in range(0, len(want), 64):
            chunk = want[c0:c0 + 64]
            bb = _BandBatch(self.dev, self.n, self.kl, len(chunk))
            self._factor_batch(bb, chunk)
            self._batches.append(bb)
            for i, z in enumerate(chunk):
                made.setdefault(z, (bb, i))
                self._zmap.setdefault(z, (bb, i))
        out = {}
        for z in zs:
            bb, i = made[z]
            adj = None
            if self.hermitian:
                ab, ai = made[z.conjugate()]
                adj = _BandFactor(z.conjugate(), batch=ab, idx=ai)
            out[z] = _BandFactor(z, batch=bb, idx=i, adj=adj)
        return out

    def factorize(self, z):
        z = complex(z)
        if self.partitioned:
            return self.prefactorize([z])[z]
        dev, n, kl, torch = self.dev, self.n, self.kl, self.dev.torch
        w = dev.empty(n, 3 * kl + 1, True)     # column-major band working array
        ipiv = torch.empty(max(n, 1), dtype=torch.int32, device=dev.tdev)
        info = torch.empty(1, dtype=torch.int32, device=dev.tdev)
        FA, FB = self.FA, self.FB
        dev.check(dev.lib.fb_band_factor(dev.h, n, kl, z.real, z.imag, FA.re, FA.im,
                                         FB.re if FB is not None else None,
                                         FB.im if FB is not None else None, FA.ld,
                                         w.re, w.im, ipiv.data_ptr(), info.data_ptr()), "band_factor")
        self.factorizations += 1
        bad = dev.read_info(info.data_ptr())
        if bad >= 0:
            raise SingularMatrixError(f"zero pivot at band column {bad}")
        return _BandFactor(z, w, ipiv, info)

    # -- solves ----------------------------------------------------------------------
    def solve_pass(self, Y: Planar, hermitian: bool):
        """Every resident shift solved against this pass's Y in one call per batch
        (A^H solves of Hermitian pencils are the direct solves of conj(z))."""
        self._pass = {}
        if not self.partitioned:
            return
        dev, n, m = self.dev, self.n, Y.cols
        for bb in self._batches:
            cnt = bb.count
            X, mp = self._xwork(bb, m)
            fr, fi, fs, piv, ps, aux, as_ = bb.args()
            # every shift reads the pass's Y directly (stride 0, real or planar)
            dev.check(dev.lib.fb_band_solve_batched_rhs(dev.h, cnt, n, self.kl, m, fr, fi, fs, piv, ps, aux, as_,
                                                        Y.re, Y.im, Y.ld, 0, X[0].data_ptr(), X[1].data_ptr(),
                                                        mp, n * mp),
                      "band_solve_batched_rhs")
            for i in range(cnt):
                self._pass[(id(bb), i)] = (X, i, m)

    def _xwork(self, bb, m):
        mp = m + (m & 1)   # even leading dimension: 16-byte rows
        X = self._xbuf.get(id(bb))
        if X is None or X.shape[3] != mp:
            X = self.dev.torch.empty((2, bb.count, self.n, mp), dtype=self.dev.torch.float64, device=self.dev.tdev)
            self._xbuf[id(bb)] = X
        return X, mp

    def solve_pass_accumulate(self, Y: Planar, spec, radius, Q: Planar):
        """The whole contour pass in one call (fb_band_solve_accumulate): every
        shift of ``spec`` = [(z, adjoint, variant, w, theta)] solved against Y
        and its quadrature term folded into Q in that order, the spike
        correction applied inside the accumulation kernel.  Returns False
        (nothing done) unless all of the pass's shifts sit in one factor batch."""
        self._pass = {}
        if not self.partitioned or not spec or len(spec) > 64:
            return False
        hits = [self._zmap.get(complex(z).conjugate() if adj else complex(z)) for z, adj, *_ in spec]
        if any(h is None for h in hits) or any(h[0] is not hits[0][0] for h in hits):
            return False
        bb = hits[0][0]
        dev, n, m, k = self.dev, self.n, Y.cols, len(spec)
        X, mp = self._xwork(bb, m)
        fr, fi, fs, piv, ps, aux, as_ = bb.args()
        item = (ctypes.c_int * k)(*[h[1] for h in hits])
        var = (ctypes.c_int * k)(*[int(t[2]) for t in spec])
        w = (ctypes.c_double * k)(*[float(t[3]) for t in spec])
        th = (ctypes.c_double * k)(*[float(t[4]) for t in spec])
        dev.check(dev.lib.fb_band_solve_accumulate(
            dev.h, bb.count, n, self.kl, m, fr, fi, fs, piv, ps, aux, as_, Y.re, Y.im, Y.ld,
            X[0].data_ptr(), X[1].data_ptr(), mp, n * mp, k, item, var, w, float(radius), th,
            Q.re, Q.im, Q.ld), "band_solve_accumulate")
        return True

    def pass_result(self, z, adjoint):
        """Planar view of this pass's solve for shift z (A^H: the conj(z) factor)."""
        z = complex(z)
        hit = self._zmap.get(z.conjugate() if adjoint else z)
        if hit is None:
            return None
        got = self._pass.get((id(hit[0]), hit[1]))
        if got is None:
            return None
        X, i, m = got
        return Planar(X[:, i], True, X.shape[2], m, X.shape[3])

    def _solve_batched(self, f, W: Planar):
        hit = self._pass.get((id(f.batch), f.idx))
        if hit is not None:
            X, i, _ = hit
            W.plane(0).copy_(X[0, i][:, :W.cols])
            W.plane(1).copy_(X[1, i][:, :W.cols])
            return
        dev = self.dev
        fr, fi, fs, piv, ps, aux, as_ = f.batch.args(f.idx)
        dev.check(dev.lib.fb_band_solve_batched(dev.h, 1, self.n, self.kl, W.cols, fr, fi, fs, piv, ps, aux, as_,
                                                W.re, W.im, W.ld, 0), "band_solve_batched")

    def _solve(self, f, W: Planar, adjoint):
        if f.batch is not None:
            if adjoint:
                if f.adj is None:
                    raise AssertionError("adjoint band solve needs the conj(z) factor")
                self._solve_batched(f.adj, W)
            else:
                self._solve_batched(f, W)
            return
        dev = self.dev
        dev.check(dev.lib.fb_band_solve(dev.h, self.n, self.kl, W.cols, f.w.re, f.w.im,
                                        f.ipiv.data_ptr(), 1 if adjoint else 0, W.re, W.im, W.ld),
                  "band_solve")

    def solve(self, f, W):
        self._solve(f, W, False)

    def solve_adjoint(self, f, W):
        self._solve(f, W, True)

    def _mult(self, mv, X, Y):
        dev, (F, kl) = self.dev, mv
        dev.check(dev.lib.fb_band_matvec(dev.h, self.n, kl, X.cols, F.re, F.im, F.ld,
                                         X.re, X.im, X.ld, Y.re, Y.im, Y.ld), "band_matvec")

    def multiply_a(self, X, Y):
        self._mult(self._mv_a, X, Y)

    def multiply_b(self, X, Y):
        if self.FB is None:
            Y.copy_from(X)
        else:
            self._mult(self._mv_b, X, Y)


class B200BandOps:
    """Numpy-protocol adapter (for the reference's run_rci) over DeviceBandOps;
    ``fa``/``fb`` in the full-band layout of expand_band."""

    def __init__(self, fa, fb, kl, hermitian=None, device=None):
        fa = np.asarray(fa)
        self._lock = threading.RLock()
        self.hermitian = np.iscomplexobj(fa) if hermitian is None else hermitian
        self.dev = get_device(device)
        FA = self.dev.upload(fa, cplx=self.hermitian)
        FB = None if fb is None else self.dev.upload(np.asarray(fb), cplx=self.hermitian)
        self._ops = DeviceBandOps(self.dev, FA, FB, kl, self.hermitian)
        self.n = fa.shape[1]

    def factorize(self, z):
        # feastlib's run_rci calls this from a ThreadPoolExecutor when
        # parallel_contour > 1 (_driver.py:51-54): one GPU context, one stream,
        # shared factor cache -> calls are serialised
        with self._lock:
            return self._ops.factorize(z)

    def _solve(self, f, rhs, adjoint):
        W = self.dev.upload(np.asarray(rhs, dtype=np.complex128), cplx=True)
        with self._lock:
            self._ops._solve(f, W, adjoint)
            return self.dev.download(W)

    def solve(self, f, rhs):
        return self._solve(f, rhs, False)

    def solve_adjoint(self, f, rhs):
        return self._solve(f, rhs, True)

    def _mult(self, fn, x):
        X = self.dev.upload(np.asarray(x), cplx=self.hermitian)
        Y = self.dev.empty(self.n, X.cols, self.hermitian)
        with self._lock:
            fn(X, Y)
            return self.dev.download(Y)

    def multiply_a(self, x):
        return self._mult(self._ops.multiply_a, x)

    def multiply_b(self, x):
        return self._mult(self._ops.multiply_b, x)


def _banded_driver(a, kla, b, klb, emin, emax, m0, uplo, fpm, options, x0, hermitian, device=None,
                   engine_kwargs=None):
    options = options or SolverOptions()
    fpm = FeastParams.coerce(fpm) if fpm is not None else feastinit()
    uplo = (uplo or "F").upper()
    if not _is_torch(a):
        a = np.asarray(a)
    n = a.shape[1] if a.ndim == 2 else 0
    single = str(a.dtype).endswith(("float32", "complex64"))
    scalar = (np.complex64 if single else np.complex128) if hermitian else (np.float32 if single else np.float64)
    t = ("C" if single else "Z") if hermitian else ("S" if single else "D")
    routine = f"{t}FEAST_{'HB' if hermitian else 'SB'}{'GV' if b is not None else 'EV'}"
    cls = HermitianRci if hermitian else SymmetricRci
    kernel = cls(n, m0, emin, emax, fpm, seed=options.seed, block_size=options.block_size,
                 dtype=scalar, routine_name=routine, device=device, host_mirror=False,
                 **(engine_kwargs or {}))
    if uplo not in _UPLOS:
        kernel.abort(-101)
        return kernel.result
    if not 0 <= kla <= max(n - 1, 0):
        kernel.abort(-103)
        return kernel.result
    if a.ndim != 2 or a.shape[0] < band_required_rows(kla, uplo):
        kernel.abort(-105)
        return kernel.result
    if b is not None:
        if not _is_torch(b):
            b = np.asarray(b)
        if klb is None or not 0 <= klb <= max(n - 1, 0):
            kernel.abort(-106)
            return kernel.result
        if b.ndim != 2 or b.shape[1] != n or b.shape[0] < band_required_rows(klb, uplo):
            kernel.abort(-108)
            return kernel.result
    if kernel.done:
        return kernel.result
    kl = max(kla, klb if b is not None else 0)
    dev = kernel.dev
    try:
        FA = expand_band_device(dev, a, kla, uplo, hermitian, kl)
        FB = None if b is None else expand_band_device(dev, b, klb, uplo, hermitian, kl)
    except MemoryError:
        kernel.abort(-1)
        return kernel.result
    if fpm.slot(5) == 1:
        if x0 is None:
            raise ValueError("fpm(5)=1 requires an initial subspace x0")
        dev.upload(np.asarray(x0)[:, :m0], cplx=hermitian, out=kernel.X)
    try:
        mv_a = (expand_band_device(dev, a, kla, uplo, hermitian, kla), kla) if kla < kl else None
        mv_b = (expand_band_device(dev, b, klb, uplo, hermitian, klb), klb) if b is not None and klb < kl else None
    except MemoryError:
        kernel.abort(-1)
        return kernel.result
    ops = DeviceBandOps(dev, FA, FB, kl, hermitian, mv_a=mv_a, mv_b=mv_b)
    result = run_rci(kernel, ops, options)
    result.factorizations = ops.factorizations
    return result


def feast_sb(a, kla, emin, emax, m0, *, uplo="F", b=None, klb=None, fpm=None, options=None,
             x0=None, device=None):
    """Real symmetric banded driver (banded.py:240-250)."""
    return _banded_driver(a, kla, b, klb, emin, emax, m0, uplo, fpm, options, x0, False, device)


def feast_hb(a, kla, emin, emax, m0, *, uplo="F", b=None, klb=None, fpm=None, options=None,
             x0=None, device=None):
    """Complex Hermitian banded driver (banded.py:253-258)."""
    return _banded_driver(a, kla, b, klb, emin, emax, m0, uplo, fpm, options, x0, True, device)
