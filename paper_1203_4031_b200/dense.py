"""Dense drivers feast_sy / feast_he on the GPU (mirrors dense.py:1-183).

``DeviceDenseOps`` answers the engine's tasks on the device:
  factorize(z)   S = z B - A (fb_dense_shift) + blocked LU (fb_zgetrf)
  solve / solve_adjoint   fb_zgetrs in place on the engine's work2
  multiply_a / multiply_b  DMMA GEMM (fb_gemm), or a copy when B = I
``B200DenseOps`` is the same backend behind the reference's numpy ops
protocol, for plugging into feastlib's own ``run_rci``.
"""

from __future__ import annotations

import threading

import numpy as np

from ._driver import SolverOptions, run_rci
from ._errors import SingularMatrixError
from .device import Planar, get_device
from .kernel import HermitianRci, SymmetricRci
from .params import feastinit, FeastParams

_UPLOS = ("F", "L", "U")


def expand_uplo(a, uplo: str, hermitian: bool):
    """Full matrix from the stored triangle (dense.py:15-27); numpy or torch."""
    uplo = uplo.upper()
    if uplo == "F":
        return a
    if _is_torch(a):
        tri = a.tril() if uplo == "L" else a.triu()
        off = tri - tri.diagonal().diag_embed()
        return tri + (off.conj().T if hermitian else off.T)
    a = np.asarray(a)
    tri = np.tril(a) if uplo == "L" else np.triu(a)
    off = tri - np.diag(np.diag(tri))
    return tri + (off.conj().T if hermitian else off.T)


def _is_torch(x):
    return type(x).__module__.startswith("torch")


class _DenseFactor:
    """One shifted factorization: either item `idx` of a resident batch, or a
    non-resident shift re-factorized on demand into the shared slot."""

    __slots__ = ("z", "batch", "idx", "resident")

    def __init__(self, z, batch, idx, resident):
        self.z, self.batch, self.idx, self.resident = z, batch, idx, resident


class _FactorBatch:
    """Strided device storage of `count` LU factors (the C ABI batch layout)."""

    def __init__(self, dev, n, count):
        torch = dev.torch
        self.n, self.count = n, count
        self.lu = torch.empty((2, count, n, n), dtype=torch.float64, device=dev.tdev)
        self.piv = torch.empty((count, n), dtype=torch.int32, device=dev.tdev)
        self.dd = int(dev.lib.fb_zgetrf_dinv_doubles(n))
        self.dinv = torch.empty((count, self.dd), dtype=torch.float64, device=dev.tdev)
        self.info = torch.empty(count, dtype=torch.int32, device=dev.tdev)
        self.zs = [None] * count

    def args(self, i0=0):
        """(re, im, ld, lu_stride, piv, piv_stride, dinv, dinv_stride) of item i0 onwards."""
        n = self.n
        return (self.lu[0, i0].data_ptr(), self.lu[1, i0].data_ptr(), n, n * n,
                self.piv[i0].data_ptr(), n, self.dinv[i0].data_ptr(), self.dd)

    @staticmethod
    def nbytes(dev, n, count):
        return count * (16 * n * n + 4 * n + 8 * int(dev.lib.fb_zgetrf_dinv_doubles(n)))


class DeviceDenseOps:
    """Device backend for the dense drivers.

    * ``prefactorize(zs)`` forms and factors all of this rank's shifts in ONE
      batched pass (fb_dense_shift_batched + fb_zgetrf_batched) — the GPU form
      of parallel_contour (_driver.py:46-54): results are identical to
      one-at-a-time factorization.
    * ``solve_pass(Y, hermitian)`` (called by the engine at the start of every
      contour pass) solves all resident shifts against the pass's Y in one
      batched call (fb_zgetrs_batched, direct and, for Hermitian pencils,
      adjoint); the per-point SOLVE tasks then copy their block out.
    * Factor cache policy: factors stay resident while they fit in
      ``cache_bytes`` (default: 85% of free HBM at construction); shifts beyond
      that are factorized into one shared slot when solved (config 5 at
      N = 32768 holds ~8 of its 16 factors on one B200).  A factor built in
      the slot is kept in pinned host memory while the host has room
      (80 % of the available RAM, at least 24 GB left free; FB_HOST_FACTORS=0 turns
      it off), so later passes copy it back over PCIe (~0.35 s for 17 GB)
      instead of refactorizing it (~3 s at N = 32768).
    """

    on_device = True
    # bench.py instrumentation: when a list, (start, end, count) CUDA events recorded
    # on the context stream around every batched factorization are appended to it.
    lu_event_sink = None

    def __init__(self, dev, A: Planar, B: Planar | None, hermitian: bool, cache_bytes=None):
        self.dev, self.A, self.B, self.hermitian = dev, A, B, hermitian
        self.n = A.rows
        torch = dev.torch
        if cache_bytes is None:
            import os
            free, _ = torch.cuda.mem_get_info(dev.tdev)
            cache_bytes = int(0.85 * free)
            if os.environ.get("FB_FACTOR_CACHE_MB"):   # testing: force non-resident factors
                cache_bytes = min(cache_bytes, int(float(os.environ["FB_FACTOR_CACHE_MB"]) * 2**20))
        self.cache_left = cache_bytes
        self._slot = None
        self._host = {}          # z -> (lu, piv, dinv) pinned host copies of slot factors
        self.host_loads = 0
        self._host_left = self._host_budget()
        self.factorizations = 0
        self._batches = []
        self._pass = {}          # (id(batch), idx, adjoint) -> Planar result of this pass
        self._zmap = {}          # z -> (batch, idx) of resident factors
        self._xbuf = {}          # (id(batch), adjoint) -> pass result buffer, reused across passes

    # -- factorization -------------------------------------------------------------
    def _factor_batch(self, fb_, zs):
        dev, A, B, n, lib = self.dev, self.A, self.B, self.n, self.dev.lib
        import ctypes
        cnt = len(zs)
        zr = (ctypes.c_double * cnt)(*[z.real for z in zs])
        zi = (ctypes.c_double * cnt)(*[z.imag for z in zs])
        re, im, ld, slu, piv, spiv, dinv, sdinv = fb_.args()
        dev.check(lib.fb_dense_shift_batched(dev.h, cnt, n, zr, zi, A.re, A.im, A.ld,
                                             B.re if B is not None else None,
                                             B.im if B is not None else None,
                                             B.ld if B is not None else 0, re, im, ld, slu), "dense_shift")
        sink = DeviceDenseOps.lu_event_sink
        if sink is not None:
            ev = (dev.torch.cuda.Event(enable_timing=True), dev.torch.cuda.Event(enable_timing=True))
            ev[0].record()
        dev.check(lib.fb_zgetrf_batched(dev.h, cnt, n, re, im, ld, slu, piv, spiv, dinv, sdinv,
                                        fb_.info.data_ptr()), "zgetrf")
        if sink is not None:
            ev[1].record()
            sink.append((ev[0], ev[1], cnt))
        self.factorizations += cnt
        bad = (ctypes.c_int * cnt)()
        rc = lib.fb_read_info_batched(dev.h, cnt, ctypes.c_void_p(fb_.info.data_ptr()), bad)
        if rc == -2:
            k = next(i for i in range(cnt) if bad[i] >= 0)
            raise SingularMatrixError(f"zero pivot at column {bad[k]} (shift {zs[k]})")
        dev.check(rc, "read_info")
        for i, z in enumerate(zs):
            fb_.zs[i] = z

    def prefactorize(self, zs):
        """Factor every shift that fits in the cache in one batched call;
        returns {z: factor} for those (the rest are factorized on demand)."""
        zs = [complex(z) for z in zs]
        per = _FactorBatch.nbytes(self.dev, self.n, 1)
        fit = min(len(zs), max(0, self.cache_left // per))
        out = {}
        if fit == 0:
            return out
        self.cache_left -= fit * per
        fb_ = _FactorBatch(self.dev, self.n, fit)
        self._factor_batch(fb_, zs[:fit])
        self._batches.append(fb_)
        for i, z in enumerate(zs[:fit]):
            out[z] = _DenseFactor(z, fb_, i, True)
            self._zmap[z] = (fb_, i)
        return out

    def factorize(self, z):
        z = complex(z)
        got = self.prefactorize([z]) if self.cache_left >= _FactorBatch.nbytes(self.dev, self.n, 1) else {}
        if z in got:
            return got[z]
        if self._slot is None:
            self._slot = _FactorBatch(self.dev, self.n, 1)
        f = _DenseFactor(z, None, 0, False)
        self._materialize(f)
        return f

    @staticmethod
    def _host_budget():
        import os
        if os.environ.get("FB_HOST_FACTORS", "1") == "0":
            return 0
        try:
            import psutil
            avail = psutil.virtual_memory().available
            return int(max(0, min(0.8 * avail, avail - 24 * 2**30)))
        except Exception:
            return 0

    def _materialize(self, f):
        if f.resident:
            return f.batch, f.idx
        s = self._slot
        if s.zs[0] != f.z:
            s.zs[0] = None
            hit = self._host.get(f.z)
            if hit is not None:       # host tier: copy the factor back instead of refactorizing
                s.lu[:, 0].copy_(hit[0], non_blocking=True)
                s.piv[0].copy_(hit[1], non_blocking=True)
                s.dinv[0].copy_(hit[2], non_blocking=True)
                s.zs[0] = f.z
                self.host_loads += 1
            else:
                self._factor_batch(s, [f.z])
                self._keep_on_host(f.z, s)
        return s, 0

    def _keep_on_host(self, z, s):
        need = _FactorBatch.nbytes(self.dev, self.n, 1)
        if need > self._host_left:
            return
        torch = self.dev.torch
        try:
            lu = torch.empty(s.lu[:, 0].shape, dtype=s.lu.dtype, pin_memory=True)
            piv = torch.empty(s.piv[0].shape, dtype=s.piv.dtype, pin_memory=True)
            dinv = torch.empty(s.dinv[0].shape, dtype=s.dinv.dtype, pin_memory=True)
        except RuntimeError:
            self._host_left = 0
            return
        lu.copy_(s.lu[:, 0], non_blocking=True)
        piv.copy_(s.piv[0], non_blocking=True)
        dinv.copy_(s.dinv[0], non_blocking=True)
        self._host[z] = (lu, piv, dinv)
        self._host_left -= need

    # -- solves ----------------------------------------------------------------------
    def solve_pass(self, Y: Planar, hermitian: bool):
        """Batched solves of every resident shift against this pass's Y."""
        self._pass = {}
        dev, n, m = self.dev, self.n, Y.cols
        W = Y
        if not Y.cplx:   # real Y (symmetric pencils): complex copy for the solver
            W = dev.empty(n, m, True)
            W.copy_from(Y)
        for fb_ in self._batches:
            cnt = fb_.count
            for adj in ((0, 1) if hermitian else (0,)):
                # even leading dimension: the sweeps' 16-byte path also when M0
                # has shrunk to an odd column count (kernel.py:385-400)
                mp = m + (m & 1)
                X = self._xbuf.get((id(fb_), adj))
                if X is None or X.shape[3] != mp:
                    X = dev.torch.empty((2, cnt, n, mp), dtype=dev.torch.float64, device=dev.tdev)
                    self._xbuf[(id(fb_), adj)] = X
                re, im, ld, slu, piv, spiv, dinv, sdinv = fb_.args()
                dev.check(dev.lib.fb_zgetrs_batched(dev.h, cnt, n, m, re, im, ld, slu, piv, spiv, dinv, sdinv,
                                                    adj, W.re, W.im, W.ld, 0, X[0].data_ptr(),
                                                    X[1].data_ptr(), mp, n * mp), "zgetrs_batched")
                for i in range(cnt):
                    self._pass[(id(fb_), i, adj)] = (X, i, m)

    def pass_result(self, z, adjoint):
        """Planar view of this pass's solve for shift z (None if not resident)."""
        hit = self._zmap.get(complex(z))
        if hit is None:
            return None
        got = self._pass.get((id(hit[0]), hit[1], int(adjoint)))
        if got is None:
            return None
        X, i, m = got
        return Planar(X[:, i], True, X.shape[2], m, X.shape[3])

    def _solve(self, f, W: Planar, adjoint):
        if f.resident:
            hit = self._pass.get((id(f.batch), f.idx, int(adjoint)))
            if hit is not None:
                X, i, _ = hit
                W.plane(0).copy_(X[0, i][:, :W.cols])
                W.plane(1).copy_(X[1, i][:, :W.cols])
                return
        fb_, i = self._materialize(f)
        dev = self.dev
        re, im, ld, slu, piv, spiv, dinv, sdinv = fb_.args(i)
        dev.check(dev.lib.fb_zgetrs(dev.h, self.n, W.cols, re, im, ld, piv, dinv, 1 if adjoint else 0,
                                    W.re, W.im, W.ld), "zgetrs")

    def solve(self, f, W: Planar):
        self._solve(f, W, False)

    def solve_adjoint(self, f, W: Planar):
        self._solve(f, W, True)

    # ``rows`` = (r0, r1): multi-GPU row sharding -- only that row block of the
    # product is computed (the kernel reads no other rows, kernel.py _row_block)
    rows = None

    def _mult(self, M: Planar, X: Planar, Y: Planar):
        r0, r1 = self.rows if self.rows is not None else (0, self.n)
        self.dev.gemm("N", "N", r1 - r0, X.cols, self.n, 1.0, M.rows_view(r0, r1), X, 0.0,
                      Y.rows_view(r0, r1), cplx=self.hermitian)

    def multiply_a(self, X: Planar, Y: Planar):
        self._mult(self.A, X, Y)

    def multiply_b(self, X: Planar, Y: Planar):
        if self.B is None:
            Y.copy_from(X)
        else:
            self._mult(self.B, X, Y)


class B200DenseOps:
    """The reference's numpy ops protocol (dense.py:91-117) backed by the GPU:
    arrays in and out are numpy; factorizations stay on the device."""

    def __init__(self, a, b=None, hermitian=None, device=None):
        a = np.asarray(a)
        self._lock = threading.RLock()
        self.hermitian = np.iscomplexobj(a) if hermitian is None else hermitian
        self.dev = get_device(device)
        A = self.dev.upload(a, cplx=self.hermitian)
        B = None if b is None else self.dev.upload(np.asarray(b), cplx=self.hermitian)
        self._ops = DeviceDenseOps(self.dev, A, B, self.hermitian)
        self.n = a.shape[0]

    def factorize(self, z):
        # feastlib's run_rci calls this from a ThreadPoolExecutor when
        # parallel_contour > 1 (_driver.py:51-54): one GPU context, one stream,
        # shared factor cache -> calls are serialised
        with self._lock:
            return self._ops.factorize(z)

    def _solve(self, f, rhs, adjoint):
        rhs = np.asarray(rhs, dtype=np.complex128)
        W = self.dev.upload(rhs, cplx=True)
        with self._lock:
            self._ops._solve(f, W, adjoint)
            return self.dev.download(W)

    def solve(self, f, rhs):
        return self._solve(f, rhs, False)

    def solve_adjoint(self, f, rhs):
        return self._solve(f, rhs, True)

    def _mult(self, fn, x):
        x = np.asarray(x)
        X = self.dev.upload(x, cplx=self.hermitian)
        Y = self.dev.empty(self.n, X.cols, self.hermitian)
        with self._lock:
            fn(X, Y)
            return self.dev.download(Y)

    def multiply_a(self, x):
        return self._mult(self._ops.multiply_a, x)

    def multiply_b(self, x):
        return self._mult(self._ops.multiply_b, x)


def _shape(a):
    if isinstance(a, Planar):
        return (a.rows, a.cols)
    return tuple(a.shape) if hasattr(a, "shape") else np.asarray(a).shape


def _dtype_name(a):
    if isinstance(a, Planar):
        return "complex128" if a.cplx else "float64"
    return str(a.dtype)


def _dense_driver(a, b, emin, emax, m0, uplo, fpm, options, x0, hermitian, device=None,
                  engine_kwargs=None):
    options = options or SolverOptions()
    fpm = FeastParams.coerce(fpm) if fpm is not None else feastinit()
    uplo = (uplo or "F").upper()
    if not _is_torch(a) and not isinstance(a, Planar):
        a = np.asarray(a)
    shp = _shape(a)
    n = shp[0] if len(shp) >= 1 else 0
    single = _dtype_name(a).endswith(("float32", "complex64"))
    scalar = (np.complex64 if single else np.complex128) if hermitian else (np.float32 if single else np.float64)
    routine = _routine_name(hermitian, single, b is not None)
    cls = HermitianRci if hermitian else SymmetricRci
    kernel = cls(n, m0, emin, emax, fpm, seed=options.seed, block_size=options.block_size,
                 dtype=scalar, routine_name=routine, device=device, host_mirror=False,
                 **(engine_kwargs or {}))
    if uplo not in _UPLOS:
        kernel.abort(-101)
        return kernel.result
    if len(shp) != 2 or shp[0] != shp[1]:
        kernel.abort(-104)
        return kernel.result
    if b is not None:
        if not _is_torch(b) and not isinstance(b, Planar):
            b = np.asarray(b)
        if _shape(b) != shp:
            kernel.abort(-106)
            return kernel.result
    if kernel.done:
        return kernel.result
    dev = kernel.dev
    try:
        A = _upload_full(dev, a if isinstance(a, Planar) else expand_uplo(a, uplo, hermitian), hermitian)
        B = None if b is None else _upload_full(
            dev, b if isinstance(b, Planar) else expand_uplo(b, uplo, hermitian), hermitian)
    except MemoryError:
        kernel.abort(-1)
        return kernel.result
    if fpm.slot(5) == 1:
        if x0 is None:
            raise ValueError("fpm(5)=1 requires an initial subspace x0")
        x0h = x0 if _is_torch(x0) else np.asarray(x0)
        if _is_torch(x0h):
            dev.upload_torch(x0h[:, :m0], cplx=hermitian, out=kernel.X)
        else:
            dev.upload(x0h[:, :m0], cplx=hermitian, out=kernel.X)
    ops = DeviceDenseOps(dev, A, B, hermitian)
    ops.rows = kernel._rows if kernel._sharded() else None
    result = run_rci(kernel, ops, options)
    result.factorizations = ops.factorizations
    return result


def _upload_full(dev, m, hermitian):
    if isinstance(m, Planar):
        # already device-resident planar (full storage): used as is, no copy
        if m.cplx != hermitian or m.rows != m.cols:
            raise ValueError("planar input must be square and complex iff hermitian")
        return m
    if _is_torch(m):
        return dev.upload_torch(m, cplx=hermitian)
    return dev.upload(np.asarray(m), cplx=hermitian)


def _routine_name(hermitian, single, generalized):
    t = ("C" if single else "Z") if hermitian else ("S" if single else "D")
    return f"{t}FEAST_{'HE' if hermitian else 'SY'}{'GV' if generalized else 'EV'}"


def feast_sy(a, emin, emax, m0, *, uplo="F", b=None, fpm=None, options=None, x0=None, device=None):
    """Real symmetric A x = lambda x (or A x = lambda B x) on [emin, emax]
    (dense.py:166-173).  ``a``/``b`` may be numpy arrays, torch tensors or
    full-storage device ``Planar`` matrices (device-resident inputs skip the
    host->device copy; a ``Planar`` is used in place)."""
    return _dense_driver(a, b, emin, emax, m0, uplo, fpm, options, x0, False, device)


def feast_he(a, emin, emax, m0, *, uplo="F", b=None, fpm=None, options=None, x0=None, device=None):
    """Complex Hermitian analogue (dense.py:176-183); adjoint solves reuse the
    direct LU (U^H L^H with reversed pivots)."""
    return _dense_driver(a, b, emin, emax, m0, uplo, fpm, options, x0, True, device)
