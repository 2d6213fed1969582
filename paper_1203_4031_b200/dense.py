"""Dense drivers feast_sy / feast_he on the GPU (mirrors dense.py:1-183).

``DeviceDenseOps`` answers the engine's tasks on the device:
  factorize(z)   S = z B - A (fb_dense_shift) + blocked LU (fb_zgetrf)
  solve / solve_adjoint   fb_zgetrs in place on the engine's work2
  multiply_a / multiply_b  DMMA GEMM (fb_gemm), or a copy when B = I
``B200DenseOps`` is the same backend behind the reference's numpy ops
protocol, for plugging into feastlib's own ``run_rci``.
"""

from __future__ import annotations

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
    __slots__ = ("z", "lu", "piv", "dinv", "info", "resident")

    def __init__(self, z, lu, piv, dinv, info, resident):
        self.z, self.lu, self.piv, self.dinv, self.info, self.resident = z, lu, piv, dinv, info, resident


class DeviceDenseOps:
    """Device backend for the dense drivers.

    Factor cache policy: factors stay resident while they fit in
    ``cache_bytes`` (default: 85% of free HBM at construction); shifts beyond
    that are re-factorized into one shared slot when solved (config 5 at
    N = 32768 holds ~8 of its 16 factors on one B200)."""

    on_device = True
    # bench.py instrumentation: when a list, (start, end) CUDA events recorded
    # on the context stream around every fb_zgetrf call are appended to it.
    lu_event_sink = None

    def __init__(self, dev, A: Planar, B: Planar | None, hermitian: bool, cache_bytes=None):
        self.dev, self.A, self.B, self.hermitian = dev, A, B, hermitian
        self.n = A.rows
        torch = dev.torch
        if cache_bytes is None:
            free, _ = torch.cuda.mem_get_info(dev.tdev)
            cache_bytes = int(0.85 * free)
        self.cache_left = cache_bytes
        self._slot = None
        self.factorizations = 0

    def _factor_bytes(self):
        n = self.n
        return 16 * n * n + 8 * self.dev.lib.fb_zgetrf_dinv_doubles(n) + 4 * n

    def _new_factor(self, z, resident):
        dev, n, torch = self.dev, self.n, self.dev.torch
        lu = dev.empty(n, n, True)
        piv = torch.empty(n, dtype=torch.int32, device=dev.tdev)
        dinv = torch.empty(int(dev.lib.fb_zgetrf_dinv_doubles(n)), dtype=torch.float64, device=dev.tdev)
        info = torch.empty(1, dtype=torch.int32, device=dev.tdev)
        return _DenseFactor(z, lu, piv, dinv, info, resident)

    def _compute(self, f: _DenseFactor):
        dev, A, B, n, lib = self.dev, self.A, self.B, self.n, self.dev.lib
        z = f.z
        dev.check(lib.fb_dense_shift(dev.h, n, z.real, z.imag, A.re, A.im, A.ld,
                                     B.re if B is not None else None,
                                     B.im if B is not None else None,
                                     B.ld if B is not None else 0,
                                     f.lu.re, f.lu.im, f.lu.ld), "dense_shift")
        sink = DeviceDenseOps.lu_event_sink
        if sink is not None:
            ev = (dev.torch.cuda.Event(enable_timing=True), dev.torch.cuda.Event(enable_timing=True))
            ev[0].record()
        dev.check(lib.fb_zgetrf(dev.h, n, f.lu.re, f.lu.im, f.lu.ld, f.piv.data_ptr(),
                                f.dinv.data_ptr(), f.info.data_ptr()), "zgetrf")
        if sink is not None:
            ev[1].record()
            sink.append(ev)
        self.factorizations += 1
        bad = dev.read_info(f.info.data_ptr())
        if bad >= 0:
            raise SingularMatrixError(f"zero pivot at column {bad}")

    def factorize(self, z):
        z = complex(z)
        need = self._factor_bytes()
        if need <= self.cache_left:
            self.cache_left -= need
            f = self._new_factor(z, True)
            self._compute(f)
            return f
        if self._slot is None:
            self._slot = self._new_factor(None, False)
        f = _DenseFactor(z, None, None, None, None, False)
        self._materialize(f)
        return f

    def _materialize(self, f):
        if f.resident:
            return f
        s = self._slot
        if s.z != f.z:
            s.z = f.z
            try:
                self._compute(s)
            except Exception:
                s.z = None
                raise
        return s

    def _solve(self, f, W: Planar, adjoint):
        g = self._materialize(f)
        dev = self.dev
        dev.check(dev.lib.fb_zgetrs(dev.h, self.n, W.cols, g.lu.re, g.lu.im, g.lu.ld, g.piv.data_ptr(),
                                    g.dinv.data_ptr(), 1 if adjoint else 0, W.re, W.im, W.ld), "zgetrs")

    def solve(self, f, W: Planar):
        self._solve(f, W, False)

    def solve_adjoint(self, f, W: Planar):
        self._solve(f, W, True)

    def multiply_a(self, X: Planar, Y: Planar):
        self.dev.gemm("N", "N", self.n, X.cols, self.n, 1.0, self.A, X, 0.0, Y, cplx=self.hermitian)

    def multiply_b(self, X: Planar, Y: Planar):
        if self.B is None:
            Y.copy_from(X)
        else:
            self.dev.gemm("N", "N", self.n, X.cols, self.n, 1.0, self.B, X, 0.0, Y, cplx=self.hermitian)


class B200DenseOps:
    """The reference's numpy ops protocol (dense.py:91-117) backed by the GPU:
    arrays in and out are numpy; factorizations stay on the device."""

    def __init__(self, a, b=None, hermitian=None, device=None):
        a = np.asarray(a)
        self.hermitian = np.iscomplexobj(a) if hermitian is None else hermitian
        self.dev = get_device(device)
        A = self.dev.upload(a, cplx=self.hermitian)
        B = None if b is None else self.dev.upload(np.asarray(b), cplx=self.hermitian)
        self._ops = DeviceDenseOps(self.dev, A, B, self.hermitian)
        self.n = a.shape[0]

    def factorize(self, z):
        return self._ops.factorize(z)

    def _solve(self, f, rhs, adjoint):
        rhs = np.asarray(rhs, dtype=np.complex128)
        W = self.dev.upload(rhs, cplx=True)
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
        fn(X, Y)
        return self.dev.download(Y)

    def multiply_a(self, x):
        return self._mult(self._ops.multiply_a, x)

    def multiply_b(self, x):
        return self._mult(self._ops.multiply_b, x)


def _shape(a):
    return tuple(a.shape) if hasattr(a, "shape") else np.asarray(a).shape


def _dense_driver(a, b, emin, emax, m0, uplo, fpm, options, x0, hermitian, device=None,
                  engine_kwargs=None):
    options = options or SolverOptions()
    fpm = FeastParams.coerce(fpm) if fpm is not None else feastinit()
    uplo = (uplo or "F").upper()
    if not _is_torch(a):
        a = np.asarray(a)
    shp = _shape(a)
    n = shp[0] if len(shp) >= 1 else 0
    single = str(a.dtype).endswith(("float32", "complex64"))
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
        if not _is_torch(b):
            b = np.asarray(b)
        if _shape(b) != shp:
            kernel.abort(-106)
            return kernel.result
    if kernel.done:
        return kernel.result
    dev = kernel.dev
    try:
        A = _upload_full(dev, expand_uplo(a, uplo, hermitian), hermitian)
        B = None if b is None else _upload_full(dev, expand_uplo(b, uplo, hermitian), hermitian)
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
    result = run_rci(kernel, ops, options)
    result.factorizations = ops.factorizations
    return result


def _upload_full(dev, m, hermitian):
    if _is_torch(m):
        return dev.upload_torch(m, cplx=hermitian)
    return dev.upload(np.asarray(m), cplx=hermitian)


def _routine_name(hermitian, single, generalized):
    t = ("C" if single else "Z") if hermitian else ("S" if single else "D")
    return f"{t}FEAST_{'HE' if hermitian else 'SY'}{'GV' if generalized else 'EV'}"


def feast_sy(a, emin, emax, m0, *, uplo="F", b=None, fpm=None, options=None, x0=None, device=None):
    """Real symmetric A x = lambda x (or A x = lambda B x) on [emin, emax]
    (dense.py:166-173).  ``a``/``b`` may be numpy arrays or torch tensors
    (device-resident inputs skip the host->device copy)."""
    return _dense_driver(a, b, emin, emax, m0, uplo, fpm, options, x0, False, device)


def feast_he(a, emin, emax, m0, *, uplo="F", b=None, fpm=None, options=None, x0=None, device=None):
    """Complex Hermitian analogue (dense.py:176-183); adjoint solves reuse the
    direct LU (U^H L^H with reversed pivots)."""
    return _dense_driver(a, b, emin, emax, m0, uplo, fpm, options, x0, True, device)
