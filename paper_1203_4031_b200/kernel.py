"""Reverse-communication FEAST engine with device-resident state.

The task grammar, the fpm(24)/fpm(25) multiply ranges, the convergence tests
and the output ordering follow feastlib's engine (kernel.py:183-531) line for
line; what changes is where the state lives.  Y, Q, work1, work2, X and the
A-products are planar FP64 buffers on the GPU, and every O(N M0) / O(N M0^2)
step of the loop — start block, quadrature accumulation, projections
Q^H A Q / Q^H B Q, reduced eigensolve, Ritz vectors and residuals — is a call
into libfeastb200.so.  Only M0-sized scalars (eigenvalues, residuals, the
Cholesky failure index) come back to the host each refinement pass.

Two ways to drive it:

* the public RCI surface (``SymmetricRci`` / ``HermitianRci``) keeps numpy
  mirrors of ``work1``/``work2``/``x`` so a user loop written against the
  reference (kernel.py:8-22) runs unchanged: before a SOLVE the right-hand
  sides are copied to the host, after it the answer is copied back;
* the predefined drivers construct the engine with ``host_mirror=False`` and
  answer every task on the device (see ``_driver.run_rci``).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from ._errors import ReducedSolverError  # noqa: F401  (re-export parity)
from .device import get_device
from .params import (MAX_TOL_EXP_DOUBLE, MAX_TOL_EXP_SINGLE, check_problem, feastinit,
                     info_classification, validate_params, FeastParams)
from .quadrature import build_contour, gauss_legendre

DEFAULT_SEED = 42


class RciTask(enum.IntEnum):
    """Task codes (kernel.py:46-56)."""

    INIT = -1
    DONE = 0
    FACTORIZE = 10
    SOLVE = 11
    FACTORIZE_ADJOINT = 20
    SOLVE_ADJOINT = 21
    MULTIPLY_A = 30
    MULTIPLY_B = 40


@dataclass
class EigenResult:
    """Output of a solve (kernel.py:59-80)."""

    e: np.ndarray
    x: np.ndarray
    m: int
    res: np.ndarray
    epsout: float
    loop: int
    info: int
    m0: int

    @property
    def classification(self) -> str:
        return info_classification(self.info)


# --- host helpers kept for API parity (kernel.py:90-177) --------------------
_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def random_uniform(seed: int, offset: int, count: int) -> np.ndarray:
    """Host evaluation of the counter-based SplitMix64 stream (kernel.py:90-102);
    the engine itself fills Y on the device with fb_splitmix."""
    c = np.arange(offset + 1, offset + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed % (1 << 64)) + c * _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    z ^= z >> np.uint64(31)
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0


def trace_error(trace_cur: float, trace_prev: float, emin: float, emax: float) -> float:
    """|t_k - t_{k-1}| / max(|emin|, |emax|)  (kernel.py:127-129)."""
    return abs(trace_cur - trace_prev) / max(abs(emin), abs(emax))


def _ordering(evalues, res, emin, emax):
    """Permutation and count of filter_sort_flag (kernel.py:156-177)."""
    spurious = (res < 0) | ~np.isfinite(res)
    inside = (evalues >= emin) & (evalues <= emax) & ~spurious
    outside = ~inside & ~spurious
    idx_in = np.flatnonzero(inside)
    idx_in = idx_in[np.argsort(evalues[idx_in], kind="stable")]
    order = np.concatenate([idx_in, np.flatnonzero(outside), np.flatnonzero(spurious)])
    return order, len(idx_in), int(spurious.sum())


def filter_sort_flag(evalues, x, res, emin, emax) -> int:
    """In-place reorder: inside (ascending), outside, spurious (res = -1)."""
    m0 = evalues.shape[0]
    order, m, nsp = _ordering(evalues, res, emin, emax)
    evalues[:] = evalues[order]
    x[:, :m0] = x[:, order]
    res[:] = res[order]
    if nsp:
        res[m0 - nsp:] = -1.0
    return m


def accumulate_subspace(q, work2, weight, radius, theta, variant) -> None:
    """kernel.py:108-124 on numpy arrays, computed by the device kernel."""
    if q.shape != work2.shape:
        raise ValueError(f"shape mismatch: {q.shape} vs {work2.shape}")
    code = {"symmetric": 0, "hermitian-direct": 1, "hermitian-adjoint": 2}.get(variant)
    if code is None:
        raise ValueError(f"unknown variant {variant!r}")
    dev = get_device()
    cq = np.iscomplexobj(q)
    Q = dev.upload(q, cplx=cq)
    X = dev.upload(np.asarray(work2, dtype=np.complex128), cplx=True)
    dev.accumulate(code, X, Q, weight, radius, theta)
    q[...] = dev.download(Q)


def residual(a_apply, b_apply, lam, x_col, emin, emax) -> float:
    """kernel.py:132-144 (host scalar helper, API parity)."""
    ax = a_apply(x_col)
    bx = b_apply(x_col) if b_apply is not None else x_col
    den = np.abs(max(abs(emin), abs(emax)) * bx).sum()
    if den == 0.0:
        return np.inf
    return float(np.abs(ax - lam * bx).sum() / den)


# --- the engine -----------------------------------------------------------------
class _RciKernel:
    hermitian = False

    def __init__(self, n, m0, emin, emax, fpm=None, *, seed=DEFAULT_SEED, block_size=None,
                 dtype=None, routine_name=None, device=None, host_mirror=True,
                 adjoint_capable=True, points=None, q_reduce=None, rows=None, sum_reduce=None,
                 flag_reduce=None):
        self.n = int(n)
        self.m0 = int(m0)
        self._m0_init = int(m0)
        self.emin = float(emin)
        self.emax = float(emax)
        self.fpm = FeastParams.coerce(fpm) if fpm is not None else feastinit()
        self.seed = int(seed)
        self.block_size = block_size
        self.adjoint_capable = bool(adjoint_capable)
        self.host_mirror = bool(host_mirror)
        self.ze = 0j
        self.task = RciTask.INIT
        self.info = 0
        self.epsout = 1.0
        self.loop = 0
        self.m = 0
        self._done = False
        self._gen = None
        self._points = points          # contour indices served by this rank (None: all)
        self._q_reduce = q_reduce      # callable(Q planar) summing partial Q over ranks
        # multi-GPU row sharding of the projection / Ritz / residual products
        # (SURVEY.md §8e): this rank owns rows [r0, r1) of A*Q, B*Q, A*X, B*X;
        # sum_reduce(torch tensor) all-reduces the reduced matrices, the
        # residual sums and the next right-hand side; flag_reduce(code) -> the
        # most severe abort code over the ranks (0: carry on)
        self._rows = tuple(rows) if rows is not None else None
        self._sum_reduce = sum_reduce
        self._flag_reduce = flag_reduce
        self._solve_pass = None        # callable(Y, hermitian): batched solves of a pass
        self._pass_result = None       # callable(z, adjoint) -> Planar result of this pass, or None
        self._solve_pass_acc = None    # callable(Y, spec, radius, Q) -> bool: solves + accumulation fused
        self.solve_fused = False       # this pass's SOLVE tasks were answered by solve_pass
        scalar = np.dtype(dtype) if dtype is not None else (
            np.dtype(np.complex128) if self.hermitian else np.dtype(np.float64))
        self._single = scalar in (np.dtype(np.float32), np.dtype(np.complex64))
        self._out_real = np.float32 if self._single else np.float64
        self._out_work = (np.complex64 if self._single else np.complex128) if self.hermitian \
            else self._out_real
        self.routine_name = routine_name or self._default_routine_name()
        mz, nz = max(self._m0_init, 0), max(self.n, 0)
        self.e = np.zeros(mz, dtype=np.float64)
        self.res = np.zeros(mz, dtype=np.float64)
        info = check_problem(self.n, self.m0, self.emin, self.emax)
        if info == 0:
            info = validate_params(self.fpm)
        if info != 0:
            self.info = info
            self._done = True
            self._mirrors(nz, mz)
            self.dev = None
            return
        try:
            self.dev = get_device(device)
            self._alloc()
        except MemoryError:
            self.info = -1
            self._done = True
            self._mirrors(nz, mz)
            self.dev = None
            return
        self._mirrors(nz, mz)
        self._gen = self._run()
        self._pending_x0 = False

    # -- buffers -----------------------------------------------------------
    def _alloc(self):
        dev, n, m = self.dev, self.n, self._m0_init
        h = self.hermitian
        self.Y = dev.zeros(n, m, h)
        self.Q = dev.zeros(n, m, h)
        self.W1 = dev.zeros(n, m, h)
        self.W2 = dev.zeros(n, m, True)
        self.X = dev.zeros(n, m, h)
        self.AP = dev.zeros(n, m, h)
        self.AX = dev.zeros(n, m, h)
        self.BX = dev.zeros(n, m, h)
        self.AQ = dev.zeros(m, m, h)
        self.BQ = dev.zeros(m, m, h)
        self.PHI = dev.zeros(m, m, h)
        torch = dev.torch
        self.e_dev = torch.zeros(m, dtype=torch.float64, device=dev.tdev)
        self.res_dev = torch.zeros(m, dtype=torch.float64, device=dev.tdev)
        self._res_sums = torch.zeros(2 * max(m, 1), dtype=torch.float64, device=dev.tdev)

    def _mirrors(self, n, m):
        if self.host_mirror:
            wt = np.complex128 if self.hermitian else np.float64
            self.work1 = np.zeros((n, m), dtype=wt)
            self.work2 = np.zeros((n, m), dtype=np.complex128)
            self.x = np.zeros((n, m), dtype=wt)
        else:
            self.work1 = self.work2 = None
            self.x = None

    def _default_routine_name(self):
        if self.hermitian:
            return "CFEAST_HRCI" if self._single else "ZFEAST_HRCI"
        return "SFEAST_SRCI" if self._single else "DFEAST_SRCI"

    # -- caller-facing surface (kernel.py:250-302) ---------------------------
    def step(self) -> RciTask:
        if self._done:
            self.task = RciTask.DONE
            return self.task
        if self.host_mirror:
            self._push(self.task)
        try:
            self.task = next(self._gen)
        except StopIteration:
            self._done = True
            self.task = RciTask.DONE
        if self.host_mirror:
            self._pull(self.task)
        return self.task

    def _push(self, task):
        """Host mirror -> device after the caller answered ``task``."""
        m0 = self.m0
        if task == RciTask.INIT and self.fpm.slot(5) == 1:
            self.dev.upload(self.x, cplx=self.hermitian, out=self.X)
        elif task in (RciTask.SOLVE, RciTask.SOLVE_ADJOINT):
            self.dev.upload(self.work2[:, :m0], cplx=True, out=self.W2.cols_view(0, m0))
        elif task in (RciTask.MULTIPLY_A, RciTask.MULTIPLY_B):
            s = self.multiply_columns
            self.dev.upload(self.work1[:, s], cplx=self.hermitian,
                            out=self.W1.cols_view(s.start, s.stop))

    def _pull(self, task):
        """Device -> host mirror before handing ``task`` to the caller."""
        m0 = self.m0
        if task in (RciTask.SOLVE, RciTask.SOLVE_ADJOINT):
            self.work2[:, :m0] = self.dev.download(self.W2.cols_view(0, m0))
        elif task in (RciTask.MULTIPLY_A, RciTask.MULTIPLY_B):
            s = self.multiply_columns
            self.x[:, s] = self.dev.download(self.X.cols_view(s.start, s.stop))

    @property
    def multiply_columns(self) -> slice:
        first = self.fpm.slot(24) - 1
        return slice(first, first + self.fpm.slot(25))

    @property
    def done(self) -> bool:
        return self._done

    def abort(self, info: int) -> None:
        self.info = int(info)
        self._done = True
        self._gen = None
        self.task = RciTask.DONE

    def x_host(self):
        if self.dev is None or not hasattr(self, "X"):
            wt = self._out_work
            return np.zeros((max(self.n, 0), max(self._m0_init, 0)), dtype=wt)
        return self.dev.download(self.X).astype(self._out_work, copy=False)

    @property
    def result(self) -> EigenResult:
        x = self.x_host()
        if self.host_mirror and self.x is not None:
            self.x[...] = x
        r = EigenResult(e=self.e.astype(self._out_real), x=x, m=self.m,
                        res=self.res.astype(self._out_real), epsout=float(self.epsout),
                        loop=self.loop, info=self.info, m0=self.m0)
        r.history = np.array(getattr(self, "history", []), dtype=np.float64).reshape(-1, 5)
        return r

    # -- engine internals ----------------------------------------------------
    def _tolerance(self):
        if self._single:
            return 10.0 ** -min(self.fpm.slot(7), MAX_TOL_EXP_SINGLE)
        return 10.0 ** -min(self.fpm.slot(3), MAX_TOL_EXP_DOUBLE)

    def _multiply_blocks(self, task):
        m0 = self.m0
        blk = self.block_size if self.block_size else m0
        start = 0
        while start < m0:
            cols = min(blk, m0 - start)
            self.fpm.set_slot(24, start + 1)
            self.fpm.set_slot(25, cols)
            yield task
            start += cols

    def _row_block(self):
        return self._rows if self._rows is not None else (0, self.n)

    def _sharded(self):
        return self._rows is not None and self._sum_reduce is not None

    def _next_rhs(self):
        """Y <- B*X (in W1) for the next contour pass.  Row-sharded multiplies
        leave only this rank's rows of W1 valid, and every rank solves its
        shifts against the WHOLE right-hand side: own rows, zeros elsewhere,
        summed over the ranks."""
        Yn = self.Y.cols_view(0, self.m0)
        if self._sharded():
            r0, r1 = self._row_block()
            self.Y.zero_()   # the whole buffer is summed (columns past M0 stay zero)
            Yn.rows_view(r0, r1).copy_from(self.W1.cols_view(0, self.m0).rows_view(r0, r1))
            self._sum_reduce(self.Y.t)
        else:
            Yn.copy_from(self.W1.cols_view(0, self.m0))

    def _fill_random_y(self):
        nm = self.n * self._m0_init
        self.dev.splitmix(self.seed, 0, nm, self.Y)

    def _pass_spec(self, contour, points):
        """The pass's quadrature terms in accumulation order (kernel.py:350-364):
        [(z, adjoint, variant, w, theta)]."""
        spec = []
        for k in points:
            z = complex(contour.z[k])
            for adj in ((False, True) if self.hermitian else (False,)):
                variant = (2 if adj else 1) if self.hermitian else 0
                spec.append((z, adj, variant, contour.weights[k], contour.theta[k]))
        return spec

    def _pass_terms(self, spec):
        """[(variant, w, theta, X)] for every solve of this pass when the ops
        hold all of them on the device (else None: per-point path)."""
        if self._pass_result is None or not 0 < len(spec) <= 64:
            return None
        terms = []
        for z, adj, variant, w, theta in spec:
            X = self._pass_result(z, adj)
            if X is None:
                return None
            terms.append((variant, w, theta, X))
        return terms

    def _accumulate(self, weight, radius, theta, adjoint=False):
        m0 = self.m0
        variant = (2 if adjoint else 1) if self.hermitian else 0
        self.dev.accumulate(variant, self.W2.cols_view(0, m0), self.Q.cols_view(0, m0),
                            weight, radius, theta)

    def _run(self):
        dev, fpm = self.dev, self.fpm
        emin, emax, n = self.emin, self.emax, self.n
        tol = self._tolerance()
        max_loop = fpm.slot(4)
        contour = build_contour(gauss_legendre(fpm.slot(2)), emin, emax)
        scale = max(abs(emin), abs(emax))
        verbose = fpm.slot(1) == 1
        points = range(len(contour)) if self._points is None else self._points
        if verbose:
            self._print_header()

        if fpm.slot(5) == 1:
            yield from self._multiply_blocks(RciTask.MULTIPLY_B)
            self._next_rhs()
        else:
            self._fill_random_y()

        trace_prev = None
        self.loop = 0
        self.history = []     # the fpm(1) report lines: (loop, #eig, trace, error-trace, max-residual)
        while True:
            m0 = self.m0
            Q = self.Q.cols_view(0, m0)
            Q.zero_()
            self.solve_fused = False
            spec = self._pass_spec(contour, points)
            if self._solve_pass_acc is not None and self._solve_pass_acc(
                    self.Y.cols_view(0, m0), spec, contour.radius, Q):
                # solves, spike correction and all quadrature terms of the pass
                # in one device call (banded path)
                self.solve_fused = True
            elif self._solve_pass is not None:
                self._solve_pass(self.Y.cols_view(0, m0), self.hermitian)
                terms = self._pass_terms(spec)
                if terms is not None:
                    # every point's quadrature term in one sweep over Q, same
                    # order and arithmetic as the per-point accumulations below
                    dev.accumulate_terms(terms, contour.radius, Q)
                    self.solve_fused = True
            for k in points:
                self.ze = complex(contour.z[k])
                yield RciTask.FACTORIZE
                if self.hermitian and not self.adjoint_capable:
                    yield RciTask.FACTORIZE_ADJOINT
                if self.solve_fused:
                    # the pass's solves and their accumulation are done; the
                    # SOLVE tasks keep the RCI grammar (the pump skips them)
                    yield RciTask.SOLVE
                    if self.hermitian:
                        yield RciTask.SOLVE_ADJOINT
                    continue
                self.W2.cols_view(0, m0).copy_from(self.Y.cols_view(0, m0))
                yield RciTask.SOLVE
                self._accumulate(contour.weights[k], contour.radius, contour.theta[k], False)
                if self.hermitian:
                    self.W2.cols_view(0, m0).copy_from(self.Y.cols_view(0, m0))
                    yield RciTask.SOLVE_ADJOINT
                    self._accumulate(contour.weights[k], contour.radius, contour.theta[k], True)
            if self._flag_reduce is not None:
                # a rank that failed inside this pass reports through the pump
                # (run_rci) with the same collective: all ranks leave together
                code = self._flag_reduce(0)
                if code:
                    self.info = code
                    if verbose:
                        self._print_trailer()
                    return
            if self._q_reduce is not None:
                self._q_reduce(Q)

            if fpm.slot(14) == 1:
                self.X.cols_view(0, m0).copy_from(Q)
                self.epsout = 1.0
                self.info = 4
                if verbose:
                    print("==>Subspace returned after one contour (fpm(14)=1)")
                    self._print_trailer()
                return

            X = self.X.cols_view(0, m0)
            X.copy_from(Q)
            yield from self._multiply_blocks(RciTask.MULTIPLY_A)
            AP = self.AP.cols_view(0, m0)
            AP.copy_from(self.W1.cols_view(0, m0))
            yield from self._multiply_blocks(RciTask.MULTIPLY_B)
            W1 = self.W1.cols_view(0, m0)
            AQ = self.AQ.cols_view(0, m0).rows_view(0, m0)
            BQ = self.BQ.cols_view(0, m0).rows_view(0, m0)
            r0, r1 = self._row_block()
            sharded = self._sharded()
            # row block of this rank (the whole matrix on one GPU): A*Q and B*Q
            # hold valid rows r0..r1 only when the ops shard the multiplies
            Qb, APb, W1b = Q.rows_view(r0, r1), AP.rows_view(r0, r1), W1.rows_view(r0, r1)
            if sharded:
                self.AQ.zero_()   # the whole buffers are summed
                self.BQ.zero_()
            dev.gemm("C", "N", m0, m0, r1 - r0, 1.0, Qb, APb, 0.0, AQ)
            dev.gemm("C", "N", m0, m0, r1 - r0, 1.0, Qb, W1b, 0.0, BQ)
            if sharded:
                # one all-reduce of the two reduced matrices (2 * M0^2 entries)
                self._sum_reduce(self.AQ.t)
                self._sum_reduce(self.BQ.t)
            dev.symmetrize(AQ)
            dev.symmetrize(BQ)

            # shrink the subspace while the projected B fails its Cholesky
            # (kernel.py:385-400).  The reduced solve starts with that same
            # Cholesky and reports its 1-based failing pivot, so the check and
            # the solve are one launch; a failure shrinks M0 and retries.
            st = 0
            while m0 > 0:
                st = dev.reduced_eig(self.AQ, self.BQ, m0, self.e_dev.data_ptr(), self.PHI)
                if st <= 0:
                    break
                m0 = st - 1
            if m0 == 0:
                self.info = -3
                if verbose:
                    self._print_trailer()
                return
            if m0 < self.m0:
                self.X.cols_view(m0, self.m0).zero_()
                self.e[m0:] = 0
                self.res[m0:] = 0
                self.m0 = m0
                Q = Q.cols_view(0, m0)
                AP = AP.cols_view(0, m0)
                W1 = W1.cols_view(0, m0)
                X = X.cols_view(0, m0)
            if st != 0:
                self.info = -3
                if verbose:
                    self._print_trailer()
                return
            PHI = self.PHI.cols_view(0, m0).rows_view(0, m0)
            dev.gemm("N", "N", n, m0, m0, 1.0, Q, PHI, 0.0, X)
            AX = self.AX.cols_view(0, m0)
            BX = self.BX.cols_view(0, m0)
            AXb, BXb = AX.rows_view(r0, r1), BX.rows_view(r0, r1)
            dev.gemm("N", "N", r1 - r0, m0, m0, 1.0, AP.rows_view(r0, r1), PHI, 0.0, AXb)
            dev.gemm("N", "N", r1 - r0, m0, m0, 1.0, W1.rows_view(r0, r1), PHI, 0.0, BXb)
            if sharded:
                sums = self._res_sums[:2 * m0]
                dev.residual_sums(AXb, BXb, self.e_dev.data_ptr(), scale, sums.data_ptr())
                self._sum_reduce(sums)
                num, den = sums[0::2], sums[1::2]
                self.res_dev[:m0] = dev.torch.where(den > 0, num / den, dev.torch.full_like(num, float("inf")))
            else:
                dev.residuals(AX, BX, self.e_dev.data_ptr(), scale, self.res_dev.data_ptr())
            lam = self.e_dev[:m0].cpu().numpy()
            res = self.res_dev[:m0].cpu().numpy()
            self.e[:m0] = lam
            self.res[:m0] = res
            inside = (lam >= emin) & (lam <= emax)
            m = int(inside.sum())
            trace_cur = float(lam[inside].sum())
            self.epsout = 1.0 if trace_prev is None else trace_error(trace_cur, trace_prev, emin, emax)
            max_res = float(res[inside].max()) if m else 0.0
            self.history.append((self.loop, m, trace_cur, float(self.epsout), max_res))
            if verbose:
                print(f"{self.loop:<8d}{m:<7d}{trace_cur:.15e}  "
                      f"{self.epsout:.15e}  {max_res:.15e}")
            if m == 0:
                self._finalize(1, verbose, tol)
                return
            converged = (self.epsout < tol) if fpm.slot(6) == 0 else (max_res < tol)
            saturated = m == m0 and m0 < n
            if converged:
                if verbose and not saturated:
                    print("==>FEAST has successfully converged (to desired tolerance)")
                self._finalize(3 if saturated else 0, verbose, tol)
                return
            if self.loop >= max_loop:
                self._finalize(3 if saturated else 2, verbose, tol)
                return
            trace_prev = trace_cur
            self.loop += 1
            yield from self._multiply_blocks(RciTask.MULTIPLY_B)
            self._next_rhs()

    def _finalize(self, info, verbose, tol):
        """kernel.py:446-466: spurious flagging, then filter_sort_flag ordering;
        the eigenvector columns are permuted on the device."""
        m0 = self.m0
        lam = self.e[:m0]
        res = self.res[:m0]
        inside = (lam >= self.emin) & (lam <= self.emax) & np.isfinite(res) & (res >= 0)
        if inside.any():
            threshold = max(100.0 * float(np.median(res[inside])), tol * 1.0e4)
            res[inside & (res > threshold)] = -1.0
        order, m, nsp = _ordering(lam, res, self.emin, self.emax)
        lam[:] = lam[order]
        res[:] = res[order]
        if nsp:
            res[m0 - nsp:] = -1.0
        if not np.array_equal(order, np.arange(m0)):
            torch = self.dev.torch
            idx = torch.as_tensor(order, device=self.dev.tdev)
            X = self.X.cols_view(0, m0)
            for k in range(2 if self.hermitian else 1):
                pl = X.plane(k)
                pl.copy_(pl.index_select(1, idx))
        self.m = m
        self.info = info
        if verbose:
            if info == 1:
                print("==>WARNING: no eigenvalue has been found in the search interval")
            elif info == 2:
                print("==>WARNING: no convergence within the refinement loop budget")
            elif info == 3:
                print("==>WARNING: subspace size M0 is too small (M0<=M)")
            self._print_trailer()

    # -- runtime report (kernel.py:470-487) -------------------------------------
    def _print_header(self):
        print("***********************************************")
        print("*********** FEAST- BEGIN **********************")
        print("***********************************************")
        print(f"Routine {self.routine_name}")
        print("List of input parameters fpm(1:64)-- if different from default")
        for i, v in self.fpm.nondefault_slots():
            if i in (24, 25):
                continue
            print(f"   fpm({i})={v}")
        print(f"Search interval [{self.emin:.15e}; {self.emax:.15e}]")
        print(f"Size subspace {self.m0:3d}")
        print("#Loop | #Eig |     Trace           |    Error-Trace       |   Max-Residual")

    def _print_trailer(self):
        print("***********************************************")
        print("*********** FEAST- END*************************")
        print("***********************************************")


class SymmetricRci(_RciKernel):
    """Real symmetric pencils (kernel.py:490-503)."""

    hermitian = False

    def __init__(self, n, m0, emin, emax, fpm=None, **kwargs):
        kwargs.pop("adjoint_capable", None)
        super().__init__(n, m0, emin, emax, fpm, **kwargs)


class HermitianRci(_RciKernel):
    """Complex Hermitian pencils (kernel.py:506-531); SOLVE_ADJOINT is served
    from the FACTORIZE factorization unless ``adjoint_capable=False``."""

    hermitian = True

    def __init__(self, n, m0, emin, emax, fpm=None, *, adjoint_capable=True, **kwargs):
        kwargs.setdefault("dtype", np.complex128)
        super().__init__(n, m0, emin, emax, fpm, adjoint_capable=adjoint_capable, **kwargs)
