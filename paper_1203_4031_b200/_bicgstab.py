"""Iterative inner solver of the CSR drivers on the device: the reference's
diagonal-preconditioned BiCGStab (sparse.py:354-427) for every right-hand-side
column at once (fb_bicgstab, csrc/csr.cu).

The shifted matrix lives on the union pattern of A and B with aligned data
vectors (_ShiftedPattern, sparse.py:316-351); the data of z*B - A and of
its adjoint conj(z)*B - A are formed per shift, as _IterativeFactor does
(sparse.py:394-409), and stay resident for the whole solve.
"""

from __future__ import annotations

import numpy as np

from ._errors import SingularMatrixError
from .device import Planar

_FAIL = {-1: "BiCGStab breakdown (rho = 0)", -2: "BiCGStab breakdown (rhat.v = 0)",
         -3: "BiCGStab breakdown (t = 0)"}


class _ShiftedOperator:
    __slots__ = ("re", "im", "dre", "dim")


class _IterFactor:
    __slots__ = ("z", "direct", "adjoint")


class DeviceBicgstab:
    def __init__(self, dev, n, rows, cols, a_full, b_full, hermitian, tol, chunk=8, row_order=None):
        t = dev.torch
        self.row_order = row_order          # device int64 SpMM visiting order (RCM) or None
        self.dev, self.n, self.tol, self.chunk = dev, n, float(tol), chunk
        self.maxiter = max(8 * n, 200)
        keys = rows * np.int64(n) + cols
        indptr = np.zeros(n + 1, dtype=np.int64)
        indptr[1:] = np.cumsum(np.bincount(rows, minlength=n)[:n])
        self.indptr = t.from_numpy(indptr).to(dev.tdev)
        self.indices = t.from_numpy(np.ascontiguousarray(cols, dtype=np.int64)).to(dev.tdev)
        self.a_data = np.zeros(keys.size, dtype=np.complex128)
        self.b_data = np.zeros(keys.size, dtype=np.complex128)
        ra = a_full.row_of_entries()
        self.a_data[np.searchsorted(keys, ra * np.int64(n) + (a_full.ja - 1))] = a_full.values
        if b_full is None:
            d = np.arange(n, dtype=np.int64)
            self.b_data[np.searchsorted(keys, d * np.int64(n + 1))] = 1.0
        else:
            rb = b_full.row_of_entries()
            self.b_data[np.searchsorted(keys, rb * np.int64(n) + (b_full.ja - 1))] = b_full.values
        self.diag_pos = np.flatnonzero(rows == cols)
        self.diag_row = rows[self.diag_pos]
        self._ws = {}

    def _operator(self, z):
        t, dev = self.dev.torch, self.dev
        data = z * self.b_data - self.a_data
        diag = np.zeros(self.n, dtype=np.complex128)
        diag[self.diag_row] = data[self.diag_pos]
        diag[diag == 0] = 1.0
        op = _ShiftedOperator()
        op.re = t.from_numpy(np.ascontiguousarray(data.real)).to(dev.tdev)
        op.im = t.from_numpy(np.ascontiguousarray(data.imag)).to(dev.tdev)
        op.dre = t.from_numpy(np.ascontiguousarray(diag.real)).to(dev.tdev)
        op.dim = t.from_numpy(np.ascontiguousarray(diag.imag)).to(dev.tdev)
        return op

    def _order(self):
        return None if self.row_order is None else self.row_order.data_ptr()

    def factorize(self, z):
        f = _IterFactor()
        f.z = z
        f.direct = self._operator(z)
        # (z B - A)^H = conj(z) B - A for Hermitian / symmetric A, B (sparse.py:400-401)
        f.adjoint = self._operator(z.conjugate())
        return f

    def _workspace(self, m):
        ws = self._ws.get(m)
        if ws is None:
            dev, t = self.dev, self.dev.torch
            ld = m + (m & 1)
            nd = int(dev.lib.fb_bicgstab_workspace_doubles(self.n, m, ld))
            ws = (ld, t.empty(nd, dtype=t.float64, device=dev.tdev),
                  dev.empty(self.n, m, True, ld=ld),
                  t.zeros(2 * m + 2, dtype=t.int32, device=dev.tdev))
            self._ws = {m: ws}
        return ws

    def solve(self, f, W: Planar, adjoint=False):
        op = f.adjoint if adjoint else f.direct
        dev, n, m = self.dev, self.n, W.cols
        if m == 0 or n == 0:
            return
        ld, work, X, ist = self._workspace(m)
        args = (n, m, self.indptr.data_ptr(), self.indices.data_ptr(), op.re.data_ptr(), op.im.data_ptr(),
                op.dre.data_ptr(), op.dim.data_ptr(), W.re, W.im, W.ld, X.re, X.im, X.ld, self.tol,
                self.maxiter)
        dev.check(dev.lib.fb_bicgstab(dev.h, 0, *args, 0, work.data_ptr(), ld, ist.data_ptr(),
                                      self._order()), "bicgstab init")
        done, chunk = 0, self.chunk
        while True:
            # poll after 8, 16, 32, then every 64 iterations (iterations past a
            # column's convergence are no-ops, so only the poll cadence changes)
            dev.check(dev.lib.fb_bicgstab(dev.h, 1, *args, chunk, work.data_ptr(), ld, ist.data_ptr(),
                                          self._order()), "bicgstab")
            done += chunk
            chunk = min(2 * chunk, 64)
            active, fail = (int(v) for v in ist[2 * m:2 * m + 2].cpu())
            if fail:
                if fail == -4:
                    raise SingularMatrixError(
                        f"BiCGStab did not reach tol={self.tol} in {self.maxiter} iterations")
                raise SingularMatrixError(_FAIL[fail])
            if active == 0:
                break
            if done > self.maxiter + 64:              # cannot happen: maxiter fails first
                raise SingularMatrixError("BiCGStab iteration budget exceeded")
        W.copy_from(X)
