"""Device plumbing: one C-ABI context per GPU, planar device matrices.

PyTorch only owns device memory and the stream here; every arithmetic
operation is a call into libfeastb200.so.  Complex matrices are stored
PLANAR: a float64 tensor of shape (2, rows, ld) (plane 0 = real part).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from ._errors import SingularMatrixError

_P = ctypes.c_void_p


def _torch():
    import torch
    return torch


class Planar:
    """View of a row-major FP64 matrix on the device (real or planar complex)."""

    __slots__ = ("t", "cplx", "rows", "cols", "ld", "off")

    def __init__(self, t, cplx, rows, cols, ld, off=0):
        self.t, self.cplx, self.rows, self.cols, self.ld, self.off = t, cplx, rows, cols, ld, off

    @property
    def re(self):
        return self.t.data_ptr() + 8 * self.off

    @property
    def im(self):
        if not self.cplx:
            return None
        return self.t[1].data_ptr() + 8 * self.off

    def cols_view(self, c0, c1):
        return Planar(self.t, self.cplx, self.rows, c1 - c0, self.ld, self.off + c0)

    def rows_view(self, r0, r1):
        return Planar(self.t, self.cplx, r1 - r0, self.cols, self.ld, self.off + r0 * self.ld)

    def plane(self, k):
        """torch view (rows, cols) of plane k (0 = real)."""
        base = self.t[k] if self.cplx else self.t
        flat = base.reshape(-1)
        return flat[self.off:self.off + (self.rows - 1) * self.ld + self.cols].as_strided(
            (self.rows, self.cols), (self.ld, 1))

    def zero_(self):
        self.plane(0).zero_()
        if self.cplx:
            self.plane(1).zero_()

    def copy_from(self, other: "Planar"):
        """self <- other (real -> complex zero-fills the imaginary plane)."""
        self.plane(0).copy_(other.plane(0))
        if self.cplx:
            if other.cplx:
                self.plane(1).copy_(other.plane(1))
            else:
                self.plane(1).zero_()


class Device:
    """A libfeastb200 context bound to one CUDA device and torch's stream."""

    def __init__(self, index=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise _lib.FeastB200Unavailable("no CUDA device visible; the B200 build has no CPU fallback")
        self.lib = _lib.load()
        self.index = torch.cuda.current_device() if index is None else int(index)
        self.torch = torch
        self.tdev = torch.device("cuda", self.index)
        h = _P()
        stream = torch.cuda.current_stream(self.tdev).cuda_stream
        rc = self.lib.fb_ctx_create(self.index, _P(stream), ctypes.byref(h))
        if rc != 0:
            raise MemoryError("fb_ctx_create failed") if rc == -1 else RuntimeError(f"fb_ctx_create rc={rc}")
        self.h = h
        self._stream = stream
        self._info = ctypes.c_int(0)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.fb_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # -- plumbing ----------------------------------------------------------
    def bind_stream(self):
        s = self.torch.cuda.current_stream(self.tdev).cuda_stream
        if s != self._stream:
            self.lib.fb_ctx_set_stream(self.h, _P(s))
            self._stream = s

    def check(self, rc, what=""):
        if rc == 0:
            return
        msg = (self.lib.fb_ctx_last_error(self.h) or b"").decode()
        if rc == _lib.FB_ERR_ALLOC:
            raise MemoryError(f"{what}: {msg}")
        if rc == _lib.FB_ERR_SINGULAR:
            raise SingularMatrixError(f"{what}: zero pivot")
        raise RuntimeError(f"libfeastb200 {what} failed (rc={rc}): {msg}")

    def launches(self):
        return int(self.lib.fb_ctx_launch_count(self.h))

    def synchronize(self):
        self.check(self.lib.fb_ctx_synchronize(self.h), "synchronize")

    def empty(self, rows, cols, cplx, ld=None):
        ld = cols if ld is None else ld
        shape = (2, rows, ld) if cplx else (rows, ld)
        t = self.torch.empty(shape, dtype=self.torch.float64, device=self.tdev)
        return Planar(t, cplx, rows, cols, ld)

    def zeros(self, rows, cols, cplx, ld=None):
        p = self.empty(rows, cols, cplx, ld)
        p.t.zero_()
        return p

    def upload(self, arr, cplx=None, ld=None, out=None):
        """numpy (rows, cols) real or complex -> Planar."""
        arr = np.asarray(arr)
        if arr.ndim == 1:
            arr = arr[:, None]
        rows, cols = arr.shape
        is_c = np.iscomplexobj(arr)
        cplx = is_c if cplx is None else cplx
        dst = out if out is not None else self.empty(rows, cols, cplx, ld)
        torch = self.torch
        if is_c and cplx:
            host = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.complex128).view(np.float64))
            tmp = host.to(self.tdev, non_blocking=False)
            self.check(self.lib.fb_pack(self.h, rows, cols, _P(tmp.data_ptr()), cols, _P(dst.re),
                                        _P(dst.im), dst.ld, 1), "pack")
        else:
            src = np.ascontiguousarray(arr.real if is_c else arr, dtype=np.float64)
            dst.plane(0).copy_(torch.from_numpy(src))
            if cplx:
                dst.plane(1).zero_()
        return dst

    def upload_torch(self, t, cplx=None, ld=None, out=None):
        """torch tensor (real float64 or complex128, any device) -> Planar."""
        torch = self.torch
        t = t.to(self.tdev)
        is_c = t.is_complex()
        rows, cols = t.shape
        cplx = is_c if cplx is None else cplx
        dst = out if out is not None else self.empty(rows, cols, cplx, ld)
        if is_c and cplx:
            src = torch.view_as_real(t.to(torch.complex128).contiguous())
            self.check(self.lib.fb_pack(self.h, rows, cols, _P(src.data_ptr()), cols, _P(dst.re),
                                        _P(dst.im), dst.ld, 1), "pack")
        else:
            dst.plane(0).copy_(t.real if is_c else t.to(torch.float64))
            if cplx:
                dst.plane(1).zero_()
        return dst

    _BOUNCE = 32 << 20  # bytes per pinned bounce buffer

    def _d2h(self, t):
        """Device tensor -> new numpy array.  Large arrays go through two
        pinned bounce buffers (D2H of chunk k overlaps the host copy of k-1)
        instead of torch's pageable copy."""
        torch = self.torch
        t = t.contiguous()
        nbytes = t.numel() * t.element_size()
        if nbytes <= (8 << 20):
            return t.cpu().numpy()
        if getattr(self, "_pins", None) is None:
            self._pins = [torch.empty(self._BOUNCE, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
            self._pin_ev = [torch.cuda.Event() for _ in range(2)]
        npdt = {torch.float64: np.float64, torch.float32: np.float32, torch.int32: np.int32,
                torch.int64: np.int64}.get(t.dtype)
        if npdt is None:
            return t.cpu().numpy()
        out = np.empty(tuple(t.shape), dtype=npdt)
        src = t.view(-1).view(torch.uint8)
        dst = out.reshape(-1).view(np.uint8)
        pool = self._copy_pool()
        nth = pool._max_workers

        def host_copy(pbuf, poff, pn):
            # first touch of the fresh destination pages dominates: split the
            # pinned -> pageable copy over threads (numpy releases the GIL)
            step = -(-pn // nth)
            hb = pbuf[:pn].numpy()
            futs = [pool.submit(np.copyto, dst[poff + a:poff + min(pn, a + step)], hb[a:min(pn, a + step)])
                    for a in range(0, pn, step)]
            for f in futs:
                f.result()

        prev = None
        for k, off in enumerate(range(0, nbytes, self._BOUNCE)):
            n = min(self._BOUNCE, nbytes - off)
            buf, ev = self._pins[k % 2], self._pin_ev[k % 2]
            buf[:n].copy_(src[off:off + n], non_blocking=True)
            ev.record()
            if prev is not None:
                pbuf, pev, poff, pn = prev
                pev.synchronize()
                host_copy(pbuf, poff, pn)
            prev = (buf, ev, off, n)
        pbuf, pev, poff, pn = prev
        pev.synchronize()
        host_copy(pbuf, poff, pn)
        return out

    def _copy_pool(self):
        if getattr(self, "_pool", None) is None:
            import concurrent.futures
            self._pool = concurrent.futures.ThreadPoolExecutor(
                max_workers=max(1, min(8, len(os.sched_getaffinity(0)))))
        return self._pool

    def download(self, p: Planar, as_complex=None):
        """Planar -> numpy (complex128 when the view is complex)."""
        as_complex = p.cplx if as_complex is None else as_complex
        torch = self.torch
        if p.cplx:
            tmp = torch.empty((p.rows, p.cols, 2), dtype=torch.float64, device=self.tdev)
            self.check(self.lib.fb_pack(self.h, p.rows, p.cols, _P(tmp.data_ptr()), p.cols, _P(p.re),
                                        _P(p.im), p.ld, 0), "unpack")
            out = self._d2h(tmp).view(np.complex128).reshape(p.rows, p.cols)
            return out if as_complex else out.real.copy()
        out = self._d2h(p.plane(0))
        return out.astype(np.complex128) if as_complex else out

    # -- arithmetic (each is one C-ABI call) -------------------------------
    def gemm(self, opa, opb, m, n, k, alpha, A: Planar, B: Planar, beta, C: Planar, cplx=None):
        cplx = C.cplx if cplx is None else cplx
        alpha, beta = complex(alpha), complex(beta)
        rc = self.lib.fb_gemm(self.h, 1 if cplx else 0, opa.encode(), opb.encode(), m, n, k,
                              alpha.real, alpha.imag, _P(A.re), _P(A.im), A.ld, _P(B.re), _P(B.im),
                              B.ld, beta.real, beta.imag, _P(C.re), _P(C.im), C.ld)
        self.check(rc, "gemm")

    def splitmix(self, seed, off_re, off_im, out: Planar):
        rc = self.lib.fb_splitmix(self.h, ctypes.c_uint64(seed % (1 << 64)), off_re,
                                  off_im if out.cplx else 0, out.rows, out.cols, _P(out.re),
                                  _P(out.im), out.ld)
        self.check(rc, "splitmix")

    def accumulate(self, variant, X: Planar, Q: Planar, w, r, theta):
        rc = self.lib.fb_accumulate(self.h, variant, X.rows, X.cols, _P(X.re), _P(X.im), X.ld,
                                    _P(Q.re), _P(Q.im), Q.ld, float(w), float(r), float(theta))
        self.check(rc, "accumulate")

    def accumulate_terms(self, terms, radius, Q: Planar):
        """terms: [(variant, weight, theta, X: Planar)] in accumulation order."""
        k = len(terms)
        if k == 0:
            return
        ldx = terms[0][3].ld
        if any(t[3].ld != ldx for t in terms):
            raise ValueError("accumulate_terms: solve results must share one leading dimension")
        var = (ctypes.c_int * k)(*[int(t[0]) for t in terms])
        w = (ctypes.c_double * k)(*[float(t[1]) for t in terms])
        th = (ctypes.c_double * k)(*[float(t[2]) for t in terms])
        xr = (ctypes.c_void_p * k)(*[t[3].re for t in terms])
        xi = (ctypes.c_void_p * k)(*[t[3].im for t in terms])
        rc = self.lib.fb_accumulate_terms(self.h, k, var, w, float(radius), th, xr, xi, Q.rows, Q.cols, ldx,
                                          _P(Q.re), _P(Q.im), Q.ld)
        self.check(rc, "accumulate_terms")

    def symmetrize(self, M: Planar):
        self.check(self.lib.fb_symmetrize(self.h, M.rows, _P(M.re), _P(M.im), M.ld), "symmetrize")

    def residuals(self, AX: Planar, BX: Planar, lam_ptr, scale, res_ptr):
        rc = self.lib.fb_residuals(self.h, AX.rows, AX.cols, _P(AX.re), _P(AX.im), _P(BX.re),
                                   _P(BX.im), AX.ld, _P(lam_ptr), float(scale), _P(res_ptr))
        self.check(rc, "residuals")

    def residual_sums(self, AX: Planar, BX: Planar, lam_ptr, scale, sums_ptr):
        """(numerator, denominator) sums of the residuals over the rows of AX/BX
        (a row block of the multi-GPU path), interleaved per column."""
        rc = self.lib.fb_residual_sums(self.h, AX.rows, AX.cols, _P(AX.re), _P(AX.im), _P(BX.re),
                                       _P(BX.im), AX.ld, _P(lam_ptr), float(scale), _P(sums_ptr))
        self.check(rc, "residual_sums")

    def chol_check(self, Bq: Planar, m):
        fail = ctypes.c_int(0)
        rc = self.lib.fb_chol_check(self.h, m, _P(Bq.re), _P(Bq.im), Bq.ld, ctypes.byref(fail))
        self.check(rc, "chol_check")
        return fail.value

    def reduced_eig(self, Aq: Planar, Bq: Planar, m, eps_ptr, Phi: Planar):
        st = ctypes.c_int(0)
        rc = self.lib.fb_reduced_eig(self.h, m, _P(Aq.re), _P(Aq.im), _P(Bq.re), _P(Bq.im), Aq.ld,
                                     _P(eps_ptr), _P(Phi.re), _P(Phi.im), Phi.ld, ctypes.byref(st))
        if rc not in (0, _lib.FB_ERR_REDUCED):
            self.check(rc, "reduced_eig")
        return st.value

    def read_info(self, info_ptr):
        bad = ctypes.c_int(-1)
        rc = self.lib.fb_read_info(self.h, _P(info_ptr), ctypes.byref(bad))
        if rc not in (0, _lib.FB_ERR_SINGULAR):
            self.check(rc, "read_info")
        return bad.value


_DEVICES = {}


def get_device(index=None) -> Device:
    torch = _torch()
    if not torch.cuda.is_available():
        raise _lib.FeastB200Unavailable("no CUDA device visible; the B200 build has no CPU fallback")
    idx = torch.cuda.current_device() if index is None else int(index)
    dev = _DEVICES.get(idx)
    if dev is None:
        with torch.cuda.device(idx):
            dev = Device(idx)
        _DEVICES[idx] = dev
    dev.bind_stream()
    return dev
