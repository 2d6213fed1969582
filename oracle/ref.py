"""The UNMODIFIED reference package next to the oracle — TEST INFRASTRUCTURE ONLY.

``make_ref()`` copies ``/root/reference/pkg/src/feastlib`` (pure Python, no
build step) to ``oracle/_ref/feastlib``.  ``oracle/_ref/`` is git-ignored (no
reference sources in the history) but not gpurun-ignored, so the copy travels
to the GPU box, where ``/root/reference`` does not exist.  ``build()`` in
``__graft_entry__.py`` refreshes the copy whenever the reference is present.

Users: ``tests/`` (the drop-in proof: feastlib's own ``run_rci`` and RCI
kernels pumped against ``B200DenseOps`` / ``B200BandOps``) and ``bench.py``'s
``--impl reference`` / ``cpu_baseline`` legs (feastlib's kernel answered by
LAPACK ops).  The product never imports this module.
"""

from __future__ import annotations

import importlib
import os
import shutil
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src/feastlib"
REF_DST = os.path.join(_HERE, "_ref")


def make_ref(force=False):
    """Copy the reference package into oracle/_ref (no-op without /root/reference)."""
    if not os.path.isdir(REF_SRC):
        return os.path.isdir(os.path.join(REF_DST, "feastlib"))
    dst = os.path.join(REF_DST, "feastlib")
    if os.path.isdir(dst):
        if not force and all(
                os.path.exists(os.path.join(dst, f)) and
                os.path.getmtime(os.path.join(dst, f)) >= os.path.getmtime(os.path.join(REF_SRC, f))
                for f in os.listdir(REF_SRC) if f.endswith(".py")):
            return True
        shutil.rmtree(dst)
    os.makedirs(REF_DST, exist_ok=True)
    shutil.copytree(REF_SRC, dst, ignore=shutil.ignore_patterns("__pycache__"))
    return True


def available():
    return os.path.isfile(os.path.join(REF_DST, "feastlib", "__init__.py"))


def load_feastlib():
    """Import the reference package from oracle/_ref (raises ImportError if absent)."""
    if not available():
        raise ImportError("oracle/_ref/feastlib is missing: run oracle.ref.make_ref() where "
                          "/root/reference exists (python __graft_entry__.py build)")
    if REF_DST not in sys.path:
        sys.path.insert(0, REF_DST)
    return importlib.import_module("feastlib")


def reference_solve(w, ops=None, fpm=None, options=None):
    """feastlib's own kernel (SymmetricRci / HermitianRci) pumped by feastlib's
    own run_rci for a ``workloads.Workload``; ``ops`` defaults to the LAPACK
    ops of the oracle (zgetrf/zgetrs, zgbtrf/zgbtrs), i.e. the "reference
    kernel + LAPACK caller" of SURVEY.md §8(c)."""
    fl = load_feastlib()
    from feastlib import _driver as fdriver
    from feastlib import banded as fband
    from .feast_oracle import LapackBandOps, LapackDenseOps
    cls = fl.HermitianRci if w.hermitian else fl.SymmetricRci
    if fpm is None:
        fpm = fl.feastinit()
        fpm.set_slot(2, w.ne)
    k = cls(w.n, w.m0, w.emin, w.emax, fpm)
    if ops is None:
        if w.kind == "dense":
            ops = LapackDenseOps(w.a, w.b)
        else:
            kl = max(w.kla, w.klb)
            fa = fband._pad_band(fband.expand_band(w.a, w.kla, w.uplo, w.hermitian), w.kla, kl)
            fbm = None if w.b is None else fband._pad_band(
                fband.expand_band(w.b, w.klb, w.uplo, w.hermitian), w.klb, kl)
            ops = LapackBandOps(fa, fbm, kl)
    return fdriver.run_rci(k, ops, options)


def shipped_solve(w, fpm=None):
    """The reference exactly as published: feast_sy / feast_he / feast_sb / feast_hb
    with its own pure-Python LU (BASELINE.md §4 "shipped reference path")."""
    fl = load_feastlib()
    if fpm is None:
        fpm = fl.feastinit()
        fpm.set_slot(2, w.ne)
    if w.kind == "dense":
        fn = fl.feast_he if w.hermitian else fl.feast_sy
        return fn(w.a, w.emin, w.emax, w.m0, b=w.b, fpm=fpm)
    fn = fl.feast_hb if w.hermitian else fl.feast_sb
    return fn(w.a, w.kla, w.emin, w.emax, w.m0, b=w.b, klb=w.klb, uplo=w.uplo, fpm=fpm)


if __name__ == "__main__":
    print("oracle/_ref ready" if make_ref(force="--force" in sys.argv) else "reference not present")
