"""Utility-driver file formats (host plumbing in front of the GPU drivers).

Same formats and error behaviour as feastlib's io.py (io.py:1-230):

* coordinate matrix files ``<name>.A`` / ``<name>.B``: header ``N N NNZ``,
  then NNZ triplets ``i j value`` (real) or ``i j re im`` (complex), 1-based,
  ``!`` starts a comment, duplicates are kept in the triplet list and summed
  when the matrix is assembled;
* the ``<name>.in`` configuration: fixed-order value lines (problem kind s/g,
  precision s/d/c/z, UPLO, Emin, Emax, M0), then up to five fpm overrides
  (print flag, contour points, tolerance exponent -- fpm(3) for d/z, fpm(7)
  for s/c --, loop budget, convergence criterion).

Assembly targets the two storage schemes the B200 build solves: a dense
matrix for feast_sy/feast_he and the full band layout (2kl+1 rows, row kl+s
the s-th subdiagonal) for feast_sb/feast_hb.  The reference's CSR backend is
out of scope here, so the triplets are assembled straight into
those layouts, with the reference's rules: indices checked against 1..N,
'L'/'U' files may only hold their triangle, duplicates summed in file order,
the other triangle mirrored (conjugated for complex input) -- the values of
CsrMatrix.from_coo(...).to_dense() / .to_banded() (sparse.py:68-134).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .params import FeastParams, feastinit


class ParseError(ValueError):
    """Malformed input file; ``line`` is the offending 1-based line (or None)."""

    def __init__(self, message, line=None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


def _value_lines(text):
    """(1-based line number, tokens) of every line with content before '!'."""
    for no, line in enumerate(text.splitlines(), 1):
        body = line.partition("!")[0].split()
        if body:
            yield no, body


def _real(tok, no):
    try:   # Fortran exponents (1.0d-3) are accepted
        return float(tok.replace("d", "e").replace("D", "e"))
    except ValueError:
        raise ParseError(f"expected a real number, got {tok!r}", no) from None


def _int(tok, no):
    try:
        return int(tok)
    except ValueError:
        raise ParseError(f"expected an integer, got {tok!r}", no) from None


@dataclass
class CooMatrix:
    """Coordinate triplets as read (1-based, duplicates preserved)."""

    n: int
    nnz: int
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray

    def _checked(self, uplo):
        uplo = uplo.upper()
        r, c = self.rows, self.cols
        if self.nnz and (r.min() < 1 or r.max() > self.n or c.min() < 1 or c.max() > self.n):
            raise ValueError("coordinate index out of range 1..n")
        if uplo == "L" and np.any(c > r):
            raise ValueError("uplo='L' triplet above the diagonal")
        if uplo == "U" and np.any(c < r):
            raise ValueError("uplo='U' triplet below the diagonal")
        return uplo

    def to_dense(self, uplo="F", dtype=None) -> np.ndarray:
        """Assembled n x n matrix, the stored triangle mirrored for 'L'/'U'."""
        uplo = self._checked(uplo)
        vals = self.values if dtype is None else self.values.astype(dtype)
        out = np.zeros((self.n, self.n), dtype=vals.dtype)
        r, c = self.rows - 1, self.cols - 1
        np.add.at(out, (r, c), vals)          # duplicates summed in file order
        if uplo != "F":
            lower = np.tril(out, -1) if uplo == "L" else np.triu(out, 1)
            out += lower.conj().T if np.iscomplexobj(out) else lower.T
        return out

    def to_csr(self, uplo="F", dtype=None):
        """CsrMatrix in the stored triangle, duplicates summed (io.py's
        CooMatrix.to_csr, via CsrMatrix.from_coo, sparse.py:67-89)."""
        from .sparse import CsrMatrix
        uplo = self._checked(uplo)
        vals = self.values if dtype is None else self.values.astype(dtype)
        return CsrMatrix.from_coo(self.n, self.rows, self.cols, vals, uplo)

    def to_band(self, uplo="F", dtype=None):
        """(ab, kl): full band layout ab[kl + i - j, j] = A[i, j] and its
        half-bandwidth (the widest stored offset)."""
        a = self.to_dense(uplo, dtype)
        i, j = np.nonzero(a)
        kl = int(np.abs(i - j).max()) if i.size else 0
        ab = np.zeros((2 * kl + 1, self.n), dtype=a.dtype)
        ab[kl + i - j, j] = a[i, j]
        return ab, kl


def parse_coordinate(text: str, complex_values: bool = False) -> CooMatrix:
    """Coordinate file -> CooMatrix (io.py:93-140 semantics and messages)."""
    it = _value_lines(text)
    first = next(it, None)
    if first is None:
        raise ParseError("empty coordinate file")
    no, head = first
    if len(head) != 3:
        raise ParseError(f"header must be 'N N NNZ', got {' '.join(head)!r}", no)
    n, n2, nnz = (_int(t, no) for t in head)
    if n != n2:
        raise ParseError(f"matrix must be square: {n} != {n2}", no)
    if n <= 0 or nnz < 0:
        raise ParseError(f"invalid sizes N={n} NNZ={nnz}", no)
    width = 4 if complex_values else 3
    rows = np.empty(nnz, dtype=np.int64)
    cols = np.empty(nnz, dtype=np.int64)
    vals = np.empty(nnz, dtype=np.complex128 if complex_values else np.float64)
    k = 0
    for no, toks in it:
        if k == nnz:
            raise ParseError(f"more than NNZ={nnz} entries", no)
        if len(toks) != width:
            raise ParseError(f"expected {width} fields (i j {'re im' if complex_values else 'value'}), "
                             f"got {len(toks)}", no)
        i, j = _int(toks[0], no), _int(toks[1], no)
        if not (1 <= i <= n and 1 <= j <= n):
            raise ParseError(f"index ({i},{j}) outside 1..{n}", no)
        rows[k], cols[k] = i, j
        vals[k] = complex(_real(toks[2], no), _real(toks[3], no)) if complex_values else _real(toks[2], no)
        k += 1
    if k < nnz:
        raise ParseError(f"file truncated: expected NNZ={nnz} entries, found {k}")
    return CooMatrix(n, nnz, rows, cols, vals)


def write_coordinate(coo: CooMatrix) -> str:
    cplx = np.iscomplexobj(coo.values)
    lines = [f"{coo.n} {coo.n} {coo.nnz}"]
    for i, j, v in zip(coo.rows, coo.cols, coo.values):
        lines.append(f"{i} {j} {v.real:.17g} {v.imag:.17g}" if cplx else f"{i} {j} {v:.17g}")
    return "\n".join(lines) + "\n"


@dataclass
class DriverConfig:
    """A parsed ``.in`` file."""

    problem: str = "s"
    precision: str = "d"
    uplo: str = "F"
    emin: float = 0.0
    emax: float = 0.0
    m0: int = 0
    fpm: FeastParams = field(default_factory=feastinit)

    @property
    def is_complex(self) -> bool:
        return self.precision in ("c", "z")

    @property
    def is_single(self) -> bool:
        return self.precision in ("s", "c")

    @property
    def tol_slot(self) -> int:
        return 7 if self.is_single else 3


def parse_config(text: str) -> DriverConfig:
    """``.in`` text -> DriverConfig (io.py:166-210 semantics and messages)."""
    ent = list(_value_lines(text))
    if len(ent) < 6:
        raise ParseError(f"configuration needs at least 6 value lines, found {len(ent)}")
    cfg = DriverConfig()
    choices = [("problem", ("s", "g"), str.lower, "problem kind"),
               ("precision", ("s", "d", "c", "z"), str.lower, "precision"),
               ("uplo", ("F", "L", "U"), str.upper, "UPLO")]
    for (no, toks), (attr, allowed, norm, what) in zip(ent[:3], choices):
        v = norm(toks[0])
        if v not in allowed:
            raise ParseError(f"{what} must be one of {allowed}, got {toks[0]!r}", no)
        setattr(cfg, attr, v)
    cfg.emin = _real(ent[3][1][0], ent[3][0])
    cfg.emax = _real(ent[4][1][0], ent[4][0])
    cfg.m0 = _int(ent[5][1][0], ent[5][0])
    slots = (1, 2, cfg.tol_slot, 4, 6)
    extra = ent[6:]
    if len(extra) > len(slots):
        raise ParseError(f"too many parameter override lines (at most {len(slots)})", extra[len(slots)][0])
    for (no, toks), slot in zip(extra, slots):
        cfg.fpm.set_slot(slot, _int(toks[0], no))
    return cfg


def write_config(cfg: DriverConfig) -> str:
    f = cfg.fpm
    return "\n".join([
        f"{cfg.problem} ! standard or generalized",
        f"{cfg.precision} ! scalar precision",
        f"{cfg.uplo} ! UPLO",
        f"{cfg.emin:.17g} ! Emin",
        f"{cfg.emax:.17g} ! Emax",
        f"{cfg.m0} ! M0",
        "!!!!FEASTPARAM overrides",
        f"{f.slot(1)} ! print runtime report",
        f"{f.slot(2)} ! contour points",
        f"{f.slot(cfg.tol_slot)} ! tolerance exponent",
        f"{f.slot(4)} ! max refinement loops",
        f"{f.slot(6)} ! convergence criterion (0 trace, 1 residual)",
    ]) + "\n"
