"""Wire/disk formats of the reference tooling, host-side only.

* residual-history CSV ``iter,relres`` -- write_history_csv (stk/report.hpp:22-26); values
  printed like a default ``std::ostream`` (``%g``, 6 significant digits);
* result-table CSV ``method,N_h,N_t,iters,mu_mem,rank,time_s,relres,err_oracle`` --
  ResultRow / result_csv_header / to_csv / write_result_csv (stk/bench.hpp:210-242), same
  printf formats, optional ``err_oracle`` left empty, ``stable_time`` zeroes time_s;
* MatrixMarket coordinate text -- write_matrix_market / read_matrix_market
  (stk/matrix_market.hpp:16-80): 1-based indices, column-major entry order, symmetric
  matrices store the lower triangle, values with 17 significant digits; the reader accepts
  ``general|symmetric`` real coordinate files, skips ``%`` comment lines, mirrors symmetric
  off-diagonal entries and rejects duplicates / truncated lists with ArgumentError.

Sparse matrices are exchanged as :class:`SparseTriplets`; helpers convert the banded
factors this package uses (Tridiagonal, Band7) and the bidiagonal time factors.
"""
from __future__ import annotations

import io
import os
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from .errors import ArgumentError


# ------------------------------------------------------------------- history CSV ---
def _g(x: float) -> str:
    """Default std::ostream formatting of a double (precision 6, %g)."""
    s = format(float(x), ".6g")
    if s in ("inf", "-inf"):
        return s
    if s == "nan":
        return "nan"
    return s


def write_history_csv(out, report) -> None:
    """write_history_csv (stk/report.hpp:22-26): header ``iter,relres``, iterations 1-based."""
    hist = report.rel_res_history if hasattr(report, "rel_res_history") else report
    lines = ["iter,relres"] + [f"{i + 1},{_g(v)}" for i, v in enumerate(hist)]
    _emit(out, "\n".join(lines) + "\n")


# -------------------------------------------------------------------- result CSV ---
@dataclass
class ResultRow:
    """One table line per (method, N_h, N_t) run (stk/bench.hpp:210-218)."""
    method: str
    n_h: int = 0
    n_t: int = 0
    iters: int = 0
    mu_mem: int = 0
    rank: int = 0
    time_s: float = 0.0
    relres: float = 0.0
    err_oracle: float | None = None
    converged: bool = True


def result_csv_header() -> str:
    return "method,N_h,N_t,iters,mu_mem,rank,time_s,relres,err_oracle"


def to_csv(row: ResultRow, stable_time: bool = False) -> str:
    """to_csv (stk/bench.hpp:224-236): ``%s,%lld,%lld,%d,%d,%d,%.4f,%.6e,`` + ``%.6e``."""
    out = "%s,%d,%d,%d,%d,%d,%.4f,%.6e," % (row.method, row.n_h, row.n_t, row.iters,
                                           row.mu_mem, row.rank,
                                           0.0 if stable_time else row.time_s, row.relres)
    if row.err_oracle is not None:
        out += "%.6e" % row.err_oracle
    return out


def write_result_csv(out, rows: Iterable[ResultRow], stable_time: bool = False) -> None:
    lines = [result_csv_header()] + [to_csv(r, stable_time) for r in rows]
    _emit(out, "\n".join(lines) + "\n")


# ------------------------------------------------------------------ MatrixMarket ---
@dataclass
class SparseTriplets:
    """A sparse matrix as 0-based (row, col, value) entries; ``symmetric`` flags a matrix
    whose full entry set is stored (the writer keeps only the lower triangle)."""
    rows: int
    cols: int
    entries: list = field(default_factory=list)
    symmetric: bool = False

    def dense(self) -> np.ndarray:
        a = np.zeros((self.rows, self.cols))
        for i, j, v in self.entries:
            a[i, j] += v
        return a


def write_matrix_market(out, m: SparseTriplets) -> None:
    """write_matrix_market (stk/matrix_market.hpp:16-30)."""
    ents = sorted(((j, i, v) for i, j, v in m.entries if not (m.symmetric and i < j)))
    lines = ["%%MatrixMarket matrix coordinate real "
             + ("symmetric" if m.symmetric else "general"),
             f"{m.rows} {m.cols} {len(ents)}"]
    lines += [f"{i + 1} {j + 1} {format(float(v), '.17g')}" for j, i, v in ents]
    if isinstance(out, (str, os.PathLike)):
        try:
            with open(out, "w") as f:
                f.write("\n".join(lines) + "\n")
        except OSError:
            raise ArgumentError(f"write_matrix_market: cannot open {out}") from None
        return
    out.write("\n".join(lines) + "\n")


def read_matrix_market(src) -> SparseTriplets:
    """read_matrix_market (stk/matrix_market.hpp:38-74)."""
    if isinstance(src, (str, os.PathLike)):
        try:
            with open(src) as f:
                text = f.read()
        except OSError:
            raise ArgumentError(f"read_matrix_market: cannot open {src}") from None
    else:
        text = src.read()
    stream = io.StringIO(text)
    line = stream.readline()
    if not line:
        raise ArgumentError("read_matrix_market: empty input")
    line = line.rstrip("\n")
    hdr = line.split()
    hdr += [""] * (5 - len(hdr))
    banner, obj, fmt, fld, sym = hdr[:5]
    if (banner != "%%MatrixMarket" or obj != "matrix" or fmt != "coordinate" or fld != "real"
            or sym not in ("general", "symmetric")):
        raise ArgumentError("read_matrix_market: unsupported header: " + line)
    symmetric = sym == "symmetric"
    size_line = ""
    for raw in stream:
        raw = raw.rstrip("\n")
        if raw and raw[0] != "%":
            size_line = raw
            break
    try:
        rows, cols, nnz = (int(x) for x in size_line.split()[:3])
    except ValueError:
        raise ArgumentError("read_matrix_market: bad size line") from None
    tokens = stream.read().split()
    if len(tokens) < 3 * nnz:
        raise ArgumentError("read_matrix_market: truncated entry list")
    entries, seen = [], set()
    for k in range(nnz):
        try:
            i = int(tokens[3 * k]) - 1
            j = int(tokens[3 * k + 1]) - 1
            v = float(tokens[3 * k + 2])
        except ValueError:
            raise ArgumentError("read_matrix_market: truncated entry list") from None
        if (i, j) in seen:
            raise ArgumentError("read_matrix_market: duplicate entry")
        seen.add((i, j))
        entries.append((i, j, v))
        if symmetric and i != j:
            entries.append((j, i, v))
    return SparseTriplets(rows, cols, entries, symmetric)


# ----------------------------------------------------------- banded conversions ---
def tridiagonal_triplets(t) -> SparseTriplets:
    """Symmetric tridiagonal factor (M_h / A_h, stk/discretize.hpp:61-77)."""
    d, o = np.asarray(t.diag), np.asarray(t.off)
    n = d.size
    ent = []
    for j in range(n):  # column-major order
        if j > 0:
            ent.append((j - 1, j, float(o[j - 1])))
        ent.append((j, j, float(d[j])))
        if j + 1 < n:
            ent.append((j + 1, j, float(o[j])))
    return SparseTriplets(n, n, ent, True)


def bidiagonal_triplets(b) -> SparseTriplets:
    """Upper bidiagonal time factor (D / C, stk/discretize.hpp:44-58); stored general."""
    d, s = np.asarray(b.diag), np.asarray(b.sup)
    n = d.size
    ent = []
    for j in range(n):
        if j > 0:
            ent.append((j - 1, j, float(s[j - 1])))
        ent.append((j, j, float(d[j])))
    return SparseTriplets(n, n, ent, False)


def band7_triplets(b, symmetric: bool | None = None, drop_zeros: bool = True) -> SparseTriplets:
    """7-band spline Gram factor (band[d, i] = A[i, i + d - 3]).  ``symmetric=None`` marks the
    matrix symmetric only when it is exactly mirrored: the assembled spline Gram matrices
    are symmetric only up to rounding (SURVEY F-finding on check_mirrored), and the
    symmetric MatrixMarket form would silently drop the upper-triangle values."""
    n = b.n
    band = np.asarray(b.band)
    if symmetric is None:
        dense = b.dense()
        symmetric = bool(np.array_equal(dense, dense.T))
    ent = []
    for j in range(n):
        for i in range(max(0, j - 3), min(n, j + 4)):
            v = float(band[j - i + 3, i])
            if drop_zeros and v == 0.0:
                continue
            ent.append((i, j, v))
    return SparseTriplets(n, n, ent, symmetric)


def _emit(out, text: str) -> None:
    if isinstance(out, (str, os.PathLike)):
        with open(out, "w") as f:
            f.write(text)
    else:
        out.write(text)


__all__: Sequence[str] = [
    "write_history_csv", "ResultRow", "result_csv_header", "to_csv", "write_result_csv",
    "SparseTriplets", "write_matrix_market", "read_matrix_market", "tridiagonal_triplets",
    "bidiagonal_triplets", "band7_triplets",
]
