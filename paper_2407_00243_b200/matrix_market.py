"""Matrix Market coordinate I/O.

Same accepted subset and error behaviour as the reference reader
(matrix_market.cpp:21-89, matrix_market.hpp:26-59): banner
``%%MatrixMarket matrix coordinate {real|integer|pattern} {general|symmetric}``,
comments / blank lines skipped, 1-based indices, pattern entries = 1.0,
symmetric off-diagonals mirrored, duplicates summed (csr_from_triplets);
malformed input raises RuntimeError (std::runtime_error).  Writing uses
``%.17g`` so a reload reproduces the stored values exactly.
"""
from __future__ import annotations

import numpy as np

from .tilefuse import Csr

INT32_MAX = 2**31 - 1


def _fail(origin, what):
    raise RuntimeError(f"{origin}: {what}")


def parse_matrix_market(text: str, origin: str = "<string>"):
    """-> (n_rows, n_cols, rows int64, cols int64, vals float64) triplets."""
    lines = text.splitlines()
    if not lines:
        _fail(origin, "empty file")
    head = lines[0].rstrip("\r").split()
    head += [""] * (5 - len(head))
    banner, obj, fmt, field, sym = head[:5]
    obj, fmt, field, sym = obj.lower(), fmt.lower(), field.lower(), sym.lower()
    if banner != "%%MatrixMarket":
        _fail(origin, "missing %%MatrixMarket banner")
    if obj != "matrix":
        _fail(origin, f"unsupported object '{obj}'")
    if fmt != "coordinate":
        _fail(origin, "only coordinate format is supported")
    pattern = field == "pattern"
    if field not in ("real", "integer") and not pattern:
        _fail(origin, f"unsupported field '{field}'")
    symmetric = sym == "symmetric"
    if sym != "general" and not symmetric:
        _fail(origin, f"unsupported symmetry '{sym}'")
    k = 1
    while k < len(lines):
        s = lines[k].strip()
        if s and not s.startswith("%"):
            break
        k += 1
    if k >= len(lines):
        _fail(origin, "malformed size line ''")
    parts = lines[k].split()
    try:
        rows, cols, declared = int(parts[0]), int(parts[1]), int(parts[2])
    except (IndexError, ValueError):
        _fail(origin, f"malformed size line '{lines[k].rstrip()}'")
    if rows < 0 or cols < 0 or declared < 0:
        _fail(origin, f"malformed size line '{lines[k].rstrip()}'")
    if rows > INT32_MAX or cols > INT32_MAX:
        _fail(origin, "matrix dimensions exceed index range")
    body = []
    for line in lines[k + 1:]:
        s = line.strip()
        if not s or s.startswith("%"):
            continue
        body.append(s)
        if len(body) == declared:
            break
    if len(body) < declared:
        _fail(origin, "unexpected end of file")
    need = 2 if pattern else 3
    ii = np.empty(declared, np.int64)
    jj = np.empty(declared, np.int64)
    vv = np.ones(declared, np.float64)
    for q, s in enumerate(body):
        f = s.split()
        if len(f) < 2:
            _fail(origin, f"malformed entry '{s}'")
        try:
            ii[q], jj[q] = int(f[0]), int(f[1])
        except ValueError:
            _fail(origin, f"malformed entry '{s}'")
        if not pattern:
            if len(f) < need:
                _fail(origin, f"missing value in entry '{s}'")
            try:
                vv[q] = float(f[2])
            except ValueError:
                _fail(origin, f"missing value in entry '{s}'")
        if ii[q] < 1 or ii[q] > rows or jj[q] < 1 or jj[q] > cols:
            _fail(origin, f"index out of range in entry '{s}'")
    r, c = ii - 1, jj - 1
    if symmetric:
        off = r != c
        r = np.concatenate([r, c[off]])
        c = np.concatenate([c, (ii - 1)[off]])
        vv = np.concatenate([vv, vv[off]])
    return rows, cols, r, c, vv


def csr_from_triplets(n_rows, n_cols, r, c, v, dtype=np.float64) -> Csr:
    """csr.hpp:74-115: sort by (row, col), sum duplicates."""
    r = np.asarray(r, np.int64)
    c = np.asarray(c, np.int64)
    v = np.asarray(v, np.float64)
    if r.size and (r.min() < 0 or r.max() >= n_rows or c.min() < 0 or c.max() >= n_cols):
        raise ValueError("csr_from_triplets: entry out of range")
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    if r.size:
        new = np.ones(r.size, bool)
        new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        starts = np.nonzero(new)[0]
        v = np.add.reduceat(v, starts)
        r, c = r[starts], c[starts]
    if r.size > INT32_MAX:
        raise ValueError("csr_from_triplets: nnz exceeds index range")
    rp = np.zeros(n_rows + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=n_rows), out=rp[1:])
    return Csr(n_rows, n_cols, rp.astype(np.int32), c.astype(np.int32), v.astype(dtype))


def load_matrix_market(path: str, dtype=np.float64) -> Csr:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise RuntimeError(f"cannot open {path}") from None
    rows, cols, r, c, v = parse_matrix_market(text, path)
    return csr_from_triplets(rows, cols, r, c, v, dtype)


def write_matrix_market(m: Csr, path: str) -> None:
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot open {path} for writing") from None
    with f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{m.n_rows} {m.n_cols} {m.nnz}\n")
        rows = np.repeat(np.arange(m.n_rows), np.diff(m.row_ptr))
        for r, c, x in zip(rows, m.col_idx, m.values):
            f.write(f"{r + 1} {c + 1} {float(x):.17g}\n")
