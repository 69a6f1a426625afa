"""Matrix ingestion for user matrices (drop-in for trilab.io, src/io.py).

MatrixMarket `coordinate real symmetric|general` text and the reference's
binary CSR cache (`.tlcsr`: magic b"TLCSR\\0", u32 version 1, i64 n, i64 nnz,
i64 row_ptr[n+1], i64 col_idx[nnz], f64 values[nnz], little-endian).

The byte scanning runs natively (csrc/mm_parse.cpp: one pass locating the
size line and parsing every entry line with its line number); validation
keeps the reference's order and messages so IngestionError names the same
`path:line` (banner, size line, entry count, entry syntax, bounds, upper
triangle in a symmetric file, duplicates), zero off-diagonals are dropped
and counted, symmetric input is mirrored to full storage.
"""

import numpy as np

from . import _lib
from ._lib import LIB
from .matrix import CooMatrix, CsrMatrix, coo_to_csr

__all__ = ["IngestionError", "read_matrix_market", "write_matrix_market",
           "write_csr_cache", "read_csr_cache", "load_matrix"]

CACHE_MAGIC = b"TLCSR\0"
CACHE_VERSION = 1


class IngestionError(ValueError):
    """Unreadable matrix file; the message carries path:line."""

    def __init__(self, path, lineno, msg):
        self.path = str(path)
        self.lineno = lineno
        super().__init__(f"{path}:{lineno}: {msg}")


def _banner(path, first):
    toks = first.split()
    if len(toks) != 5 or toks[0].lower() != "%%matrixmarket":
        raise IngestionError(path, 1, "malformed MatrixMarket banner")
    obj, fmt, field, sym = (t.lower() for t in toks[1:])
    checks = ((obj == "matrix", f"unsupported object {obj!r}"),
              (fmt == "coordinate", f"unsupported format {fmt!r} (need coordinate)"),
              (field == "real", f"non-real field {field!r}"),
              (sym in ("symmetric", "general"), f"unsupported symmetry {sym!r}"))
    for ok, msg in checks:
        if not ok:
            raise IngestionError(path, 1, msg)
    return sym


def _size(path, lineno, text):
    parts = text.split()
    if len(parts) != 3:
        raise IngestionError(path, lineno, "size line must be 'rows cols nnz'")
    try:
        m, n, nnz = (int(p) for p in parts)
    except ValueError:
        raise IngestionError(path, lineno, "size line must hold three integers") from None
    if m != n:
        raise IngestionError(path, lineno, f"matrix is {m}x{n}; only square supported")
    if n < 0 or nnz < 0:
        raise IngestionError(path, lineno, "negative dimension")
    return n, nnz


def read_matrix_market(path):
    """src/io.py:70-163: full-storage COO, 0-based, symmetric mirrored."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if not raw:
        raise IngestionError(path, 1, "empty file")
    nl = raw.find(b"\n")
    first = (raw if nl < 0 else raw[:nl]).decode("ascii", "replace")
    sym = _banner(path, first)
    buf = _lib.ptr(np.frombuffer(raw, dtype=np.uint8))
    size_no, sb, se, body, nlines = (_lib.i64() for _ in range(5))
    _lib.check(LIB.tb_mm_locate(buf, len(raw), size_no, sb, se, body, nlines))
    if size_no.value == 0:
        raise IngestionError(path, nlines.value, "missing size line")
    n, nnz = _size(path, size_no.value, raw[sb.value:se.value].decode("ascii", "replace"))
    rows = np.empty(nnz, dtype=np.int64)
    cols = np.empty(nnz, dtype=np.int64)
    vals = np.empty(nnz, dtype=np.float64)
    lines = np.empty(nnz, dtype=np.int64)
    found, kth = _lib.i64(), _lib.i64()
    ekind = _lib.i32()
    eline, eb, ee = _lib.i64(), _lib.i64(), _lib.i64()
    _lib.check(LIB.tb_mm_entries(buf, len(raw), body.value, size_no.value + 1, nnz,
                                 _lib.ptr(rows), _lib.ptr(cols), _lib.ptr(vals),
                                 _lib.ptr(lines), found, kth, ekind, eline, eb, ee))
    if found.value != nnz:
        where = kth.value if found.value > nnz else size_no.value
        raise IngestionError(path, where, f"expected {nnz} entries, found {found.value}")
    if ekind.value:
        frag = raw[eb.value:ee.value].decode("ascii", "replace")
        msg = {1: "entry line must be 'row col value'", 2: f"bad index in {frag!r}",
               3: f"non-real value {frag!r}"}[ekind.value]
        raise IngestionError(path, eline.value, msg)
    rows -= 1
    cols -= 1
    out = (rows < 0) | (rows >= n) | (cols < 0) | (cols >= n)
    if out.any():
        k = int(np.argmax(out))
        raise IngestionError(path, int(lines[k]),
                             f"index ({rows[k] + 1}, {cols[k] + 1}) outside {n}x{n}")
    if sym == "symmetric":
        up = rows < cols
        if up.any():
            k = int(np.argmax(up))
            raise IngestionError(path, int(lines[k]),
                                 "entry above the diagonal in a symmetric file")
    if nnz > 1:
        order = np.lexsort((cols, rows))
        rs, cs = rows[order], cols[order]
        dup = (rs[1:] == rs[:-1]) & (cs[1:] == cs[:-1])
        if dup.any():
            k = int(np.argmax(dup))
            raise IngestionError(path, int(lines[order[k + 1]]),
                                 f"duplicate entry ({rs[k] + 1} {cs[k] + 1})")
    off = rows != cols
    zero = off & (vals == 0.0)
    dropped = int(zero.sum())
    if dropped:
        keep = ~zero
        rows, cols, vals, off = rows[keep], cols[keep], vals[keep], off[keep]
    if sym == "symmetric" and off.any():
        rows, cols, vals = (np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                            np.concatenate([vals, vals[off]]))
    return CooMatrix(n, rows, cols, vals, dropped_zeros=dropped)


def write_matrix_market(path, csr, comment=None):
    """src/io.py:166-180: lower triangle, coordinate real symmetric, %.17g."""
    rows = np.repeat(np.arange(csr.n, dtype=np.int64), np.diff(csr.row_ptr))
    low = csr.col_idx <= rows
    r, c, v = rows[low] + 1, csr.col_idx[low] + 1, csr.vals[low]
    head = ["%%MatrixMarket matrix coordinate real symmetric"]
    if comment:
        head += [f"% {line}" for line in str(comment).splitlines()]
    head.append(f"{csr.n} {csr.n} {r.shape[0]}")
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join(head) + "\n")
        if r.shape[0]:
            fh.write("\n".join(f"{i} {j} {x:.17g}" for i, j, x in
                               zip(r.tolist(), c.tolist(), v.tolist())) + "\n")


def write_csr_cache(path, csr):
    """src/io.py:183-190: the binary CSR cache."""
    with open(path, "wb") as fh:
        fh.write(CACHE_MAGIC)
        fh.write(np.array([CACHE_VERSION], dtype="<u4").tobytes())
        fh.write(np.array([csr.n, csr.nnz], dtype="<i8").tobytes())
        for arr, dt in ((csr.row_ptr, "<i8"), (csr.col_idx, "<i8"), (csr.vals, "<f8")):
            fh.write(np.ascontiguousarray(arr, dtype=dt).tobytes())


def read_csr_cache(path):
    """src/io.py:193-212."""
    with open(path, "rb") as fh:
        raw = fh.read()
    m = len(CACHE_MAGIC)
    if raw[:m] != CACHE_MAGIC:
        raise IngestionError(path, 0, "not a CSR cache file (bad magic)")
    if len(raw) < m + 4:
        raise IngestionError(path, 0, "truncated cache header")
    version = int(np.frombuffer(raw, dtype="<u4", count=1, offset=m)[0])
    if version != CACHE_VERSION:
        raise IngestionError(path, 0, f"unsupported cache version {version}")
    pos = m + 4
    if len(raw) < pos + 16:
        raise IngestionError(path, 0, "truncated cache header")
    n, nnz = (int(x) for x in np.frombuffer(raw, dtype="<i8", count=2, offset=pos))
    pos += 16
    need = 8 * (n + 1) + 8 * nnz + 8 * nnz
    if n < 0 or nnz < 0 or len(raw) < pos + need:
        raise IngestionError(path, 0, "truncated cache body")
    row_ptr = np.frombuffer(raw, dtype="<i8", count=n + 1, offset=pos).astype(np.int64)
    pos += 8 * (n + 1)
    col_idx = np.frombuffer(raw, dtype="<i8", count=nnz, offset=pos).astype(np.int64)
    pos += 8 * nnz
    vals = np.frombuffer(raw, dtype="<f8", count=nnz, offset=pos).astype(np.float64)
    return CsrMatrix(n, row_ptr, col_idx, vals)


def load_matrix(path, write_cache=False):
    """src/io.py:215-228: sniff the cache magic, else parse MatrixMarket
    (write_cache=True leaves `<path>.tlcsr` next to a parsed text file)."""
    with open(path, "rb") as fh:
        head = fh.read(len(CACHE_MAGIC))
    if head == CACHE_MAGIC:
        return read_csr_cache(path)
    a = coo_to_csr(read_matrix_market(path))
    if write_cache:
        write_csr_cache(str(path) + ".tlcsr", a)
    return a
