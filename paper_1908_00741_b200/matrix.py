"""Sparse containers, conversions and SpMV (drop-in for trilab.matrix).

The container types and their field names are the reference's host-side
contract (src/matrix.py:24-157).  Conversions run in the native host builder
(libhbmc_b200.so); `spmv` runs on the B200 (K/numba_backend.py:16-37
restated as sm_100a kernels) -- there is no CPU SpMV path.
"""

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import LIB, check, f64a, i64a, ptr


@dataclass
class CooMatrix:
    """Square coordinate-format matrix (src/matrix.py:24-47)."""

    n: int
    row: np.ndarray
    col: np.ndarray
    val: np.ndarray
    dropped_zeros: int = 0

    def __post_init__(self):
        self.row = i64a(self.row)
        self.col = i64a(self.col)
        self.val = f64a(self.val)
        if not (self.row.shape == self.col.shape == self.val.shape):
            raise ValueError("row/col/val length mismatch")

    @property
    def nnz(self):
        return self.val.shape[0]


def _find_diag_ptr(n, row_ptr, col_idx):
    """Diagonal slot of every row, -1 if absent (native scan, host builder)."""
    diag_ptr = np.empty(n, dtype=np.int64)
    check(LIB.tb_csr_diag_ptr(n, ptr(row_ptr), ptr(col_idx), ptr(diag_ptr)))
    return diag_ptr


@dataclass
class CsrMatrix:
    """Square CSR matrix with sorted column indices (src/matrix.py:50-90)."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    diag_ptr: np.ndarray = field(default=None)
    inserted_diag: int = 0

    def __post_init__(self):
        self.row_ptr = i64a(self.row_ptr)
        self.col_idx = i64a(self.col_idx)
        self.vals = f64a(self.vals)
        if self.diag_ptr is None:
            self.diag_ptr = _find_diag_ptr(self.n, self.row_ptr, self.col_idx)
        else:
            self.diag_ptr = i64a(self.diag_ptr)

    @property
    def nnz(self):
        return self.vals.shape[0]

    def diagonal(self):
        d = np.zeros(self.n)
        has = self.diag_ptr >= 0
        d[has] = self.vals[self.diag_ptr[has]]
        return d

    def to_dense(self):
        a = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        a[rows, self.col_idx] = self.vals
        return a


@dataclass
class SellMatrix:
    """Sliced ELLPACK, slice width = w (src/matrix.py:93-119).

    Entry t of row r sits at slice_ptr[s] + t*width + (r - s*width); padding
    is value 0 with the column pointing at the entry's own row.  `col32` is
    the int32 copy of col_idx that the device consumes.
    """

    n: int
    n_pad: int
    width: int
    slice_ptr: np.ndarray
    slice_len: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    col32: np.ndarray = field(default=None, repr=False)

    def __post_init__(self):
        self.slice_ptr = i64a(self.slice_ptr)
        self.slice_len = i64a(self.slice_len)
        self.col_idx = i64a(self.col_idx)
        self.vals = f64a(self.vals)
        if self.col32 is None:
            self.col32 = self.col_idx.astype(np.int32)

    @property
    def n_slices(self):
        return self.slice_len.shape[0]


@dataclass
class Permutation:
    """Bijection on [0, n); new_of_old[i] is where old index i lands."""

    new_of_old: np.ndarray

    def __post_init__(self):
        self.new_of_old = i64a(self.new_of_old)
        n = self.new_of_old.shape[0]
        if n:
            if self.new_of_old.min() < 0 or self.new_of_old.max() >= n:
                raise ValueError("permutation image out of range")
        seen = np.zeros(n, dtype=bool)
        seen[self.new_of_old] = True
        if not seen.all():
            raise ValueError("not a bijection")

    def __len__(self):
        return self.new_of_old.shape[0]

    @classmethod
    def identity(cls, n):
        return cls(np.arange(n, dtype=np.int64))

    @property
    def old_of_new(self):
        inv = np.empty_like(self.new_of_old)
        inv[self.new_of_old] = np.arange(len(self), dtype=np.int64)
        return inv

    def inverse(self):
        return Permutation(self.old_of_new)

    def compose(self, first):
        """Permutation applying `first`, then self."""
        return Permutation(self.new_of_old[first.new_of_old])


def coo_to_csr(coo, ensure_diagonal=True):
    """src/matrix.py:168-197, sorted by the native counting sort."""
    row, col, val = coo.row, coo.col, coo.val
    inserted = 0
    if ensure_diagonal and coo.n:
        has_diag = np.zeros(coo.n, dtype=bool)
        has_diag[row[row == col]] = True
        missing = np.nonzero(~has_diag)[0]
        inserted = missing.shape[0]
        if inserted:
            row = np.concatenate([row, missing])
            col = np.concatenate([col, missing])
            val = np.concatenate([val, np.zeros(inserted)])
    row, col, val = i64a(row), i64a(col), f64a(val)
    nnz = row.shape[0]
    row_ptr = np.empty(coo.n + 1, dtype=np.int64)
    c = np.empty(nnz, dtype=np.int64)
    v = np.empty(nnz, dtype=np.float64)
    dr, dc = _lib.i64(), _lib.i64()
    rc = LIB.tb_coo_to_csr(coo.n, nnz, ptr(row), ptr(col), ptr(val),
                           ptr(row_ptr), ptr(c), ptr(v), dr, dc)
    if rc == _lib.TB_EDUP:
        raise ValueError(f"duplicate entry at ({dr.value}, {dc.value})")
    check(rc)
    return CsrMatrix(coo.n, row_ptr, c, v, inserted_diag=inserted)


def csr_to_coo(csr):
    rows = np.repeat(np.arange(csr.n, dtype=np.int64), np.diff(csr.row_ptr))
    return CooMatrix(csr.n, rows, csr.col_idx.copy(), csr.vals.copy())


def csr_transpose(csr):
    """src/matrix.py:205-208."""
    rp = np.empty(csr.n + 1, dtype=np.int64)
    c = np.empty(csr.nnz, dtype=np.int64)
    v = np.empty(csr.nnz, dtype=np.float64)
    check(LIB.tb_csr_transpose(csr.n, ptr(csr.row_ptr), ptr(csr.col_idx),
                               ptr(csr.vals), ptr(rp), ptr(c), ptr(v)))
    return CsrMatrix(csr.n, rp, c, v)


def _reorder_rows(csr, row_order):
    inv = row_order.old_of_new
    counts = np.diff(csr.row_ptr)[inv]
    row_ptr = np.zeros(csr.n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    src_start = csr.row_ptr[inv]
    gather = (np.repeat(src_start - row_ptr[:-1], counts)
              + np.arange(row_ptr[-1], dtype=np.int64))
    return CsrMatrix(csr.n, row_ptr, csr.col_idx[gather], csr.vals[gather],
                     diag_ptr=np.full(csr.n, -1, np.int64))


def csr_to_sell(csr, width, row_order=None, want_col64=True):
    """src/matrix.py:211-261 (native fill; also emits the int32 columns)."""
    if width < 1:
        raise ValueError("width must be positive")
    if row_order is not None:
        if len(row_order) != csr.n:
            raise ValueError("row_order length mismatch")
        csr = _reorder_rows(csr, row_order)
    n = csr.n
    n_slices = -(-n // width)
    n_pad = n_slices * width
    row_len = np.zeros(n_pad, dtype=np.int64)
    row_len[:n] = np.diff(csr.row_ptr)
    slice_len = row_len.reshape(n_slices, width).max(axis=1) if n_slices else \
        np.zeros(0, dtype=np.int64)
    slice_ptr = np.zeros(n_slices + 1, dtype=np.int64)
    np.cumsum(slice_len * width, out=slice_ptr[1:])
    total = int(slice_ptr[-1])
    vals = np.empty(total)
    col64 = np.empty(total, dtype=np.int64) if want_col64 else None
    col32 = np.empty(total, dtype=np.int32)
    check(LIB.tb_csr_to_sell_fill(n, ptr(csr.row_ptr), ptr(csr.col_idx),
                                  ptr(csr.vals), width, n_slices,
                                  ptr(slice_ptr), ptr(col64), ptr(col32),
                                  ptr(vals)))
    if col64 is None:
        col64 = np.empty(0, dtype=np.int64)
    return SellMatrix(n, n_pad, width, slice_ptr, slice_len, col64, vals,
                      col32=col32)


def sell_to_csr(sell):
    """src/matrix.py:264-290: unpack, dropping (own row, 0.0) padding."""
    w = sell.width
    n = sell.n
    if n == 0:
        return coo_to_csr(CooMatrix(0, np.empty(0), np.empty(0), np.empty(0)),
                          ensure_diagonal=False)
    rows_l, pos_l = [], []
    lens = sell.slice_len
    # slots of slice s: t in [0, len_s), lane j -> position slice_ptr[s]+t*w+j
    s_of_row = np.arange(n) // w
    lane = np.arange(n) - s_of_row * w
    cnt = lens[s_of_row]
    rows = np.repeat(np.arange(n, dtype=np.int64), cnt)
    t = np.arange(int(cnt.sum()), dtype=np.int64) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    pos = sell.slice_ptr[s_of_row][rows] + lane[rows] + w * t
    c = sell.col_idx[pos]
    v = sell.vals[pos]
    keep = ~((v == 0.0) & (c == rows))
    del rows_l, pos_l
    return coo_to_csr(CooMatrix(n, rows[keep], c[keep], v[keep]),
                      ensure_diagonal=False)


def permute_system(a, b, p):
    """src/matrix.py:293-304: (i, j) -> (q[i], q[j]); b'[q[i]] = b[i]."""
    q = i64a(p.new_of_old)
    if q.shape[0] != a.n:
        raise ValueError("permutation length mismatch")
    rp = np.empty(a.n + 1, dtype=np.int64)
    c = np.empty(a.nnz, dtype=np.int64)
    v = np.empty(a.nnz, dtype=np.float64)
    check(LIB.tb_permute_csr(a.n, ptr(a.row_ptr), ptr(a.col_idx), ptr(a.vals),
                             ptr(q), ptr(rp), ptr(c), ptr(v)))
    b_new = np.empty_like(b, dtype=np.float64)
    b_new[q] = b
    return CsrMatrix(a.n, rp, c, v), b_new


def spmv_host_exact(a, x):
    """b = A x with the reference's sequential per-row order (host, once).

    Used only to form right-hand sides of the benchmark problems
    (b = A x*); every solver-path SpMV runs on the GPU.
    """
    x = f64a(x)
    out = np.empty(a.n)
    check(LIB.tb_spmv_csr_host(a.n, ptr(a.row_ptr), ptr(a.col_idx), ptr(a.vals),
                               ptr(x), ptr(out)))
    return out


def spmv(a, x, kernels=None):
    """y = A x on the B200 for CSR or SELL storage (src/matrix.py:307-323).

    `kernels` is accepted for signature compatibility and ignored (there is
    one backend).  numpy in -> numpy out; a CUDA tensor in -> CUDA tensor out.
    """
    from . import device
    return device.spmv(a, x)


def gen_laplacian_5pt(nx, ny):
    """5-point Laplacian, index iy*nx + ix, diagonal 4 (src/matrix.py:326-351)."""
    if nx < 2 or ny < 2:
        raise ValueError("grid sides must be at least 2")
    n = nx * ny
    idx = np.arange(n, dtype=np.int64).reshape(ny, nx)
    lo = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()])
    hi = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()])
    rows = np.concatenate([lo, hi, np.arange(n)])
    cols = np.concatenate([hi, lo, np.arange(n)])
    vals = np.concatenate([-np.ones(2 * lo.size), np.full(n, 4.0)])
    return coo_to_csr(CooMatrix(n, rows, cols, vals)), np.ones(n)


def gen_random_spd(n, density=0.01, seed=0):
    """Random SPD test matrix, same draws as src/matrix.py:354-374."""
    rng = np.random.default_rng(seed)
    target = max(0, int(round(density * n * n / 2)))
    i = rng.integers(0, n, size=2 * target + 8)
    j = rng.integers(0, n, size=2 * target + 8)
    keep = i < j
    pairs = np.unique(np.stack([i[keep], j[keep]], axis=1), axis=0)[:target]
    ii = pairs[:, 0]
    jj = pairs[:, 1]
    v = -rng.uniform(0.1, 1.0, size=ii.shape[0])
    rows = np.concatenate([ii, jj])
    cols = np.concatenate([jj, ii])
    vals = np.concatenate([v, v])
    diag = np.ones(n)
    np.add.at(diag, rows, np.abs(vals))
    rows = np.concatenate([rows, np.arange(n)])
    cols = np.concatenate([cols, np.arange(n)])
    vals = np.concatenate([vals, diag])
    return coo_to_csr(CooMatrix(n, rows, cols, vals))
