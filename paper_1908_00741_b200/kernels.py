"""The reference's kernel seam, backed by libhbmc_b200.so.

Drop-in for `trilab._kernels.numba_backend` (K/ = /root/reference/pkg/src/
trilab/_kernels/): the same 11 functions, same argument order and dtypes
(numpy int64 indices, float64 values), same in-place / returned outputs and
the same sentinel error convention, so a trilab maintainer can register this
module as a backend (`_BACKENDS["cuda"] = paper_1908_00741_b200.kernels`, see
INTEGRATION.md).

* construction kernels (grow_blocks, color_block_graph, greedy_color,
  ic0_factor, llt_on_pattern) run in the native host builder, bit-exact;
* hot kernels (spmv_*, fwd/bwd_*_range) run on the B200.  Host arrays are
  copied in, the kernel runs, outputs are copied back (the seam passes host
  numpy arrays); read-only matrix arrays are cached on the device keyed by
  their buffer, so repeated sweeps over one factor upload it once.  CUDA
  tensors are accepted too and then nothing is copied.
"""

import numpy as np

from . import _lib
from ._lib import LIB, check, ptr

NAME = "cuda"


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------ construction
def grow_blocks(row_ptr, col_idx, block_size):
    """K/numba_backend.py:232-270 -> (block_of, n_blocks)."""
    row_ptr, col_idx = _i64(row_ptr), _i64(col_idx)
    n = row_ptr.shape[0] - 1
    block_of = np.empty(n, dtype=np.int64)
    nb = _lib.i64()
    check(LIB.tb_grow_blocks(n, ptr(row_ptr), ptr(col_idx), int(block_size), ptr(block_of), nb))
    return block_of, nb.value


def color_block_graph(row_ptr, col_idx, block_of, n_blocks, block_ptr, block_nodes):
    """K/numba_backend.py:273-291 -> color_of_block."""
    row_ptr, col_idx = _i64(row_ptr), _i64(col_idx)
    out = np.empty(int(n_blocks), dtype=np.int64)
    check(LIB.tb_color_block_graph(row_ptr.shape[0] - 1, ptr(row_ptr), ptr(col_idx),
                                   ptr(_i64(block_of)), int(n_blocks), ptr(_i64(block_ptr)),
                                   ptr(_i64(block_nodes)), ptr(out)))
    return out


def greedy_color(row_ptr, col_idx):
    """K/numba_backend.py:174-191 -> color_of."""
    row_ptr, col_idx = _i64(row_ptr), _i64(col_idx)
    out = np.empty(row_ptr.shape[0] - 1, dtype=np.int64)
    check(LIB.tb_greedy_color(out.shape[0], ptr(row_ptr), ptr(col_idx), ptr(out)))
    return out


def ic0_factor(lrp, lci, lvals, adiag):
    """K/numba_backend.py:40-79: lvals overwritten; -> (bad_row, pivot, d, inv_d)."""
    lrp, lci, adiag = _i64(lrp), _i64(lci), _f64(adiag)
    if not (isinstance(lvals, np.ndarray) and lvals.dtype == np.float64
            and lvals.flags.c_contiguous):
        raise TypeError("lvals must be a C-contiguous float64 array (updated in place)")
    n = adiag.shape[0]
    d = np.empty(n)
    inv_d = np.empty(n)
    bad, piv = _lib.i64(), _lib.dbl()
    rc = LIB.tb_ic0_factor(n, ptr(lrp), ptr(lci), ptr(lvals), ptr(adiag), ptr(d), ptr(inv_d),
                           bad, piv)
    if rc not in (_lib.TB_OK, _lib.TB_EIC_BREAKDOWN):
        check(rc)
    return bad.value, piv.value, d, inv_d


def llt_on_pattern(lrp, lci, lvals, d):
    """K/numba_backend.py:82-111 -> (low, diag)."""
    lrp, lci, lvals, d = _i64(lrp), _i64(lci), _f64(lvals), _f64(d)
    low = np.empty(lvals.shape[0])
    diag = np.empty(d.shape[0])
    check(LIB.tb_llt_on_pattern(d.shape[0], ptr(lrp), ptr(lci), ptr(lvals), ptr(d),
                                ptr(low), ptr(diag)))
    return low, diag


# ------------------------------------------------------------ device side
_cache = {}


def _dev_ro(a, dtype):
    """Device copy of a read-only host array (cached by buffer identity)."""
    from . import device
    t = device.torch()
    if isinstance(a, t.Tensor) and a.is_cuda:
        return a.contiguous()
    arr = np.ascontiguousarray(a)
    key = (arr.__array_interface__["data"][0], arr.shape, arr.dtype.str, dtype)
    hit = _cache.get(key)
    if hit is not None and hit[0] is a:
        return hit[1]
    d = device.to_device(arr.astype(dtype, copy=False))
    if len(_cache) > 64:
        _cache.clear()
    _cache[key] = (a, d)
    return d


def _dev_in(a):
    """Device copy of an input vector (never cached: callers mutate them)."""
    from . import device
    t = device.torch()
    if isinstance(a, t.Tensor) and a.is_cuda:
        return a.contiguous()
    return device.to_device(_f64(a))


def _dev_rw(a, lo=0, hi=None):
    """(device tensor, writeback) for an in/out float64 array.

    Only rows [lo, hi) -- the ones the kernel writes -- are copied back: the
    reference calls the range kernels from several WorkerPool threads at
    once on disjoint ranges of one output array (src/precond.py:131-139), so
    writing back the whole array would overwrite a concurrent call's rows
    with this call's stale copy."""
    from . import device
    t = device.torch()
    if isinstance(a, t.Tensor) and a.is_cuda:
        return a, None
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
        raise TypeError("output must be a C-contiguous float64 array (updated in place)")
    d = device.to_device(a)
    hi = a.shape[0] if hi is None else hi

    def writeback():
        if hi > lo:
            a[lo:hi] = d[lo:hi].cpu().numpy()
    return d, writeback


def _stream():
    from . import device
    return device.current_stream()


def spmv_csr(row_ptr, col_idx, vals, x, out):
    """K/numba_backend.py:16-23 (out written in place)."""
    n = _i64(row_ptr).shape[0] - 1
    rp = _dev_ro(row_ptr, np.int64)
    ci = _dev_ro(col_idx, np.int32)
    v = _dev_ro(vals, np.float64)
    xd = _dev_in(x)
    od, wb = _dev_rw(out)
    check(LIB.tb_dev_spmv_csr(n, ptr(rp), ptr(ci), ptr(v), ptr(xd), ptr(od), _stream()))
    if wb:
        wb()


def spmv_sell(slice_ptr, slice_len, col_idx, vals, slice_width, x, out):
    """K/numba_backend.py:26-37 (out written in place)."""
    sl = _dev_ro(slice_len, np.int32)
    n_slices = int(np.asarray(slice_len).shape[0]) if isinstance(slice_len, np.ndarray) else sl.shape[0]
    sp = _dev_ro(slice_ptr, np.int64)
    ci = _dev_ro(col_idx, np.int32)
    v = _dev_ro(vals, np.float64)
    xd = _dev_in(x)
    od, wb = _dev_rw(out)
    check(LIB.tb_dev_spmv_sell(n_slices, ptr(sp), ptr(sl), ptr(ci), ptr(v), int(slice_width),
                               ptr(xd), ptr(od), _stream()))
    if wb:
        wb()


def _csr_range(forward, rp, ci, vals, inv_d, src, dst, start, end):
    rpd = _dev_ro(rp, np.int64)
    cid = _dev_ro(ci, np.int32)
    vd = _dev_ro(vals, np.float64)
    idd = _dev_ro(inv_d, np.float64)
    sd = _dev_in(src)
    dd, wb = _dev_rw(dst, int(start), int(end))
    # the range is one sequential task (rows ascending / descending)
    tpd = _dev_in(np.array([int(start), int(end)], dtype=np.float64)).to(
        dtype=__import__("torch").int64)
    check(LIB.tb_dev_csr_sweep_tasks(1 if forward else 0, ptr(rpd), ptr(cid), ptr(vd),
                                     ptr(idd), ptr(sd), ptr(dd), 0, 1, ptr(tpd), None,
                                     _stream()))
    if wb:
        wb()


def fwd_csr_range(lrp, lci, lvals, inv_d, r, y, start, end):
    """K/numba_backend.py:114-120 (y written in place)."""
    _csr_range(True, lrp, lci, lvals, inv_d, r, y, start, end)


def bwd_csr_range(urp, uci, uvals, inv_d, y, z, start, end):
    """K/numba_backend.py:123-129 (z written in place)."""
    _csr_range(False, urp, uci, uvals, inv_d, y, z, start, end)


def _sell_range(forward, slice_ptr, slice_len, col_idx, vals, inv_d, src, dst, width,
                block_rows, k0, k1):
    sp = _dev_ro(slice_ptr, np.int64)
    sl = _dev_ro(slice_len, np.int32)
    ci = _dev_ro(col_idx, np.int32)
    vd = _dev_ro(vals, np.float64)
    idd = _dev_ro(inv_d, np.float64)
    sd = _dev_in(src)
    rows_per_block = int(width) * int(block_rows)
    dd, wb = _dev_rw(dst, int(k0) * rows_per_block, int(k1) * rows_per_block)
    fn = LIB.tb_dev_fwd_sell_range if forward else LIB.tb_dev_bwd_sell_range
    check(fn(ptr(sp), ptr(sl), ptr(ci), ptr(vd), ptr(idd), ptr(sd), ptr(dd), int(width),
             int(block_rows), int(k0), int(k1), _stream()))
    if wb:
        wb()


def fwd_sell_range(slice_ptr, slice_len, col_idx, vals, inv_d, r, y, width, block_rows, k0, k1):
    """K/numba_backend.py:132-153 over level-1 blocks [k0, k1) (y in place).

    The blocks of [k0, k1) must be mutually independent (one HBMC color or
    part of one), which is how the reference's _hbmc_sweep calls it."""
    _sell_range(True, slice_ptr, slice_len, col_idx, vals, inv_d, r, y, width, block_rows, k0, k1)


def bwd_sell_range(slice_ptr, slice_len, col_idx, vals, inv_d, y, z, width, block_rows, k0, k1):
    """K/numba_backend.py:156-171 (z in place)."""
    _sell_range(False, slice_ptr, slice_len, col_idx, vals, inv_d, y, z, width, block_rows, k0, k1)


# ------------------------------------------------------------ registry
# src/_kernels/__init__.py:46-73 resolves a backend name to a kernel module.
# This package has exactly one backend (the B200 one; no multi-backend
# dispatch), so the registry has one entry.
def available_backends():
    return [NAME]


def default_backend():
    return NAME


def get_kernels(backend=None):
    """The kernel module for `backend` (None / "auto" / "cuda": this one)."""
    import sys
    if backend in (None, "auto", NAME):
        return sys.modules[__name__]
    raise ValueError(f"unknown backend {backend!r}; available: {available_backends()}")
