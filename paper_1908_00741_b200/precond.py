"""IC(0) factor and the substitution operators (drop-in for trilab.precond).

* ic0_factorize: the zero-fill shifted IC of K/numba_backend.py:40-79, run
  in the native host builder with non-contracted arithmetic (bit-exact).
* sub_forward_* / sub_backward_*: ALL run on the B200.  HBMC uses the SELL
  sweep kernel (one grid-wide phase per color); MC / BMC / natural use the
  CSR task-sweep kernel (one phase per color / per dependency level).  Every
  row's arithmetic is the reference's, so outputs are bitwise equal to
  sub_forward_seq / sub_backward_seq of the reference.

`pool=` and `kernels=` are accepted for signature compatibility and ignored
(one device backend; the GPU grid replaces the thread pool).  `counter=`
still sees exactly n_phases - 1 barrier() calls per sweep, which are the
device-side phase boundaries.
"""

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import LIB, check, i64a, ptr
from .matrix import CsrMatrix, csr_to_sell, csr_transpose

__all__ = [
    "IcBreakdownError", "IcFactor", "SellFactor", "BarrierCounter",
    "WorkerPool", "ic0_factorize", "build_sell_factor",
    "sub_forward_seq", "sub_backward_seq", "sub_forward_mc",
    "sub_backward_mc", "sub_forward_bmc", "sub_backward_bmc",
    "sub_forward_hbmc", "sub_backward_hbmc", "apply_ic_preconditioner",
]


class IcBreakdownError(ArithmeticError):
    """Non-positive pivot encountered during factorization."""

    def __init__(self, row, pivot):
        self.row = int(row)
        self.pivot = float(pivot)
        super().__init__(f"non-positive pivot {pivot:.6g} at row {row}")


@dataclass
class IcFactor:
    L: CsrMatrix
    d: np.ndarray
    inv_diag: np.ndarray
    shift: float
    layout_tag: str
    U: CsrMatrix

    @property
    def n(self):
        return self.d.shape[0]


@dataclass
class SellFactor:
    lower: object
    upper: object
    d: np.ndarray
    inv_diag: np.ndarray
    w: int
    b_s: int
    layout_tag: str = "hbmc"

    @property
    def n(self):
        return self.d.shape[0]


@dataclass
class BarrierCounter:
    """Counts synchronization points; count/phase_order reset per invocation."""

    count: int = 0
    total: int = 0
    invocations: int = 0
    phase_order: list = field(default_factory=list)

    def start(self):
        self.count = 0
        self.phase_order = []
        self.invocations += 1

    def enter_phase(self, color):
        self.phase_order.append(int(color))

    def barrier(self):
        self.count += 1
        self.total += 1


class _NullCounter:
    def start(self):
        pass

    def enter_phase(self, color):
        pass

    def barrier(self):
        pass


_NULL = _NullCounter()


class WorkerPool:
    """Kept for signature compatibility with src/precond.py:123-150.

    The device grid is the worker pool here; `threads` is recorded and
    otherwise unused by the substitution operators.
    """

    def __init__(self, threads=1):
        self.threads = max(1, int(threads))

    def run(self, fn, tasks):
        for args in tasks:
            fn(*args)

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def _strict_tri(a: CsrMatrix, upper=False):
    """src/precond.py:163-169: strictly lower (upper) part, native two-pass."""
    row_ptr = np.empty(a.n + 1, dtype=np.int64)
    check(LIB.tb_csr_tri_count(a.n, ptr(a.row_ptr), ptr(a.col_idx), 1 if upper else 0,
                               ptr(row_ptr)))
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz, dtype=np.float64)
    check(LIB.tb_csr_tri_fill(a.n, ptr(a.row_ptr), ptr(a.col_idx), ptr(a.vals),
                              1 if upper else 0, ptr(row_ptr), ptr(col), ptr(val)))
    return CsrMatrix(a.n, row_ptr, col, val, diag_ptr=np.full(a.n, -1, dtype=np.int64))


def tri_row_counts(a: CsrMatrix, upper=False):
    """Per-row entry counts of the strictly lower (upper) part (first pass
    of _strict_tri only; used to count algorithmic bytes per color phase)."""
    row_ptr = np.empty(a.n + 1, dtype=np.int64)
    check(LIB.tb_csr_tri_count(a.n, ptr(a.row_ptr), ptr(a.col_idx), 1 if upper else 0,
                               ptr(row_ptr)))
    return np.diff(row_ptr)


def _check_structural_symmetry(a: CsrMatrix):
    ok = _lib.i32()
    check(LIB.tb_csr_is_symmetric(a.n, ptr(a.row_ptr), ptr(a.col_idx), ok))
    if not ok.value:
        raise ValueError("matrix structure is not symmetric")


def ic0_factorize(a: CsrMatrix, shift=0.0, layout_tag="natural", kernels=None):
    """src/precond.py:179-200 over K/numba_backend.py:40-79."""
    if shift < 0:
        raise ValueError("shift must be non-negative")
    if (a.diag_ptr < 0).any():
        bad = int(np.nonzero(a.diag_ptr < 0)[0][0])
        raise ValueError(f"row {bad} has no diagonal entry")
    _check_structural_symmetry(a)
    low = _strict_tri(a, upper=False)
    lvals = low.vals.copy()
    adiag = a.diagonal() * (1.0 + shift)
    d = np.empty(a.n)
    inv_d = np.empty(a.n)
    bad_row, pivot = _lib.i64(), _lib.dbl()
    rc = LIB.tb_ic0_factor(a.n, ptr(low.row_ptr), ptr(low.col_idx), ptr(lvals),
                           ptr(adiag), ptr(d), ptr(inv_d), bad_row, pivot)
    if rc == _lib.TB_EIC_BREAKDOWN:
        raise IcBreakdownError(bad_row.value, pivot.value)
    check(rc)
    L = CsrMatrix(a.n, low.row_ptr, low.col_idx, lvals,
                  diag_ptr=np.full(a.n, -1, dtype=np.int64))
    return IcFactor(L, d, inv_d, float(shift), layout_tag, csr_transpose(L))


def _check_hbmc_lower_structure(low, hl):
    """Every strictly-lower (i, j) must be same level-1 block + same lane +
    earlier step, or an earlier color (src/ordering.py:328-346): the
    dependency structure the per-color device schedule relies on."""
    w, span = hl.w, hl.w * hl.b_s
    rows = np.repeat(np.arange(low.n, dtype=np.int64), np.diff(low.row_ptr))
    cols = low.col_idx
    ki, kj = rows // span, cols // span
    same = ki == kj
    ok_in = (rows % w == cols % w) & (cols < rows)
    col_of = np.repeat(np.arange(hl.n_c, dtype=np.int64), np.diff(hl.color_lvl1_ranges))
    ok_x = col_of[kj] < col_of[ki]
    if not np.all(np.where(same, ok_in, ok_x)):
        raise ValueError("ic0_factorize_device: matrix lacks the HBMC dependency structure")


def ic0_factorize_device(a: CsrMatrix, hl, shift=0.0, layout_tag="hbmc", timings=None):
    """ic0_factorize for a system already in HBMC order, computed on the B200
    (csrc/ic0.cu: one launch per color).  Same IcFactor,
    bitwise, same IcBreakdownError; `hl` is the HbmcLayout of `a`'s ordering.
    """
    from . import device
    t = device.require_cuda()
    if shift < 0:
        raise ValueError("shift must be non-negative")
    if (a.diag_ptr < 0).any():
        bad = int(np.nonzero(a.diag_ptr < 0)[0][0])
        raise ValueError(f"row {bad} has no diagonal entry")
    if a.n != hl.n_pad:
        raise ValueError("ic0_factorize_device: matrix is not in the layout's order")
    _check_structural_symmetry(a)
    low = _strict_tri(a, upper=False)
    # the HBMC dependency structure is checked per entry by the kernel
    rp = device.to_device(low.row_ptr, np.int64)
    ci = device.to_device(low.col_idx, np.int32)
    lv = device.to_device(low.vals, np.float64)
    ad = device.to_device(a.diagonal() * (1.0 + shift), np.float64)
    d = t.empty(a.n, dtype=t.float64, device="cuda")
    inv_d = t.empty_like(d)
    ws = t.empty_like(d)
    cr = np.ascontiguousarray(hl.color_lvl1_ranges, dtype=np.int64)
    bad_row, pivot = _lib.i64(), _lib.dbl()
    t.cuda.synchronize()
    t0 = time.perf_counter()
    rc = LIB.tb_dev_ic0_hbmc(a.n, ptr(rp), ptr(ci), ptr(lv), ptr(ad), ptr(d), ptr(inv_d),
                             hl.w, hl.b_s, hl.n_c, ptr(cr), ptr(ws), bad_row, pivot,
                             device.current_stream())
    if timings is not None:   # the call synchronises on the breakdown flag
        timings["kernel_s"] = time.perf_counter() - t0
    if rc == _lib.TB_EIC_BREAKDOWN:
        raise IcBreakdownError(bad_row.value, pivot.value)
    check(rc)
    L = CsrMatrix(a.n, low.row_ptr, low.col_idx, lv.cpu().numpy(),
                  diag_ptr=np.full(a.n, -1, dtype=np.int64))
    return IcFactor(L, d.cpu().numpy(), inv_d.cpu().numpy(), float(shift), layout_tag,
                    csr_transpose(L))


def build_sell_factor(f: IcFactor, hl):
    """src/precond.py:263-270: L and U in SELL with slice width w."""
    if f.layout_tag != "hbmc":
        raise ValueError(f"factor tag {f.layout_tag!r}; need 'hbmc'")
    if f.n != hl.n_pad:
        raise ValueError("factor size does not match padded layout size")
    return SellFactor(csr_to_sell(f.L, hl.w), csr_to_sell(f.U, hl.w),
                      f.d, f.inv_diag, hl.w, hl.b_s)


def _require_tag(f, expected):
    if f.layout_tag != expected:
        raise ValueError(f"factor was built under {f.layout_tag!r}, kernel needs {expected!r}")


# ------------------------------------------------------------ schedules
def level_schedule(tri: CsrMatrix, forward):
    """Dependency levels of a strict triangle -> (phase_ptr, task_ptr, rows)."""
    from .ordering import _group
    level = np.empty(tri.n, dtype=np.int64)
    nl = _lib.i64()
    check(LIB.tb_level_schedule(tri.n, ptr(tri.row_ptr), ptr(tri.col_idx),
                                1 if forward else 0, ptr(level), nl))
    if not forward:
        # backward sweeps run their phases last-to-first (like the color
        # phases of MC / BMC), so level 0 must be the LAST phase
        level = nl.value - 1 - level
    phase_ptr, rows = _group(level, nl.value)
    return phase_ptr, None, rows


def _sched_for(kind, f, layout):
    """(fwd_sched, bwd_sched) of the CSR task sweeps (MC / BMC / natural)."""
    if kind == "mc":
        s = (i64a(layout.color_ranges), None, None)
        return s, s
    if kind == "bmc":
        s = (i64a(layout.color_block_ranges), i64a(layout.block_bounds), None)
        return s, s
    return level_schedule(f.L, True), level_schedule(f.U, False)


def _task_plan(f, kind, layout):
    """Cached preconditioner-only device plan of an IcFactor."""
    from . import device
    cache = f.__dict__.setdefault("_tb_plans", {})
    key = (kind, id(layout))
    hit = cache.get(key)
    if hit is not None and hit[0] is layout:
        return hit[1]
    fs, bs = _sched_for(kind, f, layout)
    plan = device.DevicePlan(kind=_lib.TB_PRECOND_TASKS, n=f.n, n_real=f.n,
                             inv_d=f.inv_diag, spmv_format=_lib.TB_SPMV_NONE,
                             L_csr=f.L, U_csr=f.U, fwd_sched=fs, bwd_sched=bs)
    plan.n_phases_fwd = fs[0].shape[0] - 1
    plan.n_phases_bwd = bs[0].shape[0] - 1
    cache[key] = (layout, plan)
    return plan


def _hbmc_plan(sf, hl):
    from . import device
    cache = sf.__dict__.setdefault("_tb_plans", {})
    hit = cache.get(id(hl))
    if hit is not None and hit[0] is hl:
        return hit[1]
    plan = device.DevicePlan(kind=_lib.TB_PRECOND_HBMC, n=hl.n_pad, n_real=hl.n,
                             inv_d=sf.inv_diag, spmv_format=_lib.TB_SPMV_NONE,
                             w=sf.w, b_s=sf.b_s,
                             color_lvl1_ranges=hl.color_lvl1_ranges,
                             L_sell=sf.lower, U_sell=sf.upper)
    cache[id(hl)] = (hl, plan)
    return plan


def release_plans(f):
    """Free the device plans the sub_*/apply_* calls cached on factor `f`."""
    for _, plan in f.__dict__.pop("_tb_plans", {}).values():
        plan.close()


def _count(counter, phases):
    counter.start()
    for idx, c in enumerate(phases):
        counter.enter_phase(c)
        if idx < len(phases) - 1:
            counter.barrier()


def _run(plan, fn_name, v, n):
    from . import device
    vt, was_np = device.vec_in(v, n)
    out = device.empty(n)
    getattr(plan, fn_name)(vt, out)
    return device.vec_out(out, was_np)


def sub_forward_seq(f: IcFactor, r, kernels=None):
    """src/precond.py:285-290 (device, dependency-level schedule)."""
    return _run(_task_plan(f, "seq", None), "forward", r, f.n)


def sub_backward_seq(f: IcFactor, y, kernels=None):
    """src/precond.py:293-298."""
    return _run(_task_plan(f, "seq", None), "backward", y, f.n)


def sub_forward_mc(f: IcFactor, coloring, r, pool=None, counter=None, kernels=None):
    """src/precond.py:320-326."""
    _require_tag(f, "mc")
    out = _run(_task_plan(f, "mc", coloring), "forward", r, f.n)
    _count(counter or _NULL, list(range(coloring.n_c)))
    return out


def sub_backward_mc(f: IcFactor, coloring, y, pool=None, counter=None, kernels=None):
    """src/precond.py:329-335."""
    _require_tag(f, "mc")
    out = _run(_task_plan(f, "mc", coloring), "backward", y, f.n)
    _count(counter or _NULL, list(range(coloring.n_c - 1, -1, -1)))
    return out


def sub_forward_bmc(f: IcFactor, layout, r, pool=None, counter=None, kernels=None):
    """src/precond.py:361-366."""
    _require_tag(f, "bmc")
    out = _run(_task_plan(f, "bmc", layout), "forward", r, f.n)
    _count(counter or _NULL, list(range(layout.n_c)))
    return out


def sub_backward_bmc(f: IcFactor, layout, y, pool=None, counter=None, kernels=None):
    """src/precond.py:369-374."""
    _require_tag(f, "bmc")
    out = _run(_task_plan(f, "bmc", layout), "backward", y, f.n)
    _count(counter or _NULL, list(range(layout.n_c - 1, -1, -1)))
    return out


def sub_forward_hbmc(sf: SellFactor, hl, r, pool=None, counter=None, kernels=None):
    """src/precond.py:395-400: one device phase per color, ascending."""
    _require_tag(sf, "hbmc")
    out = _run(_hbmc_plan(sf, hl), "forward", r, hl.n_pad)
    _count(counter or _NULL, list(range(hl.n_c)))
    return out


def sub_backward_hbmc(sf: SellFactor, hl, y, pool=None, counter=None, kernels=None):
    """src/precond.py:403-408: colors descending."""
    _require_tag(sf, "hbmc")
    out = _run(_hbmc_plan(sf, hl), "backward", y, hl.n_pad)
    _count(counter or _NULL, list(range(hl.n_c - 1, -1, -1)))
    return out


def apply_ic_preconditioner(kind, f, layout, r, pool=None, counter=None, kernels=None):
    """src/precond.py:411-425: z = (L L^T)^-1 r via the selected pair."""
    if kind in ("seq", "natural"):
        return sub_backward_seq(f, sub_forward_seq(f, r))
    if kind == "mc":
        y = sub_forward_mc(f, layout, r, pool, counter)
        return sub_backward_mc(f, layout, y, pool, counter)
    if kind == "bmc":
        y = sub_forward_bmc(f, layout, r, pool, counter)
        return sub_backward_bmc(f, layout, y, pool, counter)
    if kind == "hbmc":
        y = sub_forward_hbmc(f, layout, r, pool, counter)
        return sub_backward_hbmc(f, layout, y, pool, counter)
    raise ValueError(f"unknown kernel selector {kind!r}")
