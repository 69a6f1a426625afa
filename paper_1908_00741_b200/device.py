"""Device plumbing: torch CUDA buffers, streams and the native plan handle.

PyTorch provides device memory and the current stream; every operator is a
kernel in libhbmc_b200.so called through the C ABI.  Without a CUDA device
every entry point here raises -- there is no CPU fallback.
"""

import ctypes as C
import os

import numpy as np

from . import _lib
from ._lib import LIB, check, ptr

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(
            "paper_1908_00741_b200: a CUDA device (B200) is required; this "
            "operator has no CPU implementation")
    return t


def current_stream():
    t = require_cuda()
    return t.cuda.current_stream().cuda_stream


def is_cuda_tensor(x):
    t = torch() if _torch is not None or _has_torch() else None
    return t is not None and isinstance(x, t.Tensor) and x.is_cuda


def _has_torch():
    try:
        torch()
        return True
    except ImportError:
        return False


# ------------------------------------------------------------------ host I/O
# numpy <-> device copies of large vectors go through a cached pinned buffer:
# the pageable <-> pinned copies are split over a thread pool (numpy releases
# the GIL inside copyto) and the DMA runs from / to pinned memory at full
# link speed.  A caller of apply_ic_preconditioner(numpy r) on config 5 moves
# 1 GiB each way per call; pageable torch copies did that at ~2 GB/s.
_STAGE_MIN = 4 << 20          # bytes: smaller vectors take the plain path
_stage = {"buf": None, "pool": None}


def _pinned(nbytes):
    t = require_cuda()
    buf = _stage["buf"]
    if buf is None or buf.numel() < nbytes:
        _stage["buf"] = buf = t.empty(int(nbytes), dtype=t.uint8, pin_memory=True)
    return buf


def _par_copy(dst, src):
    """dst[:] = src for 1-D numpy arrays of equal size, split over threads."""
    import concurrent.futures as cf
    n = dst.shape[0]
    k = min(16, os.cpu_count() or 1, max(1, n // (1 << 18)))
    if k <= 1:
        np.copyto(dst, src)
        return
    if _stage["pool"] is None:
        _stage["pool"] = cf.ThreadPoolExecutor(max_workers=16)
    bounds = [n * i // k for i in range(k + 1)]
    list(_stage["pool"].map(lambda i: np.copyto(dst[bounds[i]:bounds[i + 1]],
                                                src[bounds[i]:bounds[i + 1]]), range(k)))


def to_device(a, dtype=None):
    """numpy -> CUDA tensor (contiguous copy)."""
    t = require_cuda()
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    if arr.nbytes < _STAGE_MIN or arr.ndim != 1:
        return t.from_numpy(arr).to("cuda", non_blocking=False)
    pin = _pinned(arr.nbytes)
    host = pin[: arr.nbytes].numpy().view(arr.dtype)
    t.cuda.current_stream().synchronize()   # the buffer may still feed a D2H
    _par_copy(host, arr)
    out = t.empty(arr.shape[0], dtype=t.from_numpy(arr[:1]).dtype, device="cuda")
    out.copy_(pin[: arr.nbytes].view(out.dtype), non_blocking=True)
    t.cuda.current_stream().synchronize()   # the pinned buffer is reused next call
    return out


def empty(n, dtype="f64"):
    """Output buffer.  TB_POISON=1 (set by the test suite) fills it with NaN
    so a kernel that leaves an entry unwritten, or reads its own output
    before writing it, cannot pass on stale memory from the allocator."""
    t = require_cuda()
    dt = {"f64": t.float64, "i32": t.int32, "i64": t.int64}[dtype]
    if os.environ.get("TB_POISON") == "1" and dtype == "f64":
        return t.full((int(n),), float("nan"), dtype=dt, device="cuda")
    return t.empty(int(n), dtype=dt, device="cuda")


def vec_in(x, n):
    """Accept numpy or CUDA tensor of length n; returns (tensor, was_numpy)."""
    t = require_cuda()
    if isinstance(x, t.Tensor):
        if not x.is_cuda:
            x = x.to("cuda")
        if x.dtype != t.float64:
            x = x.to(t.float64)
        x = x.contiguous()
        if x.shape[0] != n:
            raise ValueError(f"vector length {x.shape[0]}, expected {n}")
        return x, False
    a = np.ascontiguousarray(x, dtype=np.float64)
    if a.shape[0] != n:
        raise ValueError(f"vector length {a.shape[0]}, expected {n}")
    return to_device(a), True


def vec_out(tensor, as_numpy):
    if not as_numpy:
        return tensor
    t = require_cuda()
    nbytes = tensor.numel() * tensor.element_size()
    if nbytes < _STAGE_MIN or tensor.dim() != 1 or not tensor.is_cuda:
        return tensor.cpu().numpy()
    pin = _pinned(nbytes)
    pin[:nbytes].view(tensor.dtype).copy_(tensor, non_blocking=True)
    t.cuda.current_stream().synchronize()
    out = np.empty(tensor.numel(), dtype=np.dtype(str(tensor.dtype).replace("torch.", "")))
    _par_copy(out, pin[:nbytes].numpy().view(out.dtype))
    return out


# ------------------------------------------------------------------ matrices
class DeviceSell:
    """Device copy of a SellMatrix (int32 columns)."""

    def __init__(self, s):
        self.n_slices = s.n_slices
        self.width = s.width
        self.n = s.n
        self.n_pad = s.n_pad
        self.slice_ptr = to_device(s.slice_ptr, np.int64)
        self.slice_len = to_device(s.slice_len, np.int32)
        self.col = to_device(s.col32, np.int32)
        self.vals = to_device(s.vals, np.float64)


class DeviceCsr:
    def __init__(self, a):
        self.n = a.n
        self.row_ptr = to_device(a.row_ptr, np.int64)
        self.col = to_device(a.col_idx, np.int32)
        self.vals = to_device(a.vals, np.float64)


def device_copy(obj):
    """Cached device copy of a (never mutated) CsrMatrix / SellMatrix."""
    from .matrix import CsrMatrix, SellMatrix
    dev = getattr(obj, "_tb_dev", None)
    if dev is None:
        if isinstance(obj, SellMatrix):
            dev = DeviceSell(obj)
        elif isinstance(obj, CsrMatrix):
            dev = DeviceCsr(obj)
        else:
            raise TypeError(f"spmv: unsupported matrix type {type(obj).__name__}")
        object.__setattr__(obj, "_tb_dev", dev)
    return dev


def spmv(a, x):
    """src/matrix.py:307-323 on the device."""
    from .matrix import CsrMatrix, SellMatrix
    t = require_cuda()
    if isinstance(a, SellMatrix):
        xt, was_np = vec_in_pad(x, a.n_pad)
        d = device_copy(a)
        out = empty(a.n_pad)
        check(LIB.tb_dev_spmv_sell(d.n_slices, ptr(d.slice_ptr), ptr(d.slice_len),
                                   ptr(d.col), ptr(d.vals), d.width, ptr(xt),
                                   ptr(out), current_stream()))
        return vec_out(out[:a.n], was_np)
    if isinstance(a, CsrMatrix):
        xt, was_np = vec_in(x, a.n)
        d = device_copy(a)
        out = empty(a.n)
        check(LIB.tb_dev_spmv_csr(a.n, ptr(d.row_ptr), ptr(d.col), ptr(d.vals),
                                  ptr(xt), ptr(out), current_stream()))
        return vec_out(out, was_np)
    del t
    raise TypeError(f"spmv: unsupported matrix type {type(a).__name__}")


def vec_in_pad(x, n_pad):
    t = require_cuda()
    if isinstance(x, t.Tensor):
        xt, was = vec_in(x, x.shape[0])
    else:
        a = np.ascontiguousarray(x, dtype=np.float64)
        xt, was = to_device(a), True
    if xt.shape[0] < n_pad:
        xp = t.zeros(n_pad, dtype=t.float64, device="cuda")
        xp[:xt.shape[0]] = xt
        xt = xp
    return xt, was


# ------------------------------------------------------------------ plans
def _sell_host(s, keep):
    """tb_sell_host view of a SellMatrix (arrays kept alive in `keep`)."""
    sp = np.ascontiguousarray(s.slice_ptr, dtype=np.int64)
    sl = np.ascontiguousarray(s.slice_len, dtype=np.int32)
    col = np.ascontiguousarray(s.col32, dtype=np.int32)
    v = np.ascontiguousarray(s.vals, dtype=np.float64)
    keep.extend([sp, sl, col, v])
    return _lib.TbSellHost(s.n_slices, s.width, ptr(sp), ptr(sl), ptr(col), ptr(v))


def _csr_host(a, keep):
    rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(a.col_idx, dtype=np.int32)
    v = np.ascontiguousarray(a.vals, dtype=np.float64)
    keep.extend([rp, col, v])
    return _lib.TbCsrHost(a.n, ptr(rp), ptr(col), ptr(v))


def _sched_host(sched, keep):
    if sched is None:
        return _lib.TbSchedHost(0, None, None, None, 0)
    phase_ptr, task_ptr, rows = sched
    pp = np.ascontiguousarray(phase_ptr, dtype=np.int64)
    keep.append(pp)
    tp_ptr = None
    if task_ptr is not None:   # None = one row per task
        tp = np.ascontiguousarray(task_ptr, dtype=np.int64)
        keep.append(tp)
        tp_ptr = ptr(tp)
    rp = None
    nr = 0
    if rows is not None:
        rr = np.ascontiguousarray(rows, dtype=np.int64)
        keep.append(rr)
        rp = ptr(rr)
        nr = rr.shape[0]
    return _lib.TbSchedHost(pp.shape[0] - 1, ptr(pp), tp_ptr, rp, nr)


class DevicePlan:
    """Owns a tb_plan: factor(s), A and the solver vectors resident in HBM."""

    def __init__(self, *, kind, n, n_real, inv_d, spmv_format,
                 w=0, b_s=0, color_lvl1_ranges=None, L_sell=None, U_sell=None,
                 L_csr=None, U_csr=None, fwd_sched=None, bwd_sched=None,
                 A_sell=None, A_csr=None, device=None, partitioned=False, real_pos=None):
        t = require_cuda()
        self.handle = None
        keep = []
        desc = _lib.TbPlanDesc()
        desc.precond_kind = kind
        desc.spmv_format = spmv_format
        desc.n = n
        desc.n_real = n_real
        desc.flags = _lib.TB_PLAN_PARTITIONED if partitioned else 0
        if real_pos is not None and 0 < n_real < n:
            rp = np.ascontiguousarray(real_pos, dtype=np.int64)
            if rp.shape[0] != n_real:
                raise ValueError("real_pos length must equal n_real")
            keep.append(rp)
            desc.real_pos = ptr(rp)
        inv = np.ascontiguousarray(inv_d, dtype=np.float64)
        keep.append(inv)
        desc.inv_d = ptr(inv)
        if kind == _lib.TB_PRECOND_HBMC:
            cr = np.ascontiguousarray(color_lvl1_ranges, dtype=np.int64)
            keep.append(cr)
            desc.w, desc.b_s, desc.n_c = w, b_s, cr.shape[0] - 1
            desc.color_lvl1_ranges = ptr(cr)
            desc.L_sell = _sell_host(L_sell, keep)
            desc.U_sell = _sell_host(U_sell, keep)
        else:
            desc.L_csr = _csr_host(L_csr, keep)
            desc.U_csr = _csr_host(U_csr, keep)
            desc.fwd_sched = _sched_host(fwd_sched, keep)
            desc.bwd_sched = _sched_host(bwd_sched, keep)
        if spmv_format == _lib.TB_SPMV_SELL:
            desc.A_sell = _sell_host(A_sell, keep)
        elif spmv_format == _lib.TB_SPMV_CSR:
            desc.A_csr = _csr_host(A_csr, keep)
        self.device = t.cuda.current_device() if device is None else device
        h = C.c_void_p()
        check(LIB.tb_plan_create(C.byref(desc), self.device, C.byref(h)))
        self.handle = h
        self.n = n
        self.n_real = n_real
        self.kind = kind

    def close(self):
        if self.handle is not None:
            LIB.tb_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- operators on CUDA tensors (length n, float64, contiguous)
    def forward(self, r, y, stream=None):
        check(LIB.tb_plan_forward(self.handle, ptr(r), ptr(y),
                                  stream if stream is not None else current_stream()))

    def backward(self, y, z, stream=None):
        check(LIB.tb_plan_backward(self.handle, ptr(y), ptr(z),
                                   stream if stream is not None else current_stream()))

    def precond(self, r, z, stream=None):
        check(LIB.tb_plan_precond(self.handle, ptr(r), ptr(z),
                                  stream if stream is not None else current_stream()))

    def spmv(self, x, y, stream=None):
        check(LIB.tb_plan_spmv(self.handle, ptr(x), ptr(y),
                               stream if stream is not None else current_stream()))

    def sweep_phase(self, forward, phase, src, dst, stream=None):
        check(LIB.tb_plan_sweep_phase(self.handle, 1 if forward else 0, int(phase),
                                      ptr(src), ptr(dst),
                                      stream if stream is not None else current_stream()))

    def sweep_phase_push(self, forward, phase, src, dst, desc, stream=None):
        """One color phase with the halo push fused in (tb_plan_sweep_phase_push)."""
        check(LIB.tb_plan_sweep_phase_push(self.handle, 1 if forward else 0, int(phase),
                                           ptr(src), ptr(dst), C.byref(desc),
                                           stream if stream is not None else current_stream()))

    def phase_info(self, forward, phase):
        vals = [_lib.i32() for _ in range(4)]
        check(LIB.tb_plan_phase_info(self.handle, 1 if forward else 0, int(phase), *vals))
        return dict(zip(("staged", "warps", "grid", "max_slots"), (v.value for v in vals)))

    def persistent(self):
        vals = [_lib.i32() for _ in range(3)]
        check(LIB.tb_plan_persistent(self.handle, *vals))
        return dict(zip(("precond", "pcg", "grid"), (v.value for v in vals)))

    def flow_info(self):
        """Item-pipelined dataflow preconditioner kernel: grid (0 = not used), stages, smem."""
        g, st, sm = _lib.i32(), _lib.i32(), _lib.i64()
        check(LIB.tb_plan_flow_info(self.handle, g, st, sm))
        return {"grid": g.value, "stages": st.value, "smem": sm.value}

    def barriers_per_sweep(self):
        v = _lib.i64()
        check(LIB.tb_plan_barriers_per_sweep(self.handle, v))
        return v.value

    def device_bytes(self):
        v = _lib.i64()
        check(LIB.tb_plan_device_bytes(self.handle, v))
        return v.value

    def pcg(self, b, x, tol, max_iters, stream=None):
        """Device-resident PCG; returns (report struct, history ndarray)."""
        rep = _lib.TbPcgReport()
        hist = np.empty(max_iters + 1)
        rc = LIB.tb_pcg(self.handle, ptr(b), ptr(x), float(tol), int(max_iters), 0,
                        stream if stream is not None else current_stream(),
                        C.byref(rep), ptr(hist))
        if rc not in (_lib.TB_OK, _lib.TB_ECG_BREAKDOWN):
            check(rc)
        return rep, hist[:rep.iterations + 1].copy()
