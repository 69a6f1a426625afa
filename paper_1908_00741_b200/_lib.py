"""ctypes binding of libhbmc_b200.so (the C ABI in include/hbmc_b200.h).

This is the only way the package reaches native code.  If the library is
missing it is built in-tree when nvcc is available; otherwise importing the
package fails loudly -- there is no Python or CPU fallback for any operator.
"""

import ctypes as C
import os

import numpy as np

from . import _build

TB_OK = 0
TB_EINVAL = 1
TB_EIC_BREAKDOWN = 2
TB_ECG_BREAKDOWN = 3
TB_ECUDA = 4
TB_ENOMEM = 5
TB_EDUP = 6
TB_ENODEV = 7

TB_PRECOND_HBMC = 0
TB_PRECOND_TASKS = 1
TB_SPMV_SELL = 0
TB_SPMV_CSR = 1
TB_SPMV_NONE = 2

ABI_VERSION = 3
TB_PLAN_PARTITIONED = 1

i64 = C.c_int64
i32 = C.c_int32
dbl = C.c_double
vp = C.c_void_p
P_i64 = C.POINTER(i64)
P_dbl = C.POINTER(dbl)


class TbSellHost(C.Structure):
    _fields_ = [("n_slices", i64), ("width", i64), ("slice_ptr", vp),
                ("slice_len", vp), ("col_idx", vp), ("vals", vp)]


class TbCsrHost(C.Structure):
    _fields_ = [("n", i64), ("row_ptr", vp), ("col_idx", vp), ("vals", vp)]


class TbSchedHost(C.Structure):
    _fields_ = [("n_phases", i64), ("phase_ptr", vp), ("task_ptr", vp),
                ("rows", vp), ("n_rows", i64)]


class TbPlanDesc(C.Structure):
    _fields_ = [("precond_kind", i32), ("spmv_format", i32), ("n", i64),
                ("n_real", i64), ("inv_d", vp), ("w", i64), ("b_s", i64),
                ("n_c", i64), ("color_lvl1_ranges", vp),
                ("L_sell", TbSellHost), ("U_sell", TbSellHost),
                ("L_csr", TbCsrHost), ("U_csr", TbCsrHost),
                ("fwd_sched", TbSchedHost), ("bwd_sched", TbSchedHost),
                ("A_sell", TbSellHost), ("A_csr", TbCsrHost), ("flags", i64),
                ("real_pos", vp)]


TB_MAX_PEERS = 16


class TbPushDesc(C.Structure):
    _fields_ = [("row0", i64), ("nrows", i64), ("ptr", vp), ("peer", vp), ("off", vp),
                ("npeers", i32), ("peer_dst", vp * TB_MAX_PEERS),
                ("peer_flag", vp * TB_MAX_PEERS), ("epoch", C.c_uint32), ("done_ctr", vp)]


class TbPcgReport(C.Structure):
    _fields_ = [("iterations", i64), ("converged", i32), ("status", i32),
                ("breakdown_iter", i64), ("breakdown_value", dbl),
                ("kernel_launches", i64), ("host_syncs", i64)]


# name -> (restype, argtypes); every function returns an int status
_SIGS = {
    "tb_abi_version": [],
    "tb_grow_blocks": [i64, vp, vp, i64, vp, P_i64],
    "tb_color_block_graph": [i64, vp, vp, vp, i64, vp, vp, vp],
    "tb_greedy_color": [i64, vp, vp, vp],
    "tb_ic0_factor": [i64, vp, vp, vp, vp, vp, vp, P_i64, P_dbl],
    "tb_llt_on_pattern": [i64, vp, vp, vp, vp, vp, vp],
    "tb_group_by_label": [i64, vp, i64, vp, vp],
    "tb_pad_colors_count": [i64, vp, i64, i64, vp, P_i64],
    "tb_pad_colors_fill": [i64, i64, vp, vp, vp, vp, i64, i64, vp, i64, P_i64],
    "tb_hbmc_compose": [i64, vp, i64, i64, vp, vp],
    "tb_coo_to_csr": [i64, i64, vp, vp, vp, vp, vp, vp, P_i64, P_i64],
    "tb_permute_csr": [i64, vp, vp, vp, vp, vp, vp, vp],
    "tb_csr_transpose": [i64, vp, vp, vp, vp, vp, vp],
    "tb_csr_to_sell_fill": [i64, vp, vp, vp, i64, i64, vp, vp, vp, vp],
    "tb_spmv_csr_host": [i64, vp, vp, vp, vp, vp],
    "tb_level_schedule": [i64, vp, vp, C.c_int, vp, P_i64],
    "tb_dev_spmv_sell": [i64, vp, vp, vp, vp, i64, vp, vp, vp],
    "tb_dev_spmv_csr": [i64, vp, vp, vp, vp, vp, vp],
    "tb_dev_fwd_sell_range": [vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, vp],
    "tb_dev_bwd_sell_range": [vp, vp, vp, vp, vp, vp, vp, i64, i64, i64, i64, vp],
    "tb_dev_csr_sweep_tasks": [C.c_int, vp, vp, vp, vp, vp, vp, i64, i64, vp, vp, vp],
    "tb_plan_create": [C.POINTER(TbPlanDesc), C.c_int, C.POINTER(vp)],
    "tb_plan_destroy": [vp],
    "tb_plan_device_bytes": [vp, P_i64],
    "tb_plan_forward": [vp, vp, vp, vp],
    "tb_plan_backward": [vp, vp, vp, vp],
    "tb_plan_precond": [vp, vp, vp, vp],
    "tb_plan_spmv": [vp, vp, vp, vp],
    "tb_plan_barriers_per_sweep": [vp, P_i64],
    "tb_plan_sweep_phase": [vp, C.c_int, i64, vp, vp, vp],
    "tb_plan_trace": [vp, vp],
    "tb_plan_persistent": [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32)],
    "tb_plan_flow_info": [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i64)],
    "tb_plan_phase_info": [vp, C.c_int, i64, C.POINTER(i32), C.POINTER(i32),
                           C.POINTER(i32), C.POINTER(i32)],
    "tb_pcg": [vp, vp, vp, dbl, i64, i64, vp, C.POINTER(TbPcgReport), vp],
    "tb_dev_gather": [i64, vp, vp, vp, vp],
    "tb_dev_dot": [i64, vp, vp, vp, i32, vp, vp],
    "tb_dev_cg_xr": [i64, vp, i32, i32, vp, vp, vp, vp, i32, vp, vp],
    "tb_dev_cg_p": [i64, vp, i32, i32, vp, vp, vp],
    "tb_plan_sweep_phase_push": [vp, C.c_int, i64, vp, vp, C.POINTER(TbPushDesc), vp],
    "tb_dev_cg_p_push": [i64, vp, i32, i32, vp, vp, C.POINTER(TbPushDesc), vp],
    "tb_csr_diag_ptr": [i64, vp, vp, vp],
    "tb_csr_is_symmetric": [i64, vp, vp, C.POINTER(i32)],
    "tb_csr_tri_count": [i64, vp, vp, i32, vp],
    "tb_csr_tri_fill": [i64, vp, vp, vp, i32, vp, vp, vp],
    "tb_p2p_alloc": [i64, C.POINTER(vp), vp],
    "tb_p2p_free": [vp],
    "tb_p2p_open": [vp, C.POINTER(vp)],
    "tb_p2p_close": [vp],
    "tb_p2p_push": [i64, vp, vp, vp, vp, C.c_uint32, vp, vp],
    "tb_p2p_wait": [vp, i32, i32, C.c_uint32, vp],
    "tb_mm_locate": [vp, i64, P_i64, P_i64, P_i64, P_i64, P_i64],
    "tb_mm_entries": [vp, i64, i64, i64, i64, vp, vp, vp, vp, P_i64, P_i64,
                      C.POINTER(i32), P_i64, P_i64, P_i64],
    "tb_dev_ic0_hbmc": [i64, vp, vp, vp, vp, vp, vp, i64, i64, i64, vp, vp, P_i64, P_dbl, vp],
}

EXPORTED = sorted(_SIGS) + ["tb_last_error"]


def _load():
    path = _build.LIB
    if not os.path.exists(path) or _build.needs_build():
        try:
            _build.build()
        except Exception as exc:  # no nvcc on this box and no prebuilt .so
            if not os.path.exists(path):
                raise ImportError(
                    f"libhbmc_b200.so is missing and could not be built ({exc}); "
                    "run `python -c 'import __graft_entry__ as g; g.build()'`"
                ) from exc
    lib = C.CDLL(path)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = C.c_int
        fn.argtypes = args
    lib.tb_last_error.restype = C.c_char_p
    lib.tb_last_error.argtypes = []
    if lib.tb_abi_version() != ABI_VERSION:
        raise ImportError("libhbmc_b200.so ABI version mismatch; rebuild it")
    return lib


LIB = _load()
LIB_PATH = _build.LIB


class NativeError(RuntimeError):
    def __init__(self, code, message):
        self.code = code
        super().__init__(message)


def last_error():
    return LIB.tb_last_error().decode("utf-8", "replace")


def check(rc):
    """Map a non-zero status to an exception (the caller refines breakdowns)."""
    if rc == TB_OK:
        return
    msg = last_error()
    if rc in (TB_EINVAL, TB_EDUP):
        raise ValueError(msg)
    if rc == TB_ENOMEM:
        raise MemoryError(msg)
    raise NativeError(rc, msg)


def ptr(a):
    """Raw data pointer of a contiguous numpy array or torch tensor."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    return a.data_ptr()


def i64a(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def f64a(a):
    return np.ascontiguousarray(a, dtype=np.float64)
