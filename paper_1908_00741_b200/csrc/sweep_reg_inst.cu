// Instantiations of the register-pipelined HBMC sweep for one (direction,
// b_s) pair, selected by -DTB_FWD and -DTB_BS (see _build.py): splitting the
// 60 shapes over 6 translation units lets the build compile them in parallel.
#include <cuda_runtime.h>

#include "sweep_reg.cuh"

#ifndef TB_FWD
#error "compile with -DTB_FWD=0|1 -DTB_BS=4|8|16"
#endif

#define TB_CAT3(a, b, c) a##b##c
#define TB_SELECT_NAME(D, B) TB_CAT3(select_, D, _##B)

namespace sweep_reg {
#if TB_FWD
#define TB_DIR fwd
#else
#define TB_DIR bwd
#endif
#define TB_EXPAND(D, B) TB_SELECT_NAME(D, B)
KernelFn TB_EXPAND(TB_DIR, TB_BS)(int maxl, int pf) {
  return pick_maxl<TB_FWD != 0, TB_BS>(maxl, pf);
}
}  // namespace sweep_reg
