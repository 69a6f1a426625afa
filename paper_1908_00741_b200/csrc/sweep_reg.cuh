// HBMC substitution sweep, register-pipelined version (sm_100a).
//
// Same arithmetic as K/numba_backend.py:132-171 (bitwise).  Mapping as in
// sell_sweep: one thread per (level-1 block k, lane j), j = one BMC block;
// the thread walks its b_s rows.  The difference is the schedule: with b_s
// (B_S) and the phase's maximum slice length (MAXL) known at compile time the
// whole walk is unrolled and software-pipelined in registers:
//
//   * the slice offsets and lengths of all B_S steps are loaded up front (one
//     batch; slices may be stored in any order, e.g. step-major);
//   * the column / value / rhs / inv_d loads of step l + PF are issued while
//     step l computes (PF = prefetch distance; PF = B_S loads everything at
//     once when it fits the register budget);
//   * the cross-color gathers of step l + 1 are issued before step l's chain,
//     so their L2 latency overlaps the chain;
//   * in-block operands (same lane, earlier step) come from the thread's own
//     results, held in registers and selected by step index.
// Slot order, __dmul_rn products and __dsub_rn updates are the reference's,
// and a padding slot (col == own row, v == 0) multiplies the in-progress
// value exactly as the reference does.

#pragma once

namespace sweep_reg {

template <int B_S>
__device__ __forceinline__ double pick(const double (&h)[B_S], int idx) {
  double r = 0.0;
#pragma unroll
  for (int u = 0; u < B_S; ++u)
    if (u == idx) r = h[u];
  return r;
}

template <bool FWD, int B_S, int MAXL, int PF>
__global__ void __launch_bounds__(256)
    sweep_kernel(const long long *__restrict__ slice_ptr, const int *__restrict__ slice_len,
                 const int *__restrict__ col,
                 const double *__restrict__ val, const double *__restrict__ inv_d,
                 const double *__restrict__ src, double *__restrict__ dst, int w,
                 long long k0, long long nthreads, const int *done) {
  if (done && *(const volatile int *)done) return;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nthreads) return;
  const long long k = k0 + g / w;
  const int j = (int)(g % w);
  const long long blk_row0 = k * B_S * w;
  const long long blk_row1 = blk_row0 + (long long)B_S * w;

  // step order: forward l = 0..B_S-1, backward l = B_S-1..0; index i is the
  // position in the walk, step(i) the slice within the block.
  long long off[B_S];
  int lens[B_S];
#pragma unroll
  for (int u = 0; u < B_S; ++u) {
    off[u] = slice_ptr[k * B_S + u];
    lens[u] = slice_len[k * B_S + u];
  }

  int c[B_S][MAXL];
  double v[B_S][MAXL];
  double rr[B_S], id[B_S], x[B_S][MAXL], hist[B_S];
#pragma unroll
  for (int u = 0; u < B_S; ++u) hist[u] = 0.0;

  auto load_step = [&](int i) {
    const int l = FWD ? i : B_S - 1 - i;
    const int len = lens[l];
    const long long base = off[l] + j;
#pragma unroll
    for (int t = 0; t < MAXL; ++t) {
      if (t < len) {
        c[i][t] = __ldg(col + base + (long long)t * w);
        v[i][t] = __ldg(val + base + (long long)t * w);
      } else {
        c[i][t] = -1;
        v[i][t] = 0.0;
      }
    }
    const long long row = blk_row0 + (long long)l * w + j;
    rr[i] = __ldg(src + row);
    id[i] = __ldg(inv_d + row);
  };
  auto gather_step = [&](int i) {
#pragma unroll
    for (int t = 0; t < MAXL; ++t) {
      const long long cc = c[i][t];
      const bool cross = cc >= 0 && (cc < blk_row0 || cc >= blk_row1);
      x[i][t] = cross ? __ldg(dst + cc) : 0.0;
    }
  };

#pragma unroll
  for (int i = 0; i < (PF < B_S ? PF : B_S); ++i) load_step(i);
  gather_step(0);
#pragma unroll
  for (int i = 0; i < B_S; ++i) {
    if (i + PF < B_S) load_step(i + PF);
    if (i + 1 < B_S) gather_step(i + 1);
    const int l = FWD ? i : B_S - 1 - i;
    const long long row = blk_row0 + (long long)l * w + j;
    double y = rr[i];
#pragma unroll
    for (int t = 0; t < MAXL; ++t) {
      const long long cc = c[i][t];
      if (cc >= 0) {
        double prod;
        if (cc < blk_row0 || cc >= blk_row1) {
          prod = __dmul_rn(v[i][t], x[i][t]);
        } else if (cc == row) {
          prod = __dmul_rn(v[i][t], y);
        } else {
          // in-block: same lane, step lp, which the walk produced at i' =
          // (FWD ? lp : B_S-1-lp)
          const int lp = (int)((cc - blk_row0) / w);
          prod = __dmul_rn(v[i][t], pick<B_S>(hist, FWD ? lp : B_S - 1 - lp));
        }
        y = __dsub_rn(y, prod);
      }
    }
    y = __dmul_rn(y, id[i]);
    hist[i] = y;
    dst[row] = y;
  }
}

// ---- dispatch over the compiled shapes (instantiated in sweep_reg_*.cu)
using KernelFn = void (*)(const long long *, const int *, const int *, const double *,
                          const double *,
                          const double *, double *, int, long long, long long, const int *);

// Prefetch distances compiled per MAXL: everything up front for the light
// phases (MAXL <= 2), else 1 or 2 steps ahead.
template <bool FWD, int B_S, int MAXL>
inline KernelFn pick_pf(int pf) {
  if (MAXL <= 2) return pf >= B_S ? sweep_kernel<FWD, B_S, MAXL, B_S> : sweep_kernel<FWD, B_S, MAXL, 2>;
  return pf >= 2 ? sweep_kernel<FWD, B_S, MAXL, 2> : sweep_kernel<FWD, B_S, MAXL, 1>;
}
template <bool FWD, int B_S>
inline KernelFn pick_maxl(int maxl, int pf) {
  switch (maxl) {
    case 1: return pick_pf<FWD, B_S, 1>(pf);
    case 2: return pick_pf<FWD, B_S, 2>(pf);
    case 4: return pick_pf<FWD, B_S, 4>(pf);
    case 8: return pick_pf<FWD, B_S, 8>(pf);
    case 16: return pick_pf<FWD, B_S, 16>(pf);
  }
  return nullptr;
}
// One (direction, b_s) pair per translation unit: sweep_reg_inst.cu is
// compiled once per pair with -DTB_FWD=0/1 -DTB_BS=4/8/16.
#define TB_DECL_SELECT(D, B) KernelFn select_##D##_##B(int maxl, int pf);
TB_DECL_SELECT(fwd, 4) TB_DECL_SELECT(fwd, 8) TB_DECL_SELECT(fwd, 16)
TB_DECL_SELECT(bwd, 4) TB_DECL_SELECT(bwd, 8) TB_DECL_SELECT(bwd, 16)
#undef TB_DECL_SELECT

// b_s in {4, 8, 16}, maxl in {1, 2, 4, 8, 16}; nullptr if not compiled
template <bool FWD>
inline KernelFn select(int b_s, int maxl, int pf) {
  switch (b_s) {
    case 4: return FWD ? select_fwd_4(maxl, pf) : select_bwd_4(maxl, pf);
    case 8: return FWD ? select_fwd_8(maxl, pf) : select_bwd_8(maxl, pf);
    case 16: return FWD ? select_fwd_16(maxl, pf) : select_bwd_16(maxl, pf);
  }
  return nullptr;
}

}  // namespace sweep_reg
