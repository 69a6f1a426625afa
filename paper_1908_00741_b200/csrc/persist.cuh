// Persistent cooperative kernels for the HBMC ICCG path (sm_100a).
//
// One launch runs a whole preconditioner application (mode PRECOND) or a
// whole PCG solve (mode PCG, src/solver.py:157-193): every phase that used to
// be a kernel boundary -- a color phase of a sweep, the SpMV, a vector
// update, a dot product -- is separated by a software grid barrier instead.
// The grid is exactly the co-resident CTA count (cooperative launch), so the
// barrier cannot deadlock; it also carries a clock64 watchdog that traps
// (kernel error) instead of hanging the GPU if it ever waited for seconds.
//
// Arithmetic is the same as the per-phase kernels (and the reference):
//   * sweep rows: y = rhs; y = y - v*x in stored slot order (__dmul_rn,
//     __dsub_rn); y *= inv_d  (K/numba_backend.py:132-171);
//   * SpMV rows: acc = 0; acc = acc + v*x (K/numba_backend.py:26-37);
//   * x += alpha p; r -= alpha ap; p = z + beta p with separate roundings.
// Dot products: per-thread partials in a fixed grid-stride order, a fixed
// CTA tree, then EVERY CTA sums the CTA partials in index order -- so every
// CTA computes bitwise-identical alpha / beta / residuals and takes the same
// branch at every convergence test.
// Vectors written inside the launch are read with ld.global.cg (never a
// possibly stale L1 line); the factor / matrix arrays with the read-only path.

#pragma once

#include "sweep_lean.cuh"

namespace persist {

constexpr int kThreads = 256;
constexpr int kSlots = 4;  // reduction slots (bb / pap / rr / rz)

struct Params {
  int mode;      // 0 = preconditioner only (src -> dst), 1 = full PCG
  int n;         // system size (n_pad)
  int w, b_s, n_c;
  const int *color_lvl1;  // [n_c+1] level-1 block ranges per color
  // factor (SELL, slice width w; int32 offsets fit: checked on the host)
  const long long *Lsp, *Usp;
  const int *Lsl, *Usl, *Lcol, *Ucol;
  const double *Lval, *Uval;
  const double *inv_d;
  // matrix A (SELL, slice width aw)
  const long long *Asp;
  const int *Asl, *Acol;
  const double *Aval;
  int aw;
  // vectors
  const double *b;
  double *x, *r, *y, *z, *p, *ap;
  const double *pre_src;  // mode 0
  double *pre_dst;
  double *hist;
  double *partials;       // [kSlots][gridDim.x]
  unsigned *bar_count, *bar_gen;
  void *state;            // PcgState*
  long long watchdog;     // cycles
};

__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }

// ---------------------------------------------------------------- barrier
__device__ __forceinline__ void grid_sync(const Params &P) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned *gen = P.bar_gen;
    const unsigned g = *gen;
    __threadfence();
    const unsigned arrived = atomicAdd(P.bar_count, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(P.bar_count, 0u);
      __threadfence();
      atomicAdd(P.bar_gen, 1u);
    } else {
      const long long t0 = clock64();
      while (*gen == g) {
        if (clock64() - t0 > P.watchdog) __trap();
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Deterministic grid-wide sum: CTA tree -> partials[slot][cta] -> barrier ->
// every CTA sums all CTA partials in index order.  Result in all threads.
__device__ __forceinline__ double grid_sum(const Params &P, double v, int slot, double *sh) {
  const unsigned full = 0xffffffffu;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(full, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += sh[q];
    P.partials[(size_t)slot * gridDim.x + blockIdx.x] = s;
  }
  grid_sync(P);
  // every CTA: fixed-order sum of the CTA partials (warp 0, strided + tree)
  double acc = 0.0;
  if (warp == 0) {
    for (unsigned q = lane; q < gridDim.x; q += 32)
      acc += __ldcg(P.partials + (size_t)slot * gridDim.x + q);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(full, acc, o);
    if (lane == 0) sh[32] = acc;
  }
  __syncthreads();
  const double tot = sh[32];
  __syncthreads();
  return tot;
}

// ---------------------------------------------------------------- sweep
// Whole sweep: n_c color phases (ascending / descending), barrier between.
// Each lane walk is sweep_lean::lane_chain with cg loads for vectors.
template <bool FWD, int KC>
__device__ __forceinline__ void sweep(const Params &P, const double *src, double *dst,
                                      double *ys, int *offs, int *lens) {
  const long long *sp = FWD ? P.Lsp : P.Usp;
  const int *sl = FWD ? P.Lsl : P.Usl;
  const int *col = FWD ? P.Lcol : P.Ucol;
  const double *val = FWD ? P.Lval : P.Uval;
  const int gthreads = gridDim.x * blockDim.x;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  for (int ci = 0; ci < P.n_c; ++ci) {
    const int c = FWD ? ci : P.n_c - 1 - ci;
    const int k0 = P.color_lvl1[c], k1 = P.color_lvl1[c + 1];
    const int nl = (k1 - k0) * P.w;
    for (int g = gtid; g < nl; g += gthreads) {
      const int kq = g / P.w;
      if (P.w == 32)
        sweep_lean::lane_chain<FWD, KC, 32, true>(sp, sl, col, val, P.inv_d, src, dst, 32,
                                                  P.b_s, k0 + kq, g - kq * 32, ys, offs, lens);
      else
        sweep_lean::lane_chain<FWD, KC, 0, true>(sp, sl, col, val, P.inv_d, src, dst, P.w,
                                                 P.b_s, k0 + kq, g - kq * P.w, ys, offs, lens);
    }
    grid_sync(P);
  }
}

// ---------------------------------------------------------------- SpMV
// ap = A p (K/numba_backend.py:26-37); returns this thread's p.ap partial.
__device__ __forceinline__ double spmv_dot(const Params &P) {
  constexpr int CH = 8;
  const int gthreads = gridDim.x * blockDim.x;
  double part = 0.0;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < P.n; row += gthreads) {
    const int s = row / P.aw;
    const int j = row - s * P.aw;
    const int off = (int)P.Asp[s] + j;
    const int len = P.Asl[s];
    double acc = 0.0;
    for (int t0 = 0; t0 < len; t0 += CH) {
      int c[CH];
      double v[CH], xv[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const bool in = t0 + u < len;
        c[u] = in ? __ldg(P.Acol + off + (t0 + u) * P.aw) : 0;
        v[u] = in ? __ldg(P.Aval + off + (t0 + u) * P.aw) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < CH; ++u) xv[u] = t0 + u < len ? ldcg(P.p + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < CH; ++u)
        if (t0 + u < len) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
    }
    P.ap[row] = acc;
    part += ldcg(P.p + row) * acc;
  }
  return part;
}

}  // namespace persist
