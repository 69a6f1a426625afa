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
  // dataflow sweeps (w == 32): per level-1 block dependency lists and flags
  const int *fdep_ptr, *fdep, *bdep_ptr, *bdep;
  unsigned *fflag, *bflag;
  const unsigned char *small;  // per level-1 block: bit0 L slices <= 2 slots, bit1 U
  unsigned long long *trace;   // optional phase timestamps (TB_TRACE), or null
  int n_lvl1;             // 0 = use the barrier-separated color phases
  unsigned epoch;         // epoch of the first preconditioner application
  const unsigned *epoch_dev;  // mode 0 in a CUDA graph: epoch read from here (else null)
  // flow2.cuh: per item of [forward | backward] a -1 padded dependency list
  const int *dep2;
  int dep_stride;
  const int *Lce, *Uce;  // encoded column arrays (flow2::encode_cols)
  const int2 *item_meta;  // [2 n_lvl1][b_s] {slice offset, length} per item and walk step
  const int *item_k;      // [2 n_lvl1] level-1 block of each item
};

__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }

// Phase trace: CTA 0 / thread 0 stamps %globaltimer into P.trace[slot]
// (only when tracing is on; used by scripts to break an iteration down).
__device__ __forceinline__ void stamp(const Params &P, int slot) {
  if (P.trace && blockIdx.x == 0 && threadIdx.x == 0 && slot < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    P.trace[slot] = t;
  }
}

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
        if (P.watchdog > 0 && clock64() - t0 > P.watchdog) __trap();
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

// ---------------------------------------------------------------- dataflow
// Sync-free HBMC sweep pair (w == 32): the level-1 blocks of the forward
// sweep (colors ascending = k ascending) followed by those of the backward
// sweep (colors descending = k descending) form one global item sequence.
// Warp gw processes items gw, gw + W, ... in increasing order.  Before item
// k it waits (ld.acquire.gpu) until every level-1 block it reads from has
// published epoch e: forward -> the earlier-color blocks of its L rows;
// backward -> its own forward block (rhs = y) and the later-color blocks of
// its U rows.  After the item lane 0 publishes flag[k] = e (st.release.gpu).
// Every dependency has a lower global index than the waiting item and each
// warp walks its items in order, so the lowest unfinished item can always
// run: no deadlock, and no grid barrier inside the preconditioner.
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Lanes poll their share of the dependency flags with relaxed loads; once
// all are seen, one acquire fence per warp orders the warp's later loads
// after the producers' releases (instead of an acquire -- and an L1
// invalidation -- per lane and per poll).
__device__ __forceinline__ void wait_flags(const Params &P, const unsigned *flags,
                                           const int *dep, int d0, int d1, unsigned epoch,
                                           const unsigned *extra = nullptr) {
  const int lane = threadIdx.x & 31;
  if (extra && lane == 0 && ld_relaxed(extra) < epoch) {
    const long long t0 = clock64();
    while (ld_relaxed(extra) < epoch)
      if (P.watchdog > 0 && clock64() - t0 > P.watchdog) __trap();
  }
  for (int q = d0 + lane; q < d1; q += 32) {
    const unsigned *f = flags + dep[q];
    if (ld_relaxed(f) < epoch) {
      const long long t0 = clock64();
      while (ld_relaxed(f) < epoch)
        if (P.watchdog > 0 && clock64() - t0 > P.watchdog) __trap();
    }
  }
  __syncwarp();
  // every lane: relaxed observation + acquire fence = acquire pattern (the
  // fence is one warp instruction)
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Returns this thread's partial of dotv . dst over the rows it produced in
// the backward sweep (dotv == nullptr: 0) -- r . z fused into the sweep.
template <int KC>
__device__ __forceinline__ double sweep_pair_dataflow(const Params &P, const double *src,
                                                      double *mid, double *dst,
                                                      unsigned epoch, const double *dotv,
                                                      double *ys, int *offs, int *lens) {
  const int lane = threadIdx.x & 31;
  const int W = gridDim.x * (blockDim.x >> 5);
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int n = P.n_lvl1;
  double dot = 0.0;
  // blocks whose slices hold <= 2 slots (e.g. the first color of the forward
  // sweep: in-block entries only) run the short KC = 2 chain
  constexpr int KS = KC < 2 ? KC : 2;
  auto fwd_item = [&](int k) {
    wait_flags(P, P.fflag, P.fdep, P.fdep_ptr[k], P.fdep_ptr[k + 1], epoch);
    if (P.small[k] & 1)
      sweep_lean::lane_chain<true, KS, 32, true>(P.Lsp, P.Lsl, P.Lcol, P.Lval, P.inv_d, src,
                                                 mid, 32, P.b_s, k, lane, ys, offs, lens);
    else
      sweep_lean::lane_chain<true, KC, 32, true>(P.Lsp, P.Lsl, P.Lcol, P.Lval, P.inv_d, src,
                                                 mid, 32, P.b_s, k, lane, ys, offs, lens);
    __syncwarp();
    if (lane == 0) st_release(P.fflag + k, epoch);
  };
  auto bwd_item = [&](int k) {
    // deps: own rows' rhs (= forward result of block k) + later-color blocks
    wait_flags(P, P.bflag, P.bdep, P.bdep_ptr[k], P.bdep_ptr[k + 1], epoch, P.fflag + k);
    if (P.small[k] & 2)
      sweep_lean::lane_chain<false, KS, 32, true>(P.Usp, P.Usl, P.Ucol, P.Uval, P.inv_d, mid,
                                                  dst, 32, P.b_s, k, lane, ys, offs, lens, dotv,
                                                  &dot);
    else
      sweep_lean::lane_chain<false, KC, 32, true>(P.Usp, P.Usl, P.Ucol, P.Uval, P.inv_d, mid,
                                                  dst, 32, P.b_s, k, lane, ys, offs, lens, dotv,
                                                  &dot);
    __syncwarp();
    if (lane == 0) st_release(P.bflag + k, epoch);
  };
  // item sequence: forward k ascending, then backward k descending
  for (int it = gw; it < 2 * n; it += W) {
    if (it < n)
      fwd_item(it);
    else
      bwd_item(2 * n - 1 - it);
  }
  return dot;
}

// ---------------------------------------------------------------- SpMV
// ap = A p (K/numba_backend.py:26-37); returns this thread's p.ap partial.
// Two rows per trip (rows i and i + stride) so two rows' loads and gathers
// are in flight together; 8 slots per chunk.  Row order of the partial sum
// is fixed (i, then i + stride).
__device__ __forceinline__ double spmv_dot(const Params &P) {
  constexpr int CH = 8;
  const int gthreads = gridDim.x * blockDim.x;
  double part = 0.0;
  auto row_chunk = [&](int row, int t0, int len, int off, double &acc) {
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
  };
  int row = blockIdx.x * blockDim.x + threadIdx.x;
  for (; row + gthreads < P.n; row += 2 * gthreads) {
    const int r1 = row + gthreads;
    const int s0 = row / P.aw, s1 = r1 / P.aw;
    const int off0 = (int)P.Asp[s0] + row - s0 * P.aw;
    const int off1 = (int)P.Asp[s1] + r1 - s1 * P.aw;
    const int len0 = P.Asl[s0], len1 = P.Asl[s1];
    const double p0 = ldcg(P.p + row), p1 = ldcg(P.p + r1);
    double acc0 = 0.0, acc1 = 0.0;
    const int lm = len0 > len1 ? len0 : len1;
    for (int t0 = 0; t0 < lm; t0 += CH) {
      int c0[CH], c1[CH];
      double v0[CH], v1[CH], x0[CH], x1[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const bool i0 = t0 + u < len0, i1 = t0 + u < len1;
        c0[u] = i0 ? __ldg(P.Acol + off0 + (t0 + u) * P.aw) : 0;
        v0[u] = i0 ? __ldg(P.Aval + off0 + (t0 + u) * P.aw) : 0.0;
        c1[u] = i1 ? __ldg(P.Acol + off1 + (t0 + u) * P.aw) : 0;
        v1[u] = i1 ? __ldg(P.Aval + off1 + (t0 + u) * P.aw) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        x0[u] = t0 + u < len0 ? ldcg(P.p + c0[u]) : 0.0;
        x1[u] = t0 + u < len1 ? ldcg(P.p + c1[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        if (t0 + u < len0) acc0 = __dadd_rn(acc0, __dmul_rn(v0[u], x0[u]));
        if (t0 + u < len1) acc1 = __dadd_rn(acc1, __dmul_rn(v1[u], x1[u]));
      }
    }
    P.ap[row] = acc0;
    P.ap[r1] = acc1;
    part += p0 * acc0;
    part += p1 * acc1;
  }
  for (; row < P.n; row += gthreads) {
    const int s = row / P.aw;
    const int off = (int)P.Asp[s] + row - s * P.aw;
    const int len = P.Asl[s];
    double acc = 0.0;
    for (int t0 = 0; t0 < len; t0 += CH) row_chunk(row, t0, len, off, acc);
    P.ap[row] = acc;
    part += ldcg(P.p + row) * acc;
  }
  return part;
}

}  // namespace persist
