// Device side of the HBMC ICCG hot path for B200 (sm_100a).
//
// Kernels (all fp64, memory-bound; no tensor cores -- see DESIGN.md):
//   * sell_sweep<FWD>   HBMC forward / backward substitution over the level-1
//                       blocks of one color (K/numba_backend.py:132-171).
//                       One thread per (level-1 block, lane): the lane walks
//                       its b_s rows sequentially; 32 consecutive lanes of a
//                       level-1 block read each SELL slot column as one
//                       coalesced 256 B (vals) + 128 B (cols) transaction.
//   * spmv_sell / spmv_csr  y = A x (K/numba_backend.py:16-37), optionally
//                       fused with the p.Ap dot and the alpha update.
//   * csr_task_sweep<FWD>   MC / BMC / level-scheduled natural substitution
//                       (K/numba_backend.py:114-129).
//   * CG vector kernels with fused deterministic reductions.
// Arithmetic: every substitution and SpMV uses __dmul_rn / __dsub_rn /
// __dadd_rn in the reference's per-row order, so results are bitwise equal
// to the reference (no FMA contraction).  Dots use a fixed-shape tree, so a
// solve is bitwise reproducible run to run.
//
// The whole PCG loop (src/solver.py:157-193) runs as ONE CUDA graph launch:
// a prologue plus a conditional WHILE node whose body is one CG iteration;
// the residual-check epilogue clears the loop condition on the device.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "tb_internal.h"

using tb::fail;

#include "sweep_lean.cuh"
#include "spmv_tma.cuh"
#include "persist.cuh"
#include "flow2.cuh"

#define CU(call)                                                          \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess)                                                \
      return fail(TB_ECUDA, "%s failed: %s (%s:%d)", #call,               \
                  cudaGetErrorString(e_), __FILE__, __LINE__);            \
  } while (0)

namespace {

constexpr int kBlock = 256;        // threads per CTA for streaming kernels
constexpr int kMaxPartials = 8192; // upper bound on CTAs of a reducing kernel
constexpr int kSplitN = 0;  // tb_pcg split path from this size on (A/B: faster at config 2 and 5)

// ------------------------------------------------------------ reductions
// Deterministic CTA sum: warp shuffle tree, then warp 0 over the warp sums.
// Result valid in thread 0.  `sh` must hold 32 doubles.
__device__ __forceinline__ double block_sum(double v, double *sh) {
  const unsigned full = 0xffffffffu;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(full, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();  // protect sh from a previous use
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    v = lane < nw ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(full, v, o);
  }
  return v;
}

// Device-resident PCG state (src/solver.py:157-193 scalars).
struct PcgState {
  double bnorm, rz, pap, alpha, beta, rel, tol;
  double bd_val;
  long long iter, max_iters, bd_iter;
  int done, converged, status, pad_;
  unsigned counter[4];
  cudaGraphConditionalHandle loop;  // 0 when not running under a graph
  int has_loop, pad2_;
};

// Last-CTA-done reduction.  Every CTA deposits its partial; the CTA that
// arrives last sums the partials in index order and calls fin(total) on
// thread 0.  Fixed grid => fixed summation tree => reproducible.
template <class Fin>
__device__ __forceinline__ void grid_reduce(double v, double *partials,
                                            unsigned *counter, Fin fin) {
  __shared__ double sh[32];
  __shared__ bool last;
  const double bs = block_sum(v, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    __threadfence();
    const unsigned prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double acc = 0.0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x)
    acc += __ldcg(partials + i);
  const double tot = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    *counter = 0;
    fin(tot);
  }
}

__device__ __forceinline__ void stop_loop(PcgState *st) {
  st->done = 1;
  if (st->has_loop) cudaGraphSetConditional(st->loop, 0);
}

// ------------------------------------------------------------ substitution
// K/numba_backend.py:132-171.  Thread g of the launch handles lane j = g % w
// of level-1 block k = k0 + g / w and walks its b_s rows (ascending for the
// forward sweep, descending for the backward sweep).  For every slot t of the
// row: y = y - v * y[col] with two roundings; a padding slot (col == own row,
// v == 0) reads the row's in-progress value exactly as the reference does.
// Operands of earlier colors / earlier steps are read with ld.global.cg so a
// value written by another SM in an earlier phase is never served from a
// stale L1 line.
template <bool FWD>
__global__ void __launch_bounds__(kBlock)
    sell_sweep(const long long *__restrict__ slice_ptr,
               const int *__restrict__ slice_len, const int *__restrict__ col,
               const double *__restrict__ val, const double *__restrict__ inv_d,
               const double *__restrict__ src, double *dst, int w, int b_s,
               long long k0, long long nthreads, const PcgState *st) {
  if (st && st->done) return;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nthreads) return;
  const long long k = k0 + g / w;
  const int j = (int)(g % w);
  for (int ll = 0; ll < b_s; ++ll) {
    const int l = FWD ? ll : b_s - 1 - ll;
    const long long sid = k * b_s + l;
    const long long row = sid * w + j;
    long long off = slice_ptr[sid] + j;
    const int len = slice_len[sid];
    double y = src[row];
    for (int t = 0; t < len; ++t, off += w) {
      const int c = col[off];
      const double v = val[off];
      const double xv = (c == row) ? y : __ldcg(dst + c);
      y = __dsub_rn(y, __dmul_rn(v, xv));
    }
    y = __dmul_rn(y, inv_d[row]);
    dst[row] = y;
  }
}

// K/numba_backend.py:114-129 generalised to independent tasks.
template <bool FWD>
__global__ void __launch_bounds__(kBlock)
    csr_task_sweep(const long long *__restrict__ rp, const int *__restrict__ col,
                   const double *__restrict__ val,
                   const double *__restrict__ inv_d,
                   const double *__restrict__ src, double *dst, long long task0,
                   long long ntasks, const long long *__restrict__ task_ptr,
                   const long long *__restrict__ rows, const PcgState *st) {
  if (st && st->done) return;
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ntasks) return;
  const long long t = task0 + g;
  const long long a = task_ptr ? task_ptr[t] : t;
  const long long b = task_ptr ? task_ptr[t + 1] : t + 1;
  for (long long qq = 0; qq < b - a; ++qq) {
    const long long q = FWD ? a + qq : b - 1 - qq;
    const long long i = rows ? rows[q] : q;
    double s = src[i];
    for (long long p = rp[i]; p < rp[i + 1]; ++p)
      s = __dsub_rn(s, __dmul_rn(val[p], __ldcg(dst + col[p])));
    dst[i] = __dmul_rn(s, inv_d[i]);
  }
}

// ------------------------------------------------------------ real-row loops
// Plans with dummy rows (HBMC padding) pass rix = the sorted real positions
// (HbmcLayout.real_positions): every CG vector kernel then walks rho in
// [0, n_real) with element i = rix[rho], in exactly the thread / unit
// assignment of its plain loop over a system of n_real rows (PAIRS: a unit is
// two consecutive rho, like TB_PAIRS4's element pair).  So every dot product
// -- and every x, r, p update -- is the one the same kernels compute for the
// system without dummies: the reduction tree depends only on the sequence of
// real entries (src/solver.py:150-153 reduces over real positions only),
// and HBMC with w = 1 reproduces BMC bitwise (T/test_solver.py:137-145).
// Dummy entries of x, r, p are never touched (they stay 0: b is 0 there).
template <bool PAIRS, class F>
__device__ __forceinline__ void rloop(long long n, const int *__restrict__ rix, F f) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long nu = PAIRS ? n / 2 : n;
  long long u0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  auto unit = [&](long long u) {
    if (PAIRS) {
      f((long long)__ldg(rix + 2 * u));
      f((long long)__ldg(rix + 2 * u + 1));
    } else {
      f((long long)__ldg(rix + u));
    }
  };
  for (; u0 + 3 * stride < nu; u0 += 4 * stride) {
#pragma unroll
    for (int q = 0; q < 4; ++q) unit(u0 + q * stride);
  }
  for (; u0 < nu; u0 += stride) unit(u0);
}

// p.Ap epilogue shared by the SpMV kernels: alpha = rz / p.Ap, or the CG
// breakdown (src/solver.py:174-177).
__device__ __forceinline__ void pap_fin(PcgState *st, double pap) {
  const long long j = st->iter + 1;
  st->pap = pap;
  if (pap <= 0.0) {
    st->status = TB_ECG_BREAKDOWN;
    st->bd_iter = j;
    st->bd_val = pap;
    stop_loop(st);
    return;
  }
  st->alpha = st->rz / pap;
}

// ------------------------------------------------------------ SpMV
// K/numba_backend.py:26-37: out = 0; out += v * x[col] per slot in stored
// order.  Optional fused epilogue: pap = p . (A p) and alpha = rz / pap.
template <bool DOT>
__global__ void __launch_bounds__(kBlock)
    spmv_sell(long long n, const long long *__restrict__ slice_ptr,
              const int *__restrict__ slice_len, const int *__restrict__ col,
              const double *__restrict__ val, int w,
              const double *__restrict__ x, double *__restrict__ out,
              double *partials, PcgState *st, const int *rix = nullptr) {
  if (DOT && st->done) return;
  double part = 0.0;
  constexpr int CH = 8;  // slots whose loads / gathers are in flight together
  auto row_fn = [&](long long row) {
    const long long s = row / w;
    const int j = (int)(row - s * w);
    const long long off = slice_ptr[s] + j;
    const int len = slice_len[s];
    const double xr = DOT ? __ldg(x + row) : 0.0;
    double acc = 0.0;
    for (int t0 = 0; t0 < len; t0 += CH) {
      const int *cp = col + off + (long long)t0 * w;
      const double *vp = val + off + (long long)t0 * w;
      int c[CH];
      double v[CH], xv[CH];
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const bool in = t0 + u < len;
        c[u] = in ? __ldg(cp + (long long)u * w) : 0;
        v[u] = in ? __ldg(vp + (long long)u * w) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < CH; ++u) xv[u] = t0 + u < len ? __ldg(x + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < CH; ++u)
        if (t0 + u < len) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
    }
    out[row] = acc;
    if (DOT) part += xr * acc;
  };
  if (rix) {
    rloop<false>(n, rix, row_fn);
  } else {
    for (long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x; row < n;
         row += (long long)gridDim.x * blockDim.x)
      row_fn(row);
  }
  if (DOT) grid_reduce(part, partials, &st->counter[0], [st](double pap) { pap_fin(st, pap); });
}

// K/numba_backend.py:16-23 spmv_csr (thread per row).
template <bool DOT>
__global__ void __launch_bounds__(kBlock)
    spmv_csr(long long n, const long long *__restrict__ rp,
             const int *__restrict__ col, const double *__restrict__ val,
             const double *__restrict__ x, double *__restrict__ out,
             double *partials, PcgState *st, const int *rix = nullptr) {
  if (DOT && st->done) return;
  double part = 0.0;
  auto row_fn = [&](long long i) {
    double acc = 0.0;
    for (long long p = rp[i]; p < rp[i + 1]; ++p)
      acc = __dadd_rn(acc, __dmul_rn(val[p], x[col[p]]));
    out[i] = acc;
    if (DOT) part += x[i] * acc;
  };
  if (rix) {
    rloop<false>(n, rix, row_fn);
  } else {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
      row_fn(i);
  }
  if (DOT) grid_reduce(part, partials, &st->counter[0], [st](double pap) { pap_fin(st, pap); });
}

// p . Ap over the real rows after a plain SpMV (plans with dummy rows whose
// SpMV is the TMA-staged kernel, which has no real-row loop).
__global__ void __launch_bounds__(kBlock)
    cg_dot_pap(long long n, const double *__restrict__ p, const double *__restrict__ ap,
               const int *__restrict__ rix, double *partials, PcgState *st) {
  if (st->done) return;
  double part = 0.0;
  rloop<false>(n, rix, [&](long long i) { part += __ldcg(p + i) * __ldcg(ap + i); });
  grid_reduce(part, partials, &st->counter[0], [st](double pap) { pap_fin(st, pap); });
}

// TMA-staged SpMV (spmv_tma.cuh) with the fused p . Ap and alpha epilogue
// of spmv_sell<true>: same grid_reduce, same state updates.
__global__ void __launch_bounds__(spmv_tma::kThreads, 2)
    spmv_tma_dot(const __grid_constant__ spmv_tma::Params p, double *partials, PcgState *st) {
  extern __shared__ __align__(128) unsigned char smem[];
  if (st->done) return;
  spmv_tma::init_bars(p, smem);
  unsigned phase = 0;
  const double part = spmv_tma::run<true>(p, smem, phase);
  grid_reduce(part, partials, &st->counter[0], [st](double pap) { pap_fin(st, pap); });
}

// ------------------------------------------------------------ CG vectors
// x = 0; r = b; bnorm = ||b|| (src/solver.py:159-167).
__global__ void __launch_bounds__(kBlock)
    cg_init(long long n, const double *__restrict__ b, double *__restrict__ x,
            double *__restrict__ r, double *partials, PcgState *st,
            double *hist, long long n_red = 0, const int *rix = nullptr) {
  double part = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    if (!rix) part += bi * bi;
  }
  if (rix) rloop<false>(n_red, rix, [&](long long i) { part += b[i] * b[i]; });
  grid_reduce(part, partials, &st->counter[1], [st, hist](double bb) {
    st->bnorm = sqrt(bb);
    st->iter = 0;
    st->status = TB_OK;
    if (st->bnorm == 0.0) {  // src/solver.py:165-167
      st->converged = 1;
      hist[0] = 0.0;
      stop_loop(st);
    } else {
      hist[0] = 1.0;
    }
  });
}

// Grid-stride loops below process 4 strided elements per trip with all their
// loads issued together (fixed order => deterministic partial sums).
#define TB_GRID_STRIDE4(...)                                                   \
  {                                                                            \
    const long long stride = (long long)gridDim.x * blockDim.x;               \
    long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;          \
    for (; i0 + 3 * stride < n; i0 += 4 * stride) {                           \
      _Pragma("unroll") for (int u = 0; u < 4; ++u) {                          \
        const long long i = i0 + u * stride;                                   \
        __VA_ARGS__                                                            \
      }                                                                        \
    }                                                                          \
    for (long long i = i0; i < n; i += stride) {                               \
      __VA_ARGS__                                                              \
    }                                                                          \
  }

// Same over element PAIRS (16-byte accesses), i = first index of the pair;
// requires n even.
#define TB_PAIRS4(...)                                                         \
  {                                                                            \
    const long long stride = 2LL * gridDim.x * blockDim.x;                    \
    long long i0 = 2LL * ((long long)blockIdx.x * blockDim.x + threadIdx.x);  \
    for (; i0 + 3 * stride < n; i0 += 4 * stride) {                           \
      _Pragma("unroll") for (int u = 0; u < 4; ++u) {                          \
        const long long i = i0 + u * stride;                                   \
        __VA_ARGS__                                                            \
      }                                                                        \
    }                                                                          \
    for (long long i = i0; i < n; i += stride) {                               \
      __VA_ARGS__                                                              \
    }                                                                          \
  }

// x += alpha p; r -= alpha ap; rel = ||r|| / ||b|| (src/solver.py:178-186).
// FOLDX: x += alpha p is deferred to the next p update (cg_rz_p_coop<true>)
// or, after the loop, to cg_x_final -- this pass then only streams r and ap.
template <bool PAIRS = false, bool FOLDX = false>
__global__ void __launch_bounds__(kBlock)
    cg_update_xr(long long n, const double *__restrict__ p,
                 const double *__restrict__ ap, double *__restrict__ x,
                 double *__restrict__ r, double *partials, PcgState *st,
                 double *hist, const int *rix = nullptr) {
  if (st->done) return;
  const double alpha = st->alpha;
  double part = 0.0;
  if (rix) {     // real rows only, same association (n = real rows)
    rloop<PAIRS>(n, rix, [&](long long i) {
      if (!FOLDX) x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
      const double ri = __dsub_rn(r[i], __dmul_rn(alpha, ap[i]));
      r[i] = ri;
      part += ri * ri;
    });
  } else if (PAIRS) {   // 16-byte accesses (n even)
    TB_PAIRS4({
      if (!FOLDX) {
        const double2 xo = *(const double2 *)(x + i), po = *(const double2 *)(p + i);
        double2 xn;
        xn.x = __dadd_rn(xo.x, __dmul_rn(alpha, po.x));
        xn.y = __dadd_rn(xo.y, __dmul_rn(alpha, po.y));
        *(double2 *)(x + i) = xn;
      }
      const double2 ro = *(const double2 *)(r + i), ao = *(const double2 *)(ap + i);
      double2 rn;
      rn.x = __dsub_rn(ro.x, __dmul_rn(alpha, ao.x));
      rn.y = __dsub_rn(ro.y, __dmul_rn(alpha, ao.y));
      *(double2 *)(r + i) = rn;
      part += rn.x * rn.x;
      part += rn.y * rn.y;
    })
  } else {
    TB_GRID_STRIDE4({
      x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
      const double ri = __dsub_rn(r[i], __dmul_rn(alpha, ap[i]));
      r[i] = ri;
      part += ri * ri;
    })
  }
  grid_reduce(part, partials, &st->counter[2], [st, hist](double rr) {
    const long long j = st->iter + 1;
    const double rel = sqrt(rr) / st->bnorm;
    st->rel = rel;
    st->iter = j;
    hist[j] = rel;
    if (rel < st->tol) {
      st->converged = 1;
      stop_loop(st);
    } else if (j >= st->max_iters) {
      stop_loop(st);
    }
  });
}

// Grid barrier + deterministic grid sum for the cooperative vector kernels
// (every CTA adds the CTA partials in index order after the barrier).
__device__ __forceinline__ void coop_sync(unsigned *bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned *gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      const long long t0 = clock64();
      while (*gen == g)
        if (clock64() - t0 > 4000000000LL) __trap();
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ double coop_sum(double v, double *partials, unsigned *bar,
                                           double *sh) {
  const double bsum = block_sum(v, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = bsum;
  coop_sync(bar);
  double acc = 0.0;
  if (threadIdx.x < 32) {
    for (unsigned q = threadIdx.x; q < gridDim.x; q += 32) acc += __ldcg(partials + q);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) sh[32] = acc;
  }
  __syncthreads();
  const double tot = sh[32];
  __syncthreads();
  return tot;
}

// r . z, beta and p = z + beta p in ONE cooperative launch (src/solver.py:
// 190-193), 16-byte accesses, n even: the deterministic grid sum (CTA
// partials added in index order by every CTA after a grid barrier) replaces
// cg_rz's last-CTA reduction, and the p update follows without a second
// launch.  Every CTA reads the old rz before the barrier; CTA 0 publishes
// the new rz / beta after it.
template <bool FOLDX = false>
__global__ void __launch_bounds__(kBlock)
    cg_rz_p_coop(long long n, const double *__restrict__ r, const double *__restrict__ z,
                 double *__restrict__ p, double *partials, unsigned *bar, PcgState *st,
                 double *__restrict__ x, unsigned *epoch_bump, const int *rix) {
  __shared__ double sh[33];
  if (st->done) return;
  const double rz_old = st->rz;
  const double alpha = st->alpha;   // this iteration's, for the deferred x update
  double part = 0.0;
  if (rix) {
    rloop<true>(n, rix, [&](long long i) { part += r[i] * z[i]; });
  } else {
    TB_PAIRS4({
      const double2 zi = *(const double2 *)(z + i), ri = *(const double2 *)(r + i);
      part += ri.x * zi.x;
      part += ri.y * zi.y;
    })
  }
  const double rzn = coop_sum(part, partials, bar, sh);
  const double beta = rzn / rz_old;
  if (rix) {
    rloop<true>(n, rix, [&](long long i) {
      const double po = p[i];
      if (FOLDX) x[i] = __dadd_rn(x[i], __dmul_rn(alpha, po));
      p[i] = __dadd_rn(z[i], __dmul_rn(beta, po));
    });
  } else TB_PAIRS4({
    const double2 zi = *(const double2 *)(z + i), po = *(const double2 *)(p + i);
    if (FOLDX) {   // x += alpha p with the p this iteration's x/r pass used
      const double2 xo = *(const double2 *)(x + i);
      double2 xn;
      xn.x = __dadd_rn(xo.x, __dmul_rn(alpha, po.x));
      xn.y = __dadd_rn(xo.y, __dmul_rn(alpha, po.y));
      *(double2 *)(x + i) = xn;
    }
    double2 pn;
    pn.x = __dadd_rn(zi.x, __dmul_rn(beta, po.x));
    pn.y = __dadd_rn(zi.y, __dmul_rn(beta, po.y));
    *(double2 *)(p + i) = pn;
  })
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->beta = beta;
    st->rz = rzn;
    if (epoch_bump) *epoch_bump += 1u;   // graph-replayed precond: next epoch
  }
}

// After the loop of a FOLDX solve: the last iteration's x += alpha p (its
// p update never ran: every exit happens at the residual check or before).
__global__ void __launch_bounds__(kBlock)
    cg_x_final(long long n, const double *__restrict__ p, double *__restrict__ x,
               const PcgState *st, const int *rix) {
  if (st->status != TB_OK || st->iter < 1) return;
  const double alpha = st->alpha;
  if (rix) {
    rloop<false>(n, rix, [&](long long i) { x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i])); });
    return;
  }
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
}

// rz_new = r . z; beta = rz_new / rz; rz = rz_new (src/solver.py:190-192).
// FIRST: the prologue's rz = r . z and p = z.
template <bool FIRST, bool PAIRS = false>
__global__ void __launch_bounds__(kBlock)
    cg_rz(long long n, const double *__restrict__ r,
          const double *__restrict__ z, double *__restrict__ p,
          double *partials, PcgState *st, const int *rix = nullptr) {
  if (st->done) return;
  double part = 0.0;
  if (rix) {
    rloop<PAIRS>(n, rix, [&](long long i) {
      const double zi = z[i];
      part += r[i] * zi;
      if (FIRST) p[i] = zi;
    });
  } else if (PAIRS) {
    TB_PAIRS4({
      const double2 zi = *(const double2 *)(z + i), ri = *(const double2 *)(r + i);
      part += ri.x * zi.x;
      part += ri.y * zi.y;
      if (FIRST) *(double2 *)(p + i) = zi;
    })
  } else {
    TB_GRID_STRIDE4({
      const double zi = z[i];
      part += r[i] * zi;
      if (FIRST) p[i] = zi;
    })
  }
  grid_reduce(part, partials, &st->counter[3], [st](double rz) {
    if (FIRST) {
      st->rz = rz;
    } else {
      st->beta = rz / st->rz;
      st->rz = rz;
    }
  });
}

// p = z + beta p (src/solver.py:193).
template <bool PAIRS = false>
__global__ void __launch_bounds__(kBlock)
    cg_update_p(long long n, const double *__restrict__ z,
                double *__restrict__ p, const PcgState *st, const int *rix = nullptr) {
  if (st->done) return;
  const double beta = st->beta;
  if (rix) {
    rloop<PAIRS>(n, rix, [&](long long i) { p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i])); });
  } else if (PAIRS) {
    TB_PAIRS4({
      const double2 zi = *(const double2 *)(z + i), po = *(const double2 *)(p + i);
      double2 pn;
      pn.x = __dadd_rn(zi.x, __dmul_rn(beta, po.x));
      pn.y = __dadd_rn(zi.y, __dmul_rn(beta, po.y));
      *(double2 *)(p + i) = pn;
    })
  } else {
    TB_GRID_STRIDE4({ p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i])); })
  }
}

// Next preconditioner epoch for graph-replayed dataflow launches.
__global__ void epoch_bump(unsigned *e) { *e += 1u; }

// ------------------------------------------------------------ persistent
// Whole preconditioner application (mode 0) or whole PCG solve (mode 1) in
// one cooperative launch; see persist.cuh.  Writes the final PcgState.
// __grid_constant__: device functions take `const Params &`; without it the
// parameter block would be copied to local memory and every field access
// would become a local load.
constexpr int kPersistMinB = 2;   // co-resident CTAs per SM the persistent kernel is built for
template <int KC, bool FLOW>
__global__ void __launch_bounds__(persist::kThreads, kPersistMinB)
    pcg_persistent(const __grid_constant__ persist::Params P) {
  extern __shared__ __align__(16) double psm[];
  const int T = blockDim.x, b_s = P.b_s;
  double *ys = psm;
  int *offs = (int *)(ys + (size_t)b_s * T);
  int *lens = offs + (size_t)b_s * T;
  double *sh = (double *)(lens + (size_t)b_s * T + (((size_t)b_s * T) & 1));
  PcgState *st = (PcgState *)P.state;
  const int gthreads = gridDim.x * blockDim.x;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = P.n;
  // z = M src; returns this thread's partial of dotv . z (dotv may be null).
  // Dataflow path: both sweeps with per-block flags and no grid barrier;
  // the caller's next grid_sum / grid_sync orders z before its readers.
  auto precond = [&](const double *src, double *dst, unsigned epoch, const double *dotv) {
    if constexpr (FLOW)
      return persist::sweep_pair_dataflow<KC>(P, src, P.y, dst, epoch, dotv, ys, offs, lens);
    persist::sweep<true, KC>(P, src, P.y, ys, offs, lens);
    persist::sweep<false, KC>(P, P.y, dst, ys, offs, lens);
    double d = 0.0;
    if (dotv)
      for (int i = gtid; i < n; i += gthreads) d += __ldcg(dotv + i) * __ldcg(dst + i);
    return d;
  };
  if (P.mode == 0) {
    precond(P.pre_src, P.pre_dst, P.epoch_dev ? *P.epoch_dev : P.epoch, nullptr);
    return;
  }
  const double tol = st->tol;
  const long long max_iters = st->max_iters;
  // x = 0; r = b; bnorm = ||b||  (src/solver.py:159-167)
  double part = 0.0;
  for (int i = gtid; i < n; i += gthreads) {
    const double bi = P.b[i];
    P.x[i] = 0.0;
    P.r[i] = bi;
    part += bi * bi;
  }
  const double bnorm = sqrt(persist::grid_sum(P, part, 0, sh));
  if (bnorm == 0.0) {
    if (gtid == 0) {
      P.hist[0] = 0.0;
      st->bnorm = 0.0;
      st->iter = 0;
      st->converged = 1;
      st->status = TB_OK;
      st->done = 1;
    }
    return;
  }
  if (gtid == 0) P.hist[0] = 1.0;
  double rz = persist::grid_sum(P, precond(P.r, P.z, P.epoch, P.r), 1, sh);
  for (int i = gtid; i < n; i += gthreads) P.p[i] = __ldcg(P.z + i);
  persist::grid_sync(P);
  long long j = 1, iters = 0;
  int converged = 0, status = TB_OK;
  double bd_val = 0.0, rel = 1.0;
  for (; j <= max_iters; ++j) {
    if (j == 3) persist::stamp(P, 0);
    const double pap = persist::grid_sum(
        P, persist::spmv_dot(P), 2, sh);
    if (j == 3) persist::stamp(P, 1);
    if (pap <= 0.0) {  // src/solver.py:176-177
      status = TB_ECG_BREAKDOWN;
      bd_val = pap;
      break;
    }
    const double alpha = rz / pap;
    part = 0.0;
    // 16-byte accesses, 4 pairs per trip (n is even: a multiple of b_s*w)
    TB_PAIRS4({
      const double2 xo = *(const double2 *)(P.x + i), po = __ldcg((const double2 *)(P.p + i));
      const double2 ro = *(const double2 *)(P.r + i), ao = __ldcg((const double2 *)(P.ap + i));
      double2 xn, rn;
      xn.x = __dadd_rn(xo.x, __dmul_rn(alpha, po.x));
      xn.y = __dadd_rn(xo.y, __dmul_rn(alpha, po.y));
      rn.x = __dsub_rn(ro.x, __dmul_rn(alpha, ao.x));
      rn.y = __dsub_rn(ro.y, __dmul_rn(alpha, ao.y));
      *(double2 *)(P.x + i) = xn;
      *(double2 *)(P.r + i) = rn;
      part += rn.x * rn.x;
      part += rn.y * rn.y;
    })
    rel = sqrt(persist::grid_sum(P, part, 3, sh)) / bnorm;
    if (j == 3) persist::stamp(P, 2);
    if (gtid == 0) P.hist[j] = rel;
    iters = j;
    if (rel < tol) {
      converged = 1;
      break;
    }
    if (j == max_iters) break;
    const double rzn =
        persist::grid_sum(P, precond(P.r, P.z, P.epoch + (unsigned)j, P.r), 1, sh);
    if (j == 3) persist::stamp(P, 3);
    const double beta = rzn / rz;
    rz = rzn;
    TB_PAIRS4({
      const double2 zo = __ldcg((const double2 *)(P.z + i));
      const double2 po = *(const double2 *)(P.p + i);
      double2 pn;
      pn.x = __dadd_rn(zo.x, __dmul_rn(beta, po.x));
      pn.y = __dadd_rn(zo.y, __dmul_rn(beta, po.y));
      *(double2 *)(P.p + i) = pn;
    })
    persist::grid_sync(P);
    if (j == 3) persist::stamp(P, 4);
  }
  if (gtid == 0) {
    st->bnorm = bnorm;
    st->iter = iters;
    st->rel = rel;
    st->converged = converged;
    st->status = status;
    st->bd_iter = status ? j : 0;
    st->bd_val = bd_val;
    st->rz = rz;
    st->done = 1;
  }
}

// ------------------------------------------------------------ helpers
inline unsigned grid_for(long long n, int per_block = kBlock) {
  long long g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return (unsigned)g;
}

inline unsigned reduce_grid(long long n, int per_thread = 4) {
  // Fixed for a given n (=> fixed summation tree), capped at kMaxPartials.
  long long g = (n + (long long)kBlock * per_thread - 1) / ((long long)kBlock * per_thread);
  if (g < 1) g = 1;
  if (g > kMaxPartials) g = kMaxPartials;
  return (unsigned)g;
}

template <class T>
int upload(T **dst, const T *src, long long count) {
  *dst = nullptr;
  if (count <= 0) return TB_OK;
  CU(cudaMalloc((void **)dst, sizeof(T) * (size_t)count));
  if (src) CU(cudaMemcpy(*dst, src, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice));
  return TB_OK;
}

struct DevSell {
  long long n_slices = 0, width = 0, slots = 0;
  long long *slice_ptr = nullptr;
  int *slice_len = nullptr, *col = nullptr;
  double *val = nullptr;
};

struct DevCsr {
  long long n = 0, nnz = 0;
  long long *rp = nullptr;
  int *col = nullptr;
  double *val = nullptr;
};

struct DevSched {
  long long n_phases = 0;
  std::vector<long long> phase_ptr;  // host copy
  long long *task_ptr = nullptr, *rows = nullptr;
};

int upload_sell(DevSell &d, const tb_sell_host &h) {
  d.n_slices = h.n_slices;
  d.width = h.width;
  d.slots = h.n_slices > 0 ? h.slice_ptr[h.n_slices] : 0;
  int rc;
  if ((rc = upload(&d.slice_ptr, (const long long *)h.slice_ptr, h.n_slices + 1))) return rc;
  if ((rc = upload(&d.slice_len, h.slice_len, h.n_slices))) return rc;
  if ((rc = upload(&d.col, h.col_idx, d.slots))) return rc;
  if ((rc = upload(&d.val, h.vals, d.slots))) return rc;
  return TB_OK;
}

// Upload an HBMC factor in STEP-MAJOR slice order: within each color, all
// level-1 blocks' step-0 slices, then all step-1 slices, ... (steps in walk
// order: ascending for the forward factor L, descending for U).  The warps
// of one color phase advance through their steps together, so this places
// the data they read at the same time next to each other in DRAM.  Slice
// contents are unchanged; slice_ptr[sid] points at the new place and the
// kernels take lengths from slice_len.
int upload_sell_step_major(DevSell &d, const tb_sell_host &h,
                           const std::vector<long long> &color_lvl1, long long b_s,
                           bool descending) {
  d.n_slices = h.n_slices;
  d.width = h.width;
  d.slots = h.n_slices > 0 ? h.slice_ptr[h.n_slices] : 0;
  const long long w = h.width;
  std::vector<long long> sp(h.n_slices + 1);
  std::vector<int> col(d.slots);
  std::vector<double> val(d.slots);
  long long pos = 0;
  const long long n_c = (long long)color_lvl1.size() - 1;
  for (long long c = 0; c < n_c; ++c)
    for (long long ii = 0; ii < b_s; ++ii) {
      const long long l = descending ? b_s - 1 - ii : ii;
      for (long long k = color_lvl1[c]; k < color_lvl1[c + 1]; ++k) {
        const long long sid = k * b_s + l;
        const long long o = h.slice_ptr[sid], n = (long long)h.slice_len[sid] * w;
        sp[sid] = pos;
        memcpy(col.data() + pos, h.col_idx + o, sizeof(int) * (size_t)n);
        memcpy(val.data() + pos, h.vals + o, sizeof(double) * (size_t)n);
        pos += n;
      }
    }
  sp[h.n_slices] = pos;
  if (pos != d.slots) return fail(TB_EINVAL, "step-major upload: slice lengths inconsistent");
  int rc;
  if ((rc = upload(&d.slice_ptr, sp.data(), h.n_slices + 1))) return rc;
  if ((rc = upload(&d.slice_len, h.slice_len, h.n_slices))) return rc;
  if ((rc = upload(&d.col, col.data(), d.slots))) return rc;
  if ((rc = upload(&d.val, val.data(), d.slots))) return rc;
  return TB_OK;
}

int upload_csr(DevCsr &d, const tb_csr_host &h) {
  d.n = h.n;
  d.nnz = h.n > 0 ? h.row_ptr[h.n] : 0;
  int rc;
  if ((rc = upload(&d.rp, (const long long *)h.row_ptr, h.n + 1))) return rc;
  if ((rc = upload(&d.col, h.col_idx, d.nnz))) return rc;
  if ((rc = upload(&d.val, h.vals, d.nnz))) return rc;
  return TB_OK;
}

int upload_sched(DevSched &d, const tb_sched_host &h) {
  d.n_phases = h.n_phases;
  d.phase_ptr.assign(h.phase_ptr, h.phase_ptr + h.n_phases + 1);
  const long long n_tasks = d.phase_ptr.back();
  int rc;
  if (h.task_ptr &&
      (rc = upload(&d.task_ptr, (const long long *)h.task_ptr, n_tasks + 1)))
    return rc;
  if (h.rows && (rc = upload(&d.rows, (const long long *)h.rows, h.n_rows))) return rc;
  return TB_OK;
}

void free_sell(DevSell &d) {
  cudaFree(d.slice_ptr);
  cudaFree(d.slice_len);
  cudaFree(d.col);
  cudaFree(d.val);
  d = DevSell();
}
void free_csr(DevCsr &d) {
  cudaFree(d.rp);
  cudaFree(d.col);
  cudaFree(d.val);
  d = DevCsr();
}
void free_sched(DevSched &d) {
  cudaFree(d.task_ptr);
  cudaFree(d.rows);
  d = DevSched();
}

}  // namespace

// ===================================================================== plan
struct tb_plan {
  int device = 0;
  int precond_kind = 0, spmv_format = 0;
  long long n = 0, n_real = 0;
  // HBMC
  long long w = 0, b_s = 0, n_c = 0;
  std::vector<long long> color_lvl1;  // host copy [n_c+1]
  DevSell L, U, A;
  // staged (TMA) sweep configuration per color, forward (L) and backward (U)
  struct ColorLaunch {
    long long k0 = 0, k1 = 0, n_tasks = 0;
    int max_slots = 0, warps = 0;  // staged: task capacity; ring: lmax
    int ring = 0;                  // ring depth (ring kernel)
    size_t smem = 0;
    unsigned grid = 0;
    int kind = 0;                  // 0 simple, 4 lean
    int block = 256;               // threads per CTA (lean)
  };
  std::vector<ColorLaunch> cl_fwd, cl_bwd;
  int num_sms = 148;
  // task sweeps
  DevCsr Lc, Uc, Ac;
  DevSched fs, bs;
  double *inv_d = nullptr;
  // internal vectors and PCG state
  double *r = nullptr, *y = nullptr, *z = nullptr, *p = nullptr, *ap = nullptr;
  double *vec_pool = nullptr;   // r, y, z, p, ap in one allocation (L2 window)
  bool l2_window = false;       // the ICCG graph carries the vector window
  int g_win = -1;               // TB_L2WIN the graph was built with
  size_t l2_persist = 0;        // set-aside while the graph runs
  double *partials = nullptr;
  PcgState *st = nullptr;
  double *hist = nullptr;
  long long hist_cap = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  // cached whole-solve graph
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t graph = nullptr;
  const double *g_b = nullptr;
  double *g_x = nullptr;
  long long g_hist_cap = 0;
  long long launches_prologue = 0, launches_per_iter = 0;
  // persistent cooperative path (HBMC + SELL A, 32-bit indexing)
  bool persist_ok = false, persist_pcg_ok = false;
  int persist_kc = 0, persist_grid = 0;
  size_t persist_smem = 0;
  int *color_lvl1_dev = nullptr;
  unsigned *bar = nullptr;  // [count, generation]
  double *ppartials = nullptr;
  // dataflow sweeps: per level-1 block dependency lists + completion flags
  long long n_lvl1_flow = 0;  // 0 = barrier-separated color phases
  int *fdep_ptr = nullptr, *fdep = nullptr, *bdep_ptr = nullptr, *bdep = nullptr;
  unsigned *flags = nullptr;  // [2 * n_lvl1]: forward, backward
  unsigned char *small = nullptr;  // per level-1 block: short-chain bits
  // item-pipelined dataflow kernel (flow2.cuh): unified dependency lists
  int *dep2 = nullptr, *Lce = nullptr, *Uce = nullptr, *item_k = nullptr;
  int2 *item_meta = nullptr;
  int dep_stride = 0, flow2_grid = 0;  // flow2_grid == 0: not configured
  size_t flow2_smem = 0;
  bool flow2_long = false;  // slices longer than 8 slots: chunked ring stages
  unsigned long long *trace = nullptr;  // TB_TRACE=1: in-kernel phase stamps
  unsigned epoch = 1;
  // TMA-staged SpMV (spmv_tma.cuh): 0 slices per chunk = not configured
  int spmv_S = 0, spmv_cap = 0, spmv_D = 0, spmv_grid = 0;

  // tb_pcg as a host-polled kernel sequence with the TMA SpMV and one
  // persistent dataflow precond launch per iteration (large systems)
  bool split_pcg = false;
  int vec_pt = 16;             // elements per thread of the CG vector kernels (grid size)
  int rzp_grid = 0;            // cg_rz_p_coop cooperative grid (0 = cg_rz + cg_update_p)
  // plans with dummy rows: the real positions (int32, sorted) the CG vector
  // kernels walk (see rloop); n_red = their count (= n without dummies)
  int *rix = nullptr;
  long long n_red = 0;
  bool in_graph = false;       // capturing the split graph: precond epochs from epoch_dev
  bool defer_bump = false;     // the iteration's cg_rz_p_coop bumps the epoch instead
  bool g_split = false;        // the instantiated graph is the split variant
  unsigned *epoch_dev = nullptr;
};

namespace {

// Execution-path switches, read at plan creation / solve time.  Defaults are
// the measured-fastest paths; the switches exist so the test suite can force
// every path (tests/test_gpu_full.py) and for diagnostics -- none changes
// results beyond the documented +-1 iteration / 1e-10 bar:
//   TB_FLOW2=0          no item-pipelined dataflow kernel (flow2.cuh): the
//                       persistent / per-phase kernels run the preconditioner
//   TB_PERSIST=0        no persistent kernels (per-phase sweeps, graph PCG)
//   TB_PERSIST_MIN_N=n  smallest n for the persistent barrier-mode kernel
//   TB_DATAFLOW=0       barrier-separated color phases instead of per-block flags
//   TB_FLOW_MAXDEP=n    longest average dependency list for the dataflow schedule
//   TB_SWEEP=simple     plain thread-per-lane sweep kernel (64-bit offsets)
//   TB_SPMV_TMA=0       thread-per-row SpMV instead of the TMA-staged one
//   TB_PCG_SPLIT=0|1    force the split (graph: TMA SpMV + dataflow precond) PCG
//   TB_PCG_SPLIT_POLL=k split path host-polled every k iterations
//   TB_PCG_NOGRAPH=k    kernel-sequence PCG host-polled every k iterations
//   TB_RZP_FUSE=0       separate r.z and p-update kernels
//   TB_VEC_PAIRS=0      scalar (8-byte) CG vector kernels
//   TB_L2WIN=0          no L2 persisting window over the CG vectors
//   TB_DEBUG_SYNC=1     synchronise after every stage of a host-polled iteration
//   TB_TRACE=1          in-kernel phase timestamps (tb_plan_trace)
//   TB_WATCHDOG_MS=n    watchdog of the in-kernel waits (default 2000; 0 = no trap)
int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// Per color: pick the sweep kernel and size its launch.
//   32-bit indexable plan, thread column of b_s steps fits shared memory
//     -> lean thread-per-lane kernel (sweep_lean.cuh), KC = the color's
//        longest slice rounded up to 2 / 4 / 6 / 8 slots;
//   otherwise -> the plain thread-per-lane kernel (sell_sweep, 64-bit
//     offsets, no shared memory).  TB_SWEEP=simple forces it (tests).
int configure_sweeps(tb_plan *pl, const tb_sell_host &h,
                     std::vector<tb_plan::ColorLaunch> &out) {
  out.assign(pl->n_c, tb_plan::ColorLaunch());
  const char *mode = getenv("TB_SWEEP");
  const bool force_simple = mode && !strcmp(mode, "simple");
  const int w = (int)pl->w, b_s = (int)pl->b_s;
  size_t smem_optin = 227 * 1024;
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, pl->device) == cudaSuccess)
    smem_optin = (size_t)v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, pl->device) == cudaSuccess)
    pl->num_sms = v;
  const bool idx32 = pl->n <= 0x7fffffffLL && h.slice_ptr[h.n_slices] <= 0x7fffffffLL;
  for (long long c = 0; c < pl->n_c; ++c) {
    tb_plan::ColorLaunch &L = out[c];
    L.k0 = pl->color_lvl1[c];
    L.k1 = pl->color_lvl1[c + 1];
    L.n_tasks = L.k1 - L.k0;
    if (force_simple || L.n_tasks <= 0) continue;
    if (idx32 && sweep_lean::smem_bytes(b_s, kBlock) <= smem_optin) {
      long long lmax = 0;
      for (long long sid = L.k0 * b_s; sid < L.k1 * b_s; ++sid)
        if (h.slice_len[sid] > lmax) lmax = h.slice_len[sid];
      L.kind = 4;
      // KC: slots loaded a step ahead; long rows (w = 32 only) get 12 / 16 /
      // 24 so the whole slice is in flight (else slots past KC are loaded
      // one after another inside the step)
      const long long lk = lmax < 24 ? lmax : 24;
      L.max_slots = lk <= 2 ? 2 : lk <= 4 ? 4 : lk <= 6 ? 6 : lk <= 8 || w != 32 ? 8
                  : lk <= 12 ? 12 : lk <= 16 ? 16 : 24;
      // KC >= 12 kernels hold ~170-250 registers: 128-thread CTAs pack
      // more warps per SM than 256-thread ones
      L.block = L.max_slots >= 12 ? 64 : kBlock;
      L.warps = L.block / 32;
      L.smem = sweep_lean::smem_bytes(b_s, L.block);
      L.grid = grid_for((L.k1 - L.k0) * w, L.block);
    }
  }
  static bool attr_done = false;
  if (!attr_done) {
#define TB_LEAN_ATTR(F, K)                                                         \
  CU(cudaFuncSetAttribute(sweep_lean::sweep_kernel<F, K, 32>,                      \
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_optin)); \
  CU(cudaFuncSetAttribute(sweep_lean::sweep_kernel<F, K, 0>,                       \
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_optin));
    TB_LEAN_ATTR(true, 2) TB_LEAN_ATTR(true, 4) TB_LEAN_ATTR(true, 6) TB_LEAN_ATTR(true, 8)
    TB_LEAN_ATTR(false, 2) TB_LEAN_ATTR(false, 4) TB_LEAN_ATTR(false, 6) TB_LEAN_ATTR(false, 8)
#undef TB_LEAN_ATTR
#define TB_LEAN_ATTR32(F, K)                                                       \
  CU(cudaFuncSetAttribute(sweep_lean::sweep_kernel<F, K, 32>,                      \
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_optin));
    TB_LEAN_ATTR32(true, 12) TB_LEAN_ATTR32(true, 16) TB_LEAN_ATTR32(true, 24)
    TB_LEAN_ATTR32(false, 12) TB_LEAN_ATTR32(false, 16) TB_LEAN_ATTR32(false, 24)
#undef TB_LEAN_ATTR32
    attr_done = true;
  }
  return TB_OK;
}

// Launch the configured kernel of one color phase.
template <bool FWD>
void launch_phase(tb_plan *pl, const tb_plan::ColorLaunch &L, const DevSell &M,
                  const double *src, double *dst, cudaStream_t s, const PcgState *st) {
  if (L.kind == 4) {
    const long long nt = (L.k1 - L.k0) * pl->w;
    const bool w32 = pl->w == 32;
    auto fn = L.max_slots == 2 ? (w32 ? sweep_lean::sweep_kernel<FWD, 2, 32> : sweep_lean::sweep_kernel<FWD, 2, 0>)
              : L.max_slots == 4 ? (w32 ? sweep_lean::sweep_kernel<FWD, 4, 32> : sweep_lean::sweep_kernel<FWD, 4, 0>)
              : L.max_slots == 6 ? (w32 ? sweep_lean::sweep_kernel<FWD, 6, 32> : sweep_lean::sweep_kernel<FWD, 6, 0>)
              : L.max_slots == 12 ? sweep_lean::sweep_kernel<FWD, 12, 32>
              : L.max_slots == 16 ? sweep_lean::sweep_kernel<FWD, 16, 32>
              : L.max_slots == 24 ? sweep_lean::sweep_kernel<FWD, 24, 32>
                                 : (w32 ? sweep_lean::sweep_kernel<FWD, 8, 32> : sweep_lean::sweep_kernel<FWD, 8, 0>);
    fn<<<L.grid, L.block, L.smem, s>>>(M.slice_ptr, M.slice_len, M.col, M.val, pl->inv_d, src,
                                      dst, (int)pl->w, (int)pl->b_s, (int)L.k0, (int)nt,
                                      st ? &st->done : nullptr);
  } else {
    const long long nt = (L.k1 - L.k0) * pl->w;
    sell_sweep<FWD><<<grid_for(nt), kBlock, 0, s>>>(M.slice_ptr, M.slice_len, M.col, M.val,
                                                   pl->inv_d, src, dst, (int)pl->w,
                                                   (int)pl->b_s, L.k0, nt, st);
  }
}

// Launch one substitution sweep (all phases) on `s`.  Returns kernel count.
int launch_forward(tb_plan *pl, const double *src, double *dst, cudaStream_t s,
                   const PcgState *st, long long *nl) {
  if (pl->precond_kind == TB_PRECOND_HBMC) {
    for (long long c = 0; c < pl->n_c; ++c) {
      const long long k0 = pl->color_lvl1[c], k1 = pl->color_lvl1[c + 1];
      const long long nt = (k1 - k0) * pl->w;
      if (nt <= 0) continue;
      launch_phase<true>(pl, pl->cl_fwd[c], pl->L, src, dst, s, st);
      ++*nl;
    }
  } else {
    for (long long ph = 0; ph < pl->fs.n_phases; ++ph) {
      const long long t0 = pl->fs.phase_ptr[ph], t1 = pl->fs.phase_ptr[ph + 1];
      if (t1 <= t0) continue;
      csr_task_sweep<true><<<grid_for(t1 - t0), kBlock, 0, s>>>(
          pl->Lc.rp, pl->Lc.col, pl->Lc.val, pl->inv_d, src, dst, t0, t1 - t0,
          pl->fs.task_ptr, pl->fs.rows, st);
      ++*nl;
    }
  }
  CU(cudaGetLastError());
  return TB_OK;
}

int launch_backward(tb_plan *pl, const double *src, double *dst, cudaStream_t s,
                    const PcgState *st, long long *nl) {
  if (pl->precond_kind == TB_PRECOND_HBMC) {
    for (long long c = pl->n_c - 1; c >= 0; --c) {
      const long long k0 = pl->color_lvl1[c], k1 = pl->color_lvl1[c + 1];
      const long long nt = (k1 - k0) * pl->w;
      if (nt <= 0) continue;
      launch_phase<false>(pl, pl->cl_bwd[c], pl->U, src, dst, s, st);
      ++*nl;
    }
  } else {
    for (long long ph = pl->bs.n_phases - 1; ph >= 0; --ph) {
      const long long t0 = pl->bs.phase_ptr[ph], t1 = pl->bs.phase_ptr[ph + 1];
      if (t1 <= t0) continue;
      csr_task_sweep<false><<<grid_for(t1 - t0), kBlock, 0, s>>>(
          pl->Uc.rp, pl->Uc.col, pl->Uc.val, pl->inv_d, src, dst, t0, t1 - t0,
          pl->bs.task_ptr, pl->bs.rows, st);
      ++*nl;
    }
  }
  CU(cudaGetLastError());
  return TB_OK;
}

void spmv_params(const tb_plan *pl, const double *x, double *out, spmv_tma::Params &P) {
  P.n = pl->n;
  P.n_slices = pl->A.n_slices;
  P.slice_ptr = pl->A.slice_ptr;
  P.slice_len = pl->A.slice_len;
  P.col = pl->A.col;
  P.val = pl->A.val;
  P.x = x;
  P.out = out;
  P.S = pl->spmv_S;
  P.cap = pl->spmv_cap;
  P.D = pl->spmv_D;
  P.n_chunks = (pl->A.n_slices + P.S - 1) / P.S;
}

int launch_spmv(tb_plan *pl, const double *x, double *out, cudaStream_t s,
                bool dot, long long *nl) {
  const long long n = pl->n;
  if (n <= 0) return TB_OK;
  if (pl->spmv_format == TB_SPMV_NONE)
    return fail(TB_EINVAL, "plan has no matrix A (preconditioner-only plan)");
  const long long nr = pl->n_red;
  if (pl->spmv_format == TB_SPMV_SELL && pl->spmv_S > 0) {
    spmv_tma::Params P;
    spmv_params(pl, x, out, P);
    if (dot && pl->rix) {   // real-row p.Ap after the plain TMA SpMV
      spmv_tma::spmv_kernel<<<pl->spmv_grid, spmv_tma::kThreads,
                              spmv_tma::smem_bytes(P.cap, P.D), s>>>(P);
      ++*nl;
      cg_dot_pap<<<reduce_grid(nr, 1), kBlock, 0, s>>>(nr, x, out, pl->rix, pl->partials,
                                                        pl->st);
    } else if (dot)
      spmv_tma_dot<<<pl->spmv_grid, spmv_tma::kThreads, spmv_tma::smem_bytes(P.cap, P.D), s>>>(
          P, pl->partials, pl->st);
    else
      spmv_tma::spmv_kernel<<<pl->spmv_grid, spmv_tma::kThreads,
                              spmv_tma::smem_bytes(P.cap, P.D), s>>>(P);
  } else if (pl->spmv_format == TB_SPMV_SELL) {
    if (dot)
      spmv_sell<true><<<reduce_grid(nr, 1), kBlock, 0, s>>>(nr, pl->A.slice_ptr, pl->A.slice_len,
                                                 pl->A.col, pl->A.val, (int)pl->A.width, x,
                                                 out, pl->partials, pl->st, pl->rix);
    else
      spmv_sell<false><<<grid_for(n), kBlock, 0, s>>>(n, pl->A.slice_ptr, pl->A.slice_len, pl->A.col,
                                          pl->A.val, (int)pl->A.width, x, out, nullptr,
                                          nullptr, nullptr);
  } else {
    if (dot)
      spmv_csr<true><<<reduce_grid(nr), kBlock, 0, s>>>(
          nr, pl->Ac.rp, pl->Ac.col, pl->Ac.val, x, out, pl->partials, pl->st, pl->rix);
    else
      spmv_csr<false><<<grid_for(n), kBlock, 0, s>>>(
          n, pl->Ac.rp, pl->Ac.col, pl->Ac.val, x, out, nullptr, nullptr);
  }
  ++*nl;
  CU(cudaGetLastError());
  return TB_OK;
}

// One CG iteration (src/solver.py:174-193) as a kernel sequence.
int launch_persistent(tb_plan *pl, int mode, const double *src, double *dst, const double *b,
                      double *x, cudaStream_t s, long long applications);

// x += alpha p folded into the p update (TB_FOLD_X=0 disables): only with
// the cooperative r.z + p kernel, which then owns that update.
bool fold_x(const tb_plan *pl) {
  return (pl->n_red % 2) == 0 && env_int("TB_VEC_PAIRS", 1) && pl->rzp_grid > 0 && pl->bar &&
         true;
}

// The deferred x update of the last iteration (FOLDX solves).
int launch_x_final(tb_plan *pl, double *x, cudaStream_t s, long long *nl) {
  if (!fold_x(pl)) return TB_OK;
  cg_x_final<<<reduce_grid(pl->n_red, pl->vec_pt), kBlock, 0, s>>>(pl->n_red, pl->p, x, pl->st,
                                                                   pl->rix);
  ++*nl;
  CU(cudaGetLastError());
  return TB_OK;
}

// z = M r inside a kernel-sequence iteration: the per-color phase kernels,
// or (split mode, host-polled loop only: the launch takes a fresh epoch from
// the host) one persistent dataflow launch.
int launch_precond_step(tb_plan *pl, cudaStream_t s, long long *nl) {
  int rc;
  if (pl->split_pcg) {
    if ((rc = launch_persistent(pl, 0, pl->r, pl->z, nullptr, nullptr, s, 1))) return rc;
    *nl += (pl->in_graph && !pl->defer_bump) ? 2 : 1;   // + the epoch bump
    return TB_OK;
  }
  if ((rc = launch_forward(pl, pl->r, pl->y, s, pl->st, nl))) return rc;
  return launch_backward(pl, pl->y, pl->z, s, pl->st, nl);
}

// TB_DEBUG_SYNC=1 (diagnostics, never inside a graph capture): synchronise
// after every stage of a kernel-sequence iteration and name the failing one.
int debug_sync(tb_plan *pl, cudaStream_t s, const char *stage) {
  if (pl->in_graph || !env_int("TB_DEBUG_SYNC", 0)) return TB_OK;
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess)
    return fail(TB_ECUDA, "%s failed: %s", stage, cudaGetErrorString(e));
  return TB_OK;
}

int launch_iteration(tb_plan *pl, double *x, cudaStream_t s, long long *nl) {
  const long long n = pl->n_red;   // the vector kernels' rows (real rows, via pl->rix)
  const unsigned rg = reduce_grid(n, pl->vec_pt);
  int rc;
  {
    if ((rc = launch_spmv(pl, pl->p, pl->ap, s, true, nl))) return rc;
    if ((rc = debug_sync(pl, s, "spmv+dot"))) return rc;
    const bool pairs = (n % 2) == 0 && env_int("TB_VEC_PAIRS", 1);
    const bool fold = fold_x(pl);
    (fold ? cg_update_xr<true, true> : pairs ? cg_update_xr<true> : cg_update_xr<false>)
        <<<rg, kBlock, 0, s>>>(n, pl->p, pl->ap, x, pl->r, pl->partials, pl->st, pl->hist,
                               pl->rix);
    ++*nl;
    if ((rc = debug_sync(pl, s, "cg_update_xr"))) return rc;
  }
  const bool coop_p = (n % 2) == 0 && env_int("TB_VEC_PAIRS", 1) && pl->rzp_grid > 0 && pl->bar;
  pl->defer_bump = pl->in_graph && pl->split_pcg && pl->n_lvl1_flow > 0 && coop_p;
  rc = launch_precond_step(pl, s, nl);
  if (rc) {
    pl->defer_bump = false;
    return rc;
  }
  if ((rc = debug_sync(pl, s, "precond"))) return rc;
  const bool pairs2 = (n % 2) == 0 && env_int("TB_VEC_PAIRS", 1);
  if (pairs2 && pl->rzp_grid > 0 && pl->bar) {
    long long nn = n;
    const double *rr = pl->r, *zz = pl->z;
    double *pp = pl->p, *pa = pl->partials, *xx = x;
    unsigned *bb = pl->bar;
    PcgState *ss = pl->st;
    unsigned *eb = pl->defer_bump ? pl->epoch_dev : nullptr;
    const int *rx = pl->rix;
    pl->defer_bump = false;
    void *args[] = {&nn, &rr, &zz, &pp, &pa, &bb, &ss, &xx, &eb, &rx};
    CU(cudaLaunchCooperativeKernel(fold_x(pl) ? (const void *)cg_rz_p_coop<true>
                                              : (const void *)cg_rz_p_coop<false>,
                                   dim3(pl->rzp_grid), dim3(kBlock), args, 0, s));
    --*nl;   // one launch instead of two
  } else {
    (pairs2 ? cg_rz<false, true> : cg_rz<false, false>)<<<rg, kBlock, 0, s>>>(
        n, pl->r, pl->z, pl->p, pl->partials, pl->st, pl->rix);
    if ((rc = debug_sync(pl, s, "cg_rz"))) return rc;
    (pairs2 ? cg_update_p<true> : cg_update_p<false>)<<<reduce_grid(n, pl->vec_pt), kBlock, 0, s>>>(
        n, pl->z, pl->p, pl->st, pl->rix);
  }
  *nl += 2;
  if ((rc = debug_sync(pl, s, "cg_update_p"))) return rc;
  CU(cudaGetLastError());
  return TB_OK;
}

int launch_prologue(tb_plan *pl, const double *b, double *x, cudaStream_t s,
                    long long *nl) {
  const long long n = pl->n, nr = pl->n_red;
  const unsigned rg = reduce_grid(nr);
  int rc;
  cg_init<<<rg, kBlock, 0, s>>>(n, b, x, pl->r, pl->partials, pl->st, pl->hist, nr, pl->rix);
  ++*nl;
  if ((rc = launch_precond_step(pl, s, nl))) return rc;
  cg_rz<true><<<rg, kBlock, 0, s>>>(nr, pl->r, pl->z, pl->p, pl->partials, pl->st, pl->rix);
  ++*nl;
  CU(cudaGetLastError());
  return TB_OK;
}

void drop_graph(tb_plan *pl) {
  if (pl->gexec) cudaGraphExecDestroy(pl->gexec);
  if (pl->graph) cudaGraphDestroy(pl->graph);
  pl->gexec = nullptr;
  pl->graph = nullptr;
}

// Build: [prologue] -> WHILE(cond) { iteration }.
// Access-policy window over the CG vector pool on pl->stream (on) or none
// (off).  The persisting set-aside is the device maximum; the hit ratio
// scales the window down to it.
// Scope guard for the persisting-L2 set-aside of a solve: raise() records
// the device's current limit and sets the new one; the destructor drops the
// persisting lines and restores the recorded limit (every exit path of
// tb_pcg, including CU() early returns).  Process-wide while it lives --
// see INTEGRATION.md.
struct L2SetAside {
  bool active = false;
  size_t prev = 0;
  void raise(size_t bytes) {
    if (cudaDeviceGetLimit(&prev, cudaLimitPersistingL2CacheSize) == cudaSuccess &&
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes) == cudaSuccess)
      active = true;
    else
      cudaGetLastError();
  }
  ~L2SetAside() {
    if (!active) return;
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prev);
    cudaGetLastError();
  }
};

void set_l2_window(tb_plan *pl, bool on) {
  cudaStreamAttrValue v;
  memset(&v, 0, sizeof(v));
  if (on) {
    int max_win = 0, max_persist = 0;
    cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, pl->device);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, pl->device);
    const long long nv = pl->n > 0 ? pl->n : 1;
    size_t bytes = sizeof(double) * (size_t)(5 * ((nv + 31) / 32 * 32));
    if (max_win <= 0 || max_persist <= 0) return;
    // only where the pool (nearly) fits the set-aside: config 2 (84 MB of
    // vectors, 1.01x the set-aside) 21.8 vs 22.5 ms; config 3 (283 MB, 3.4x)
    // 54.8 vs 51.5 ms -- the set-aside then only takes L2 from the factor
    // stream (profiles/README.md).  Ratios between those two were not
    // measured, so the gate stays at the measured gain (<= 1.25x).
    if (bytes * 4 > 5 * (size_t)max_persist || bytes > (size_t)max_win) return;
    pl->l2_persist = (size_t)max_persist;
    v.accessPolicyWindow.base_ptr = pl->vec_pool;
    v.accessPolicyWindow.num_bytes = bytes;
    v.accessPolicyWindow.hitRatio =
        bytes <= (size_t)max_persist ? 1.0f : (float)max_persist / (float)bytes;
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    pl->l2_window = true;
  }
  if (cudaStreamSetAttribute(pl->stream, cudaStreamAttributeAccessPolicyWindow, &v) !=
      cudaSuccess) {
    cudaGetLastError();
    if (on) pl->l2_window = false;
  }
}

int build_graph(tb_plan *pl, const double *b, double *x) {
  drop_graph(pl);
  cudaGraph_t g;
  CU(cudaGraphCreate(&g, 0));
  pl->graph = g;
  cudaGraphConditionalHandle handle;
  CU(cudaGraphConditionalHandleCreate(&handle, g, 1, cudaGraphCondAssignDefault));
  // publish the handle to the device state before the graph ever runs
  PcgState hs;
  CU(cudaMemcpy(&hs, pl->st, sizeof(PcgState), cudaMemcpyDeviceToHost));
  hs.loop = handle;
  hs.has_loop = 1;
  CU(cudaMemcpy(pl->st, &hs, sizeof(PcgState), cudaMemcpyHostToDevice));

  // prologue captured into the root graph
  long long nl = 0;
  pl->in_graph = pl->split_pcg;
  pl->g_split = pl->split_pcg;
  CU(cudaStreamBeginCaptureToGraph(pl->stream, g, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  int rc = launch_prologue(pl, b, x, pl->stream, &nl);
  cudaGraph_t captured;
  cudaError_t ce = cudaStreamEndCapture(pl->stream, &captured);
  if (rc || ce != cudaSuccess) pl->in_graph = false;
  if (rc) return rc;
  CU(ce);
  pl->launches_prologue = nl;

  // the conditional WHILE node depends on every current leaf of g
  size_t nn = 0;
  CU(cudaGraphGetNodes(g, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  CU(cudaGraphGetNodes(g, nodes.data(), &nn));
  std::vector<cudaGraphNode_t> leaves;
  for (auto nd : nodes) {
    size_t nd_out = 0;
    CU(cudaGraphNodeGetDependentNodes(nd, nullptr, &nd_out));
    if (nd_out == 0) leaves.push_back(nd);
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  CU(cudaGraphAddNode(&cnode, g, leaves.data(), leaves.size(), &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];

  nl = 0;
  CU(cudaStreamBeginCaptureToGraph(pl->stream, body, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  rc = launch_iteration(pl, x, pl->stream, &nl);
  ce = cudaStreamEndCapture(pl->stream, &captured);
  pl->in_graph = false;
  if (rc) return rc;
  CU(ce);
  pl->launches_per_iter = nl;
  if (fold_x(pl)) {   // epilogue after the loop: the last iteration's x update
    long long ne = 0;
    CU(cudaStreamBeginCaptureToGraph(pl->stream, g, &cnode, nullptr, 1,
                                     cudaStreamCaptureModeThreadLocal));
    rc = launch_x_final(pl, x, pl->stream, &ne);
    ce = cudaStreamEndCapture(pl->stream, &captured);
    if (rc) return rc;
    CU(ce);
    pl->launches_prologue += ne;
  }
  CU(cudaGraphInstantiate(&pl->gexec, g, 0));
  pl->g_b = b;
  pl->g_x = x;
  pl->g_hist_cap = pl->hist_cap;
  return TB_OK;
}

// ------------------------------------------------------------ persistent host side
using PersistFn = void (*)(persist::Params);

PersistFn persist_fn(int kc, bool flow) {
  switch (kc) {
    case 2: return flow ? pcg_persistent<2, true> : pcg_persistent<2, false>;
    case 4: return flow ? pcg_persistent<4, true> : pcg_persistent<4, false>;
    case 6: return flow ? pcg_persistent<6, true> : pcg_persistent<6, false>;
    default: return flow ? pcg_persistent<8, true> : pcg_persistent<8, false>;
  }
}

PersistFn flow2_fn(int kc, bool long_slices) {
  if (long_slices) return flow2::precond_kernel<8, true>;
  switch (kc) {
    case 2: return flow2::precond_kernel<2, false>;
    case 4: return flow2::precond_kernel<4, false>;
    case 6: return flow2::precond_kernel<6, false>;
    default: return flow2::precond_kernel<8, false>;
  }
}
size_t flow2_smem(int kc, int b_s) {
  switch (kc) {
    case 2: return flow2::smem_bytes<2>(b_s);
    case 4: return flow2::smem_bytes<4>(b_s);
    case 6: return flow2::smem_bytes<6>(b_s);
    default: return flow2::smem_bytes<8>(b_s);
  }
}

// Item-pipelined dataflow preconditioner (flow2.cuh): one dependency list per
// item of the sequence [forward k ascending | backward k descending] over
// the flag array [forward | backward], fixed stride, -1 padded.
int configure_flow2(tb_plan *pl, int kc, bool long_slices, const std::vector<int> &fp, const std::vector<int> &fd,
                    const std::vector<int> &bp, const std::vector<int> &bd) {
  pl->flow2_grid = 0;
  if (env_int("TB_FLOW2", 1) == 0) return TB_OK;
  const long long nl = pl->n_lvl1_flow, b_s = pl->b_s;
  if (pl->w != 32 || b_s < flow2::kStages || b_s > 32 || nl <= 0) return TB_OK;
  int ds = 1;
  for (long long k = 0; k < nl; ++k) {
    ds = std::max(ds, fp[k + 1] - fp[k]);
    ds = std::max(ds, bp[k + 1] - bp[k] + 1);
  }
  if (ds > 32) return TB_OK;
  // item order: forward k ascending; backward colors descending, k
  // ascending inside a color (blocks of one color are independent).  Any
  // order in which every dependency precedes its reader would do; a
  // wavefront order (later-color blocks a few thousand items behind the
  // blocks they read, for L2-resident gathers) measured 14 % slower at
  // config 5 and 11-33 % slower at config 3 (profiles/README.md r03f/g).
  std::vector<int> item_k((size_t)2 * nl);
  for (long long k = 0; k < nl; ++k) item_k[k] = (int)k;
  {
    long long it = nl;
    for (long long c = pl->n_c - 1; c >= 0; --c)
      for (long long k = pl->color_lvl1[c]; k < pl->color_lvl1[c + 1]; ++k) item_k[it++] = (int)k;
    if (it != 2 * nl) return TB_OK;
  }
  std::vector<int> dep((size_t)2 * nl * ds, -1);
  for (long long it = 0; it < 2 * nl; ++it) {
    const long long k = item_k[it];
    int *o = dep.data() + (size_t)it * ds;
    if (it < nl) {
      for (int q = fp[k]; q < fp[k + 1]; ++q) *o++ = fd[q];
    } else {
      *o++ = (int)k;  // the backward item's rhs is its own forward block
      for (int q = bp[k]; q < bp[k + 1]; ++q) *o++ = (int)nl + bd[q];
    }
  }
  int rc;
  if ((rc = upload(&pl->dep2, dep.data(), (long long)dep.size()))) return rc;
  // the descriptor kernel below reads plain block indices; afterwards bit 31
  // marks backward items whose block no later item reads (they publish no flag)
  if ((rc = upload(&pl->item_k, item_k.data(), (long long)item_k.size()))) return rc;
  CU(cudaMalloc((void **)&pl->item_meta, sizeof(int2) * (size_t)(2 * nl * b_s)));
  {
    const long long cnt = 2 * nl * b_s;
    flow2::build_item_meta<<<(unsigned)((cnt + 255) / 256), 256>>>(
        pl->L.slice_ptr, pl->L.slice_len, pl->U.slice_ptr, pl->U.slice_len, pl->item_k,
        pl->item_meta, (int)nl, (int)b_s);
    CU(cudaGetLastError());
  }
  {
    std::vector<char> read_by((size_t)nl, 0);
    for (int q : bd) read_by[q] = 1;      // (bd has a dummy 0 entry only when no list has entries)
    if (bp[nl] == 0) std::fill(read_by.begin(), read_by.end(), 0);
    for (long long it = nl; it < 2 * nl; ++it)
      if (!read_by[item_k[it]]) item_k[it] |= (int)0x80000000;
    CU(cudaStreamSynchronize(0));  // build_item_meta has read the plain indices
    CU(cudaMemcpy(pl->item_k, item_k.data(), sizeof(int) * item_k.size(), cudaMemcpyHostToDevice));
  }
  pl->dep_stride = ds;
  // encoded column arrays (in-block / padding slots pre-classified)
  {
    int *bad = nullptr;
    CU(cudaMalloc((void **)&bad, sizeof(int)));
    CU(cudaMemset(bad, 0, sizeof(int)));
    for (int f = 0; f < 2; ++f) {
      const DevSell &M = f ? pl->L : pl->U;
      int **dst = f ? &pl->Lce : &pl->Uce;
      CU(cudaMalloc((void **)dst, sizeof(int) * (size_t)(M.slots > 0 ? M.slots : 1)));
      const unsigned g = (unsigned)((M.n_slices + 7) / 8);
      if (g) flow2::encode_cols<<<g, 256>>>(M.slice_ptr, M.slice_len, M.col, *dst, M.n_slices,
                                            (int)b_s, f, 32, bad);
    }
    int hbad = 0;
    CU(cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(bad);
    if (hbad) {  // an in-block entry outside the lane's own level-2 block: not HBMC
      cudaFree(pl->Lce);
      cudaFree(pl->Uce);
      pl->Lce = pl->Uce = nullptr;
      return TB_OK;
    }
  }
  PersistFn fn = flow2_fn(kc, long_slices);
  const size_t smem = flow2_smem(kc, (int)b_s);
  int optin = 0;
  CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, pl->device));
  if (smem > (size_t)optin) return TB_OK;
  CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  int ps = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, fn, flow2::kThreads, smem));
  if (ps < 1) return TB_OK;
  {
    // Small systems: when a color has fewer level-1 blocks than two rounds of
    // the full grid, the items in flight overlap the blocks they depend on
    // and warps wait on flags; 4 CTAs (16 warps) per SM is faster there
    // (config 2: 81.9 vs 90.2 us with 5; profiles r03j).
    long long cmin = nl;
    for (long long c = 0; c < pl->n_c; ++c)
      cmin = std::min(cmin, pl->color_lvl1[c + 1] - pl->color_lvl1[c]);
    const long long warps_full = (long long)ps * pl->num_sms * (flow2::kThreads / 32);
    if (ps > 4 && cmin < 2 * warps_full) ps = 4;
  }
  // the descriptor / encoding kernels above ran on the default stream: done
  // before any launch on the plan's or a caller's (non-blocking) stream
  CU(cudaStreamSynchronize(0));
  pl->flow2_smem = smem;
  pl->flow2_long = long_slices;
  pl->persist_kc = kc;
  pl->flow2_grid = ps * pl->num_sms;
  return TB_OK;
}

// Decide whether the persistent kernel applies and size its cooperative grid.
int configure_persistent(tb_plan *pl, const tb_plan_desc *d) {
  pl->persist_ok = false;
  const char *e = getenv("TB_PERSIST");
  if (e && !strcmp(e, "0")) return TB_OK;
  if (pl->precond_kind != TB_PRECOND_HBMC || pl->n > 0x7fffffffLL) return TB_OK;
  if (d->L_sell.slice_ptr[d->L_sell.n_slices] > 0x7fffffffLL ||
      d->U_sell.slice_ptr[d->U_sell.n_slices] > 0x7fffffffLL)
    return TB_OK;
  if (d->spmv_format == TB_SPMV_SELL &&
      d->A_sell.slice_ptr[d->A_sell.n_slices] > 0x7fffffffLL)
    return TB_OK;
  long long lmax = 0;
  for (long long s = 0; s < d->L_sell.n_slices; ++s)
    lmax = d->L_sell.slice_len[s] > lmax ? d->L_sell.slice_len[s] : lmax;
  for (long long s = 0; s < d->U_sell.n_slices; ++s)
    lmax = d->U_sell.slice_len[s] > lmax ? d->U_sell.slice_len[s] : lmax;
  // Slices longer than the persistent kernel's 8 register slots (config 3's
  // 27-point rows, the kNN graph's): no persistent kernel -- the per-phase
  // lean kernels with the whole slice in flight are as fast or faster
  // (config 3: 832 vs 838 us; config 4: 781 vs 950 us; profiles/README.md
  // r02) -- but the item-pipelined dataflow kernel (flow2.cuh, chunked ring
  // stages) still applies when the dependency lists are short (config 3).
  const bool long_slices = lmax > 8;
  if (long_slices && (pl->w != 32 || env_int("TB_FLOW2", 1) == 0)) return TB_OK;
  const int kc = lmax <= 2 ? 2 : (lmax <= 4 ? 4 : (lmax <= 6 ? 6 : 8));
  int rc;
  if (!long_slices) {
  const size_t T = persist::kThreads;
  const size_t smem = (size_t)pl->b_s * T * 16 + 8 + 33 * 8 + 64;
  int v = 0;
  CU(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, pl->device));
  if (smem > (size_t)v) return TB_OK;
  int per_sm = 1 << 30;
  for (bool flow : {false, true}) {  // the grid must be co-resident for either variant
    PersistFn fn = persist_fn(kc, flow);
    // per-function attribute shared by all plans: the device maximum, not
    // this plan's size (a later plan with a smaller b_s must not shrink it)
    CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
    int ps = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, fn, (int)T, smem));
    per_sm = ps < per_sm ? ps : per_sm;
  }
  if (per_sm < 1) return TB_OK;
  if (per_sm > kPersistMinB) per_sm = kPersistMinB;
  pl->persist_kc = kc;
  pl->persist_smem = smem;
  pl->persist_grid = per_sm * pl->num_sms;
  std::vector<int> cl(pl->color_lvl1.begin(), pl->color_lvl1.end());
  if ((rc = upload(&pl->color_lvl1_dev, cl.data(), (long long)cl.size()))) return rc;
  CU(cudaMalloc((void **)&pl->bar, 2 * sizeof(unsigned)));
  CU(cudaMemset(pl->bar, 0, 2 * sizeof(unsigned)));
  CU(cudaMalloc((void **)&pl->ppartials, sizeof(double) * persist::kSlots * pl->persist_grid));
  pl->persist_ok = true;
  }
  // ---- dataflow sweeps (w == 32): level-1 block dependency lists.  Every
  // cross-block column of a forward row must lie in an EARLIER level-1
  // block and of a backward row in a LATER one (HBMC structure); otherwise
  // keep the barrier-separated phases.
  const char *df = getenv("TB_DATAFLOW");
  if (pl->w == 32 && !(df && !strcmp(df, "0"))) {
    const long long nl = pl->color_lvl1.back();
    const long long span = pl->b_s * 32;
    std::vector<int> fp, fd, bp, bd, tmp;
    std::vector<unsigned char> small(nl, 0);
    bool ok = true;
    auto build = [&](const tb_sell_host &M, std::vector<int> &ptr, std::vector<int> &dep,
                     bool fwd) {
      ptr.assign(nl + 1, 0);
      dep.clear();
      for (long long k = 0; k < nl && ok; ++k) {
        tmp.clear();
        int maxlen = 0;
        for (long long sid = k * pl->b_s; sid < (k + 1) * pl->b_s; ++sid)
          maxlen = M.slice_len[sid] > maxlen ? M.slice_len[sid] : maxlen;
        if (maxlen <= 2) small[k] |= fwd ? 1 : 2;
        for (long long sid = k * pl->b_s; sid < (k + 1) * pl->b_s; ++sid) {
          const long long off = M.slice_ptr[sid], cnt = (long long)M.slice_len[sid] * 32;
          for (long long q = off; q < off + cnt; ++q) {
            const long long kb = M.col_idx[q] / span;
            if (kb == k) continue;
            if (fwd ? kb > k : kb < k) ok = false;
            tmp.push_back((int)kb);
          }
        }
        std::sort(tmp.begin(), tmp.end());
        tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
        // long slices only run the flow kernel: <= 32 entries per item
        if (long_slices && tmp.size() > 31) ok = false;
        dep.insert(dep.end(), tmp.begin(), tmp.end());
        ptr[k + 1] = (int)dep.size();
      }
    };
    build(d->L_sell, fp, fd, true);
    build(d->U_sell, bp, bd, false);
    // Long dependency lists (the kNN graph with algebraic numbering: ~300
    // source blocks per level-1 block) make the per-item flag polls cost
    // more than the barriers they replace (ICCG 223 vs 166 ms at config 4);
    // structured configs have 2.5 (config 2) / 9.9 (config 3) on average.
    if (ok && nl > 0) {
      const double avg = (double)(fd.size() > bd.size() ? fd.size() : bd.size()) / (double)nl;
      if (avg > (double)env_int("TB_FLOW_MAXDEP", 64)) ok = false;
    }
    if (ok && nl > 0) {
      if (fd.empty()) fd.push_back(0);
      if (bd.empty()) bd.push_back(0);
      if ((rc = upload(&pl->fdep_ptr, fp.data(), (long long)fp.size()))) return rc;
      if ((rc = upload(&pl->fdep, fd.data(), (long long)fd.size()))) return rc;
      if ((rc = upload(&pl->bdep_ptr, bp.data(), (long long)bp.size()))) return rc;
      if ((rc = upload(&pl->bdep, bd.data(), (long long)bd.size()))) return rc;
      if ((rc = upload(&pl->small, small.data(), nl))) return rc;
      CU(cudaMalloc((void **)&pl->flags, sizeof(unsigned) * 2 * nl));
      CU(cudaMemset(pl->flags, 0, sizeof(unsigned) * 2 * nl));
      pl->n_lvl1_flow = nl;
      pl->epoch = 1;
      if ((rc = configure_flow2(pl, kc, long_slices, fp, fd, bp, bd))) return rc;
      // without the persistent kernels the flags only serve the flow kernel
      if (long_slices && pl->flow2_grid == 0) pl->n_lvl1_flow = 0;
    }
  }
  if (long_slices) return TB_OK;
  pl->persist_pcg_ok = d->spmv_format == TB_SPMV_SELL;
  // Without the dataflow schedule a small system runs faster as per-phase
  // kernels in a CUDA graph (config 1: ICCG 2.01 vs 2.44 ms, precond 36 vs
  // 61 us); large barrier-mode systems keep the single launch (config 4:
  // 165.5 vs 170.7 ms).
  if (pl->n_lvl1_flow == 0 && pl->n < (long long)env_int("TB_PERSIST_MIN_N", 1 << 20))
    pl->persist_ok = false;
  if (env_int("TB_TRACE", 0)) {
    CU(cudaMalloc((void **)&pl->trace, 64 * sizeof(unsigned long long)));
    CU(cudaMemset(pl->trace, 0, 64 * sizeof(unsigned long long)));
  }
  return TB_OK;
}

// mode 0: z = M r (src -> dst); mode 1: whole PCG (b, x; state preset).
// `applications` = preconditioner applications the launch may perform (epochs).
void pcg_persistent_fn_launch(tb_plan *pl, const persist::Params &P, cudaStream_t s) {
  switch (pl->persist_kc) {
    case 2: pcg_persistent<2, true><<<pl->persist_grid, persist::kThreads, pl->persist_smem, s>>>(P); break;
    case 4: pcg_persistent<4, true><<<pl->persist_grid, persist::kThreads, pl->persist_smem, s>>>(P); break;
    case 6: pcg_persistent<6, true><<<pl->persist_grid, persist::kThreads, pl->persist_smem, s>>>(P); break;
    default: pcg_persistent<8, true><<<pl->persist_grid, persist::kThreads, pl->persist_smem, s>>>(P); break;
  }
}

int launch_persistent(tb_plan *pl, int mode, const double *src, double *dst, const double *b,
                      double *x, cudaStream_t s, long long applications) {
  persist::Params P;
  memset(&P, 0, sizeof(P));
  if (pl->n_lvl1_flow > 0) {
    if ((unsigned long long)pl->epoch + (unsigned long long)applications + 2 > 0xF0000000ull) {
      CU(cudaMemsetAsync(pl->flags, 0, sizeof(unsigned) * 2 * pl->n_lvl1_flow, s));
      pl->epoch = 1;
    }
    P.n_lvl1 = (int)pl->n_lvl1_flow;
    P.fdep_ptr = pl->fdep_ptr;
    P.fdep = pl->fdep;
    P.bdep_ptr = pl->bdep_ptr;
    P.bdep = pl->bdep;
    P.fflag = pl->flags;
    P.bflag = pl->flags + pl->n_lvl1_flow;
    P.small = pl->small;
    P.dep2 = pl->dep2;
    P.dep_stride = pl->dep_stride;
    P.Lce = pl->Lce;
    P.Uce = pl->Uce;
    P.item_meta = pl->item_meta;
    P.item_k = pl->item_k;
  }
  P.trace = pl->trace;
  {
    P.epoch = pl->epoch;
    pl->epoch += (unsigned)(applications + 1);
  }
  P.mode = mode;
  P.n = (int)pl->n;
  P.w = (int)pl->w;
  P.b_s = (int)pl->b_s;
  P.n_c = (int)pl->n_c;
  P.color_lvl1 = pl->color_lvl1_dev;
  P.Lsp = pl->L.slice_ptr;
  P.Usp = pl->U.slice_ptr;
  P.Lsl = pl->L.slice_len;
  P.Usl = pl->U.slice_len;
  P.Lcol = pl->L.col;
  P.Ucol = pl->U.col;
  P.Lval = pl->L.val;
  P.Uval = pl->U.val;
  P.inv_d = pl->inv_d;
  P.Asp = pl->A.slice_ptr;
  P.Asl = pl->A.slice_len;
  P.Acol = pl->A.col;
  P.Aval = pl->A.val;
  P.aw = (int)(pl->A.width > 0 ? pl->A.width : 1);
  P.b = b;
  P.x = x;
  P.r = pl->r;
  P.y = pl->y;
  P.z = pl->z;
  P.p = pl->p;
  P.ap = pl->ap;
  P.pre_src = src;
  P.pre_dst = dst;
  P.hist = pl->hist;
  P.partials = pl->ppartials;
  P.bar_count = pl->bar;
  P.bar_gen = pl->bar + 1;
  P.state = pl->st;
  // per-wait watchdog of the in-kernel barriers / flag polls: traps (a sticky
  // context error) instead of hanging the GPU; TB_WATCHDOG_MS=0 disables it
  // (hosts that time-slice the GPU), default ~2 s
  P.watchdog = (long long)env_int("TB_WATCHDOG_MS", 2000) * 1900000LL;
  void *args[] = {&P};
  if (mode == 0 && P.n_lvl1 > 0 && pl->flow2_grid > 0) {
    // Item-pipelined dataflow kernel (flow2.cuh).  A cooperative launch, stand-alone and as a node of the split PCG graph
    // alike: the whole grid is guaranteed co-resident (warps wait on flags of
    // items other CTAs own).  In the graph the epoch comes from device memory
    // (bumped by the p-update kernel or a 1-thread kernel after the launch).
    if (pl->in_graph) P.epoch_dev = pl->epoch_dev;
    CU(cudaLaunchCooperativeKernel((const void *)flow2_fn(pl->persist_kc, pl->flow2_long),
                                   dim3(pl->flow2_grid), dim3(flow2::kThreads), args,
                                   pl->flow2_smem, s));
    if (pl->in_graph && !pl->defer_bump) epoch_bump<<<1, 1, 0, s>>>(pl->epoch_dev);
    CU(cudaGetLastError());
    return TB_OK;
  }
  if (mode == 0 && P.n_lvl1 > 0 && pl->in_graph) {
    // captured into the split PCG graph: the epoch comes from device memory
    // (bumped by a 1-thread kernel after each application) and the launch is
    // a plain one -- the dataflow schedule has no grid barrier, and the
    // graph runs its kernels one after another, so the grid is resident
    P.epoch_dev = pl->epoch_dev;
    pcg_persistent_fn_launch(pl, P, s);
    if (!pl->defer_bump) epoch_bump<<<1, 1, 0, s>>>(pl->epoch_dev);
    CU(cudaGetLastError());
    return TB_OK;
  }
  CU(cudaLaunchCooperativeKernel((const void *)persist_fn(pl->persist_kc, P.n_lvl1 > 0),
                                 dim3(pl->persist_grid), dim3(persist::kThreads), args,
                                 pl->persist_smem, s));
  return TB_OK;
}

// TMA-staged SpMV (spmv_tma.cuh) for a width-32 SELL A in the plain layout:
// the largest S <= 8 whose biggest chunk fits D = 4 stages in ~100 KB, grid
// = co-resident CTAs.  TB_SPMV_TMA=0 keeps the thread-per-row kernel.
int configure_spmv_tma(tb_plan *pl, const tb_sell_host &h) {
  pl->spmv_S = 0;
  if (env_int("TB_SPMV_TMA", 1) == 0 || h.width != 32 || h.n_slices <= 0)
    return TB_OK;
  const long long slots = h.slice_ptr[h.n_slices];
  if (slots > 0x7fffffffLL) return TB_OK;
  auto cap_of = [&](int S) {
    long long cap = 0;
    for (long long s0 = 0; s0 < h.n_slices; s0 += S) {
      const long long s1 = s0 + S < h.n_slices ? s0 + S : h.n_slices;
      const long long c = h.slice_ptr[s1] - h.slice_ptr[s0];
      cap = c > cap ? c : cap;
    }
    cap = (cap + 31) / 32 * 32;
    return cap < 32 ? 32LL : cap;
  };
  // candidates (slices per chunk, stages, smem budget KB) in order of
  // preference, from the A/B in profiles/README.md: 16 slices (two per warp,
  // 16 gathers in flight per lane) x 2 stages at 2 CTAs/SM for short rows;
  // one 8-slice stage at 2 CTAs/SM for long rows (27-point: 585 us vs 638
  // with one 16-slice stage at 1 CTA/SM)
  struct Cand { int S, D, kb; };
  Cand cands[4] = {{16, 2, 100}, {8, 1, 100}, {16, 1, 220}, {0, 0, 0}};
  int optin = 0;
  CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, pl->device));
  for (const Cand &c : cands) {
    if (c.S <= 0) break;
    const long long cap = cap_of(c.S);
    const size_t sm = spmv_tma::smem_bytes((int)cap, c.D);
    if (sm > (size_t)c.kb * 1024 || sm + 1024 > (size_t)optin) continue;
    // the attribute is per function, shared by every plan: set it to the
    // device maximum once instead of this plan's size
    CU(cudaFuncSetAttribute(spmv_tma::spmv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            optin));
    {  // dynamic + static (grid_reduce's) shared memory must fit the opt-in maximum
      cudaFuncAttributes fa;
      CU(cudaFuncGetAttributes(&fa, spmv_tma_dot));
      CU(cudaFuncSetAttribute(spmv_tma_dot, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - (int)fa.sharedSizeBytes));
    }
    int per_sm = 0, per_sm_dot = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmv_tma::spmv_kernel,
                                                     spmv_tma::kThreads, sm));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_dot, spmv_tma_dot,
                                                     spmv_tma::kThreads, sm));
    per_sm = per_sm_dot < per_sm ? per_sm_dot : per_sm;
    if (per_sm < 1) continue;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pl->device);
    pl->spmv_S = c.S;
    pl->spmv_cap = (int)cap;
    pl->spmv_D = c.D;
    pl->spmv_grid = per_sm * nsm;
    return TB_OK;
  }
  return TB_OK;
}

int sync_in(tb_plan *pl, void *stream) {
  CU(cudaEventRecord(pl->ev_in, (cudaStream_t)stream));
  CU(cudaStreamWaitEvent(pl->stream, pl->ev_in, 0));
  return TB_OK;
}
int sync_out(tb_plan *pl, void *stream) {
  CU(cudaEventRecord(pl->ev_out, pl->stream));
  CU(cudaStreamWaitEvent((cudaStream_t)stream, pl->ev_out, 0));
  return TB_OK;
}

}  // namespace

// ===================================================================== C ABI
extern "C" int tb_plan_create(const tb_plan_desc *d, int device, tb_plan **out) {
  *out = nullptr;
  if (!d || d->n < 0) return fail(TB_EINVAL, "plan_create: bad descriptor");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(TB_ENODEV, "plan_create: no CUDA device visible");
  if (device < 0 || device >= ndev) return fail(TB_EINVAL, "plan_create: bad device %d", device);
  if (d->n > 0x7fffffffLL) return fail(TB_EINVAL, "plan_create: n exceeds int32 columns");
  tb_plan *pl = new (std::nothrow) tb_plan();
  if (!pl) return fail(TB_ENOMEM, "plan_create: host allocation failed");
  pl->device = device;
  CU(cudaSetDevice(device));
  pl->precond_kind = d->precond_kind;
  pl->spmv_format = d->spmv_format;
  pl->n = d->n;
  pl->n_real = d->n_real;
  pl->vec_pt = 16;   // A/B: 16 > 8 > 4 > 32 elements per thread (profiles/README.md)
  int rc = TB_OK;
  auto bail = [&](int code) {
    tb_plan_destroy(pl);
    return code;
  };
  if (d->precond_kind == TB_PRECOND_HBMC) {
    if (d->w < 1 || d->b_s < 1 || d->n_c < 0 || d->n % (d->w * d->b_s))
      return bail(fail(TB_EINVAL, "plan_create: bad HBMC shape"));
    pl->w = d->w;
    pl->b_s = d->b_s;
    pl->n_c = d->n_c;
    pl->color_lvl1.assign(d->color_lvl1_ranges, d->color_lvl1_ranges + d->n_c + 1);
    if (d->L_sell.width != d->w || d->U_sell.width != d->w)
      return bail(fail(TB_EINVAL, "plan_create: factor slice width != w"));
    if ((rc = upload_sell_step_major(pl->L, d->L_sell, pl->color_lvl1, d->b_s, false)))
      return bail(rc);
    if ((rc = upload_sell_step_major(pl->U, d->U_sell, pl->color_lvl1, d->b_s, true)))
      return bail(rc);
    if ((rc = configure_sweeps(pl, d->L_sell, pl->cl_fwd))) return bail(rc);
    if ((rc = configure_sweeps(pl, d->U_sell, pl->cl_bwd))) return bail(rc);
    if (!(d->flags & TB_PLAN_PARTITIONED) && (rc = configure_persistent(pl, d)))
      return bail(rc);
  } else if (d->precond_kind == TB_PRECOND_TASKS) {
    if ((rc = upload_csr(pl->Lc, d->L_csr))) return bail(rc);
    if ((rc = upload_csr(pl->Uc, d->U_csr))) return bail(rc);
    if ((rc = upload_sched(pl->fs, d->fwd_sched))) return bail(rc);
    if ((rc = upload_sched(pl->bs, d->bwd_sched))) return bail(rc);
  } else {
    return bail(fail(TB_EINVAL, "plan_create: unknown preconditioner kind"));
  }
  if (d->spmv_format == TB_SPMV_NONE) {
    // preconditioner-only plan
  } else if (d->spmv_format == TB_SPMV_SELL) {
    if (d->A_sell.n_slices * d->A_sell.width < d->n)
      return bail(fail(TB_EINVAL, "plan_create: SELL A smaller than n"));
    if ((rc = upload_sell(pl->A, d->A_sell))) return bail(rc);
    if ((rc = configure_spmv_tma(pl, d->A_sell))) return bail(rc);
  } else {
    if ((rc = upload_csr(pl->Ac, d->A_csr))) return bail(rc);
  }
  if ((rc = upload(&pl->inv_d, d->inv_d, d->n))) return bail(rc);
  const long long nv = d->n > 0 ? d->n : 1;
  // the five work vectors are one allocation so a single L2 access-policy
  // window can cover them during the solve (tb_pcg); each starts 256-byte
  // aligned for the 16-byte / TMA paths
  const long long nv_al = (nv + 31) / 32 * 32;
  if ((rc = upload<double>(&pl->vec_pool, nullptr, 5 * nv_al))) return bail(rc);
  pl->r = pl->vec_pool;
  pl->y = pl->r + nv_al;
  pl->z = pl->y + nv_al;
  pl->p = pl->z + nv_al;
  pl->ap = pl->p + nv_al;
  if ((rc = upload<double>(&pl->partials, nullptr, kMaxPartials))) return bail(rc);
  // zero the pool (alignment gaps included: a slice-padded kernel may read
  // past n), then NaN-poison the work vectors' rows: every kernel must
  // write a row before it reads it
  if (cudaMemset(pl->vec_pool, 0, sizeof(double) * (size_t)(5 * nv_al)) != cudaSuccess)
    return bail(fail(TB_ECUDA, "plan_create: memset failed"));
  for (double *v : {pl->r, pl->y, pl->z, pl->p, pl->ap})
    if (cudaMemset(v, 0xff, sizeof(double) * (size_t)nv) != cudaSuccess)
      return bail(fail(TB_ECUDA, "plan_create: memset failed"));
  // real positions (plans with dummy rows): the reduction index of the CG
  // vector kernels; sorted, in range
  pl->n_red = d->n;
  if (d->real_pos && d->n_real > 0 && d->n_real < d->n) {
    std::vector<int> rp((size_t)d->n_real);
    for (long long i = 0; i < d->n_real; ++i) {
      const long long v = d->real_pos[i];
      if (v < 0 || v >= d->n || (i > 0 && v <= d->real_pos[i - 1]))
        return bail(fail(TB_EINVAL, "plan_create: real_pos must be sorted positions < n"));
      rp[(size_t)i] = (int)v;
    }
    if ((rc = upload(&pl->rix, rp.data(), d->n_real))) return bail(rc);
    pl->n_red = d->n_real;
    // the single-launch persistent PCG reduces over all rows: plans with
    // dummies solve through the kernel-sequence paths
    pl->persist_pcg_ok = false;
  }
  if (!pl->bar) {   // grid barrier of the cooperative vector kernels
    if (cudaMalloc((void **)&pl->bar, 2 * sizeof(unsigned)) != cudaSuccess ||
        cudaMemset(pl->bar, 0, 2 * sizeof(unsigned)) != cudaSuccess)
      return bail(fail(TB_ECUDA, "plan_create: barrier allocation failed"));
  }
  if (env_int("TB_RZP_FUSE", 1)) {   // fused r.z + p update for the kernel-sequence paths
    int ps = 0, nsm = 148;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, cg_rz_p_coop<true>, kBlock, 0));
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, pl->device);
    const long long want = ((pl->n_red + 1) / 2 + kBlock * 8 - 1) / (kBlock * 8);  // ~16 elements/thread
    long long g = (long long)ps * nsm;
    if (want < g) g = want;
    pl->rzp_grid = g > 0 ? (int)g : 0;
  }
  if (cudaMalloc((void **)&pl->st, sizeof(PcgState)) != cudaSuccess ||
      cudaMemset(pl->st, 0, sizeof(PcgState)) != cudaSuccess)
    return bail(fail(TB_ECUDA, "plan_create: state allocation failed"));
  if (cudaStreamCreateWithFlags(&pl->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&pl->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&pl->ev_out, cudaEventDisableTiming) != cudaSuccess)
    return bail(fail(TB_ECUDA, "plan_create: stream/event creation failed"));
  *out = pl;
  return TB_OK;
}

extern "C" int tb_plan_destroy(tb_plan *pl) {
  if (!pl) return TB_OK;
  cudaSetDevice(pl->device);
  drop_graph(pl);
  free_sell(pl->L);
  free_sell(pl->U);
  free_sell(pl->A);
  free_csr(pl->Lc);
  free_csr(pl->Uc);
  free_csr(pl->Ac);
  free_sched(pl->fs);
  free_sched(pl->bs);
  cudaFree(pl->inv_d);
  cudaFree(pl->vec_pool);
  cudaFree(pl->partials);
  cudaFree(pl->rix);
  cudaFree(pl->st);
  cudaFree(pl->hist);
  cudaFree(pl->color_lvl1_dev);
  cudaFree(pl->bar);
  cudaFree(pl->ppartials);
  cudaFree(pl->epoch_dev);
  cudaFree(pl->fdep_ptr);
  cudaFree(pl->fdep);
  cudaFree(pl->bdep_ptr);
  cudaFree(pl->bdep);
  cudaFree(pl->flags);
  cudaFree(pl->small);
  cudaFree(pl->dep2);
  cudaFree(pl->Lce);
  cudaFree(pl->Uce);
  cudaFree(pl->item_k);
  cudaFree(pl->item_meta);
  if (pl->ev_in) cudaEventDestroy(pl->ev_in);
  if (pl->ev_out) cudaEventDestroy(pl->ev_out);
  if (pl->stream) cudaStreamDestroy(pl->stream);
  delete pl;
  return TB_OK;
}

extern "C" int tb_plan_device_bytes(const tb_plan *pl, int64_t *bytes) {
  if (!pl) return fail(TB_EINVAL, "null plan");
  auto sb = [](const DevSell &s) {
    return (s.n_slices + 1) * 8 + s.n_slices * 4 + s.slots * 12;
  };
  auto cb = [](const DevCsr &c) { return (c.n + 1) * 8 + c.nnz * 12; };
  long long b = sb(pl->L) + sb(pl->U) + sb(pl->A) + cb(pl->Lc) + cb(pl->Uc) +
                cb(pl->Ac) + pl->n * 8 * 6 + kMaxPartials * 8;
  if (pl->flow2_grid > 0)  // flow kernel: encoded columns, item descriptors, dependency lists
    b += (pl->L.slots + pl->U.slots) * 4 + 2 * pl->n_lvl1_flow * (pl->b_s * 8 + 4 + pl->dep_stride * 4);
  if (pl->n_lvl1_flow > 0) b += 2 * pl->n_lvl1_flow * 4;  // completion flags
  *bytes = b;
  return TB_OK;
}

extern "C" int tb_plan_barriers_per_sweep(const tb_plan *pl, int64_t *count) {
  if (!pl) return fail(TB_EINVAL, "null plan");
  const long long phases = pl->precond_kind == TB_PRECOND_HBMC ? pl->n_c : pl->fs.n_phases;
  *count = phases > 0 ? phases - 1 : 0;
  return TB_OK;
}

extern "C" int tb_plan_forward(tb_plan *pl, const double *r, double *y, void *stream) {
  if (!pl) return fail(TB_EINVAL, "null plan");
  CU(cudaSetDevice(pl->device));
  long long nl = 0;
  return launch_forward(pl, r, y, (cudaStream_t)stream, nullptr, &nl);
}

extern "C" int tb_plan_backward(tb_plan *pl, const double *y, double *z, void *stream) {
  if (!pl) return fail(TB_EINVAL, "null plan");
  CU(cudaSetDevice(pl->device));
  long long nl = 0;
  return launch_backward(pl, y, z, (cudaStream_t)stream, nullptr, &nl);
}

extern "C" int tb_plan_precond(tb_plan *pl, const double *r, double *z, void *stream) {
  if (!pl) return fail(TB_EINVAL, "null plan");
  CU(cudaSetDevice(pl->device));
  // one launch for all color phases of both sweeps (the item-pipelined
  // dataflow kernel, else the persistent cooperative kernel)
  if (pl->persist_ok || pl->flow2_grid > 0)
    return launch_persistent(pl, 0, r, z, nullptr, nullptr, (cudaStream_t)stream, 1);
  long long nl = 0;
  int rc = launch_forward(pl, r, pl->y, (cudaStream_t)stream, nullptr, &nl);
  if (rc) return rc;
  return launch_backward(pl, pl->y, z, (cudaStream_t)stream, nullptr, &nl);
}

extern "C" int tb_plan_sweep_phase(tb_plan *pl, int forward, int64_t phase,
                                   const double *src, double *dst, void *stream) {
  if (!pl) return fail(TB_EINVAL, "null plan");
  if (pl->precond_kind != TB_PRECOND_HBMC || phase < 0 || phase >= pl->n_c)
    return fail(TB_EINVAL, "sweep_phase: HBMC plan and 0 <= phase < n_c required");
  CU(cudaSetDevice(pl->device));
  const cudaStream_t s = (cudaStream_t)stream;
  const long long k0 = pl->color_lvl1[phase], k1 = pl->color_lvl1[phase + 1];
  const long long nt = (k1 - k0) * pl->w;
  if (nt <= 0) return TB_OK;
  const tb_plan::ColorLaunch &L = forward ? pl->cl_fwd[phase] : pl->cl_bwd[phase];
  const DevSell &M = forward ? pl->L : pl->U;
  if (forward) launch_phase<true>(pl, L, M, src, dst, s, nullptr);
  else launch_phase<false>(pl, L, M, src, dst, s, nullptr);
  CU(cudaGetLastError());
  return TB_OK;
}

extern "C" int tb_plan_sweep_phase_push(tb_plan *pl, int forward, int64_t phase,
                                        const double *src, double *dst,
                                        const tb_push_desc *push, void *stream) {
  if (!pl || !push) return fail(TB_EINVAL, "sweep_phase_push: null argument");
  if (pl->precond_kind != TB_PRECOND_HBMC || phase < 0 || phase >= pl->n_c)
    return fail(TB_EINVAL, "sweep_phase_push: HBMC plan and 0 <= phase < n_c required");
  if (pl->w != 32 || push->npeers < 0 || push->npeers > TB_MAX_PEERS || !push->done_ctr)
    return fail(TB_EINVAL, "sweep_phase_push: w = 32 and 0 <= npeers <= %d required",
                TB_MAX_PEERS);
  const tb_plan::ColorLaunch &L = forward ? pl->cl_fwd[phase] : pl->cl_bwd[phase];
  if (L.kind != 4 && L.k1 > L.k0)
    return fail(TB_EINVAL, "sweep_phase_push: needs the lean phase kernel");
  CU(cudaSetDevice(pl->device));
  const cudaStream_t s = (cudaStream_t)stream;
  const DevSell &M = forward ? pl->L : pl->U;
  const long long nt = (L.k1 - L.k0) * 32;
  const unsigned grid = nt > 0 ? grid_for(nt) : 1;
  const size_t sm = sweep_lean::smem_bytes((int)pl->b_s, kBlock);
  static bool attr = false;
  if (!attr) {
    int optin = 0;
    CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, pl->device));
    for (auto fn : {sweep_lean::sweep_push_kernel<true, 2>, sweep_lean::sweep_push_kernel<true, 4>,
                    sweep_lean::sweep_push_kernel<true, 6>, sweep_lean::sweep_push_kernel<true, 8>,
                    sweep_lean::sweep_push_kernel<false, 2>, sweep_lean::sweep_push_kernel<false, 4>,
                    sweep_lean::sweep_push_kernel<false, 6>, sweep_lean::sweep_push_kernel<false, 8>}) {
      cudaFuncAttributes fa;
      CU(cudaFuncGetAttributes(&fa, fn));
      CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - (int)fa.sharedSizeBytes));
    }
    attr = true;
  }
  auto pick = [&](auto f2, auto f4, auto f6, auto f8) {
    return L.max_slots == 2 ? f2 : L.max_slots == 4 ? f4 : L.max_slots == 6 ? f6 : f8;
  };
  auto fn = forward ? pick(sweep_lean::sweep_push_kernel<true, 2>, sweep_lean::sweep_push_kernel<true, 4>,
                           sweep_lean::sweep_push_kernel<true, 6>, sweep_lean::sweep_push_kernel<true, 8>)
                    : pick(sweep_lean::sweep_push_kernel<false, 2>, sweep_lean::sweep_push_kernel<false, 4>,
                           sweep_lean::sweep_push_kernel<false, 6>, sweep_lean::sweep_push_kernel<false, 8>);
  fn<<<grid, kBlock, sm, s>>>(M.slice_ptr, M.slice_len, M.col, M.val, pl->inv_d, src, dst,
                              (int)pl->b_s, (int)L.k0, (int)nt, *push);
  CU(cudaGetLastError());
  return TB_OK;
}

extern "C" int tb_plan_trace(const tb_plan *pl, uint64_t *out64) {
  if (!pl) return fail(TB_EINVAL, "null plan");
  if (!pl->trace) return fail(TB_EINVAL, "plan created without TB_TRACE=1");
  CU(cudaMemcpy(out64, pl->trace, 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return TB_OK;
}

extern "C" int tb_plan_persistent(const tb_plan *pl, int32_t *precond, int32_t *pcg,
                                  int32_t *grid) {
  if (!pl) return fail(TB_EINVAL, "null plan");
  *precond = pl->persist_ok;
  *pcg = pl->persist_ok && pl->persist_pcg_ok;
  *grid = pl->persist_grid;
  return TB_OK;
}

extern "C" int tb_plan_flow_info(const tb_plan *pl, int32_t *grid, int32_t *stages,
                                 int64_t *smem_bytes) {
  if (!pl) return fail(TB_EINVAL, "null plan");
  *grid = pl->flow2_grid;
  *stages = pl->flow2_grid > 0 ? flow2::kStages : 0;
  *smem_bytes = pl->flow2_grid > 0 ? (int64_t)pl->flow2_smem : 0;
  return TB_OK;
}

extern "C" int tb_plan_phase_info(const tb_plan *pl, int forward, int64_t phase,
                                  int32_t *staged, int32_t *warps, int32_t *grid,
                                  int32_t *max_slots) {
  if (!pl || pl->precond_kind != TB_PRECOND_HBMC || phase < 0 || phase >= pl->n_c)
    return fail(TB_EINVAL, "phase_info: HBMC plan and 0 <= phase < n_c required");
  const tb_plan::ColorLaunch &L = forward ? pl->cl_fwd[phase] : pl->cl_bwd[phase];
  *staged = L.kind;
  *warps = L.warps;
  *grid = (int32_t)L.grid;
  *max_slots = L.max_slots;
  return TB_OK;
}

extern "C" int tb_plan_spmv(tb_plan *pl, const double *x, double *y, void *stream) {
  if (!pl) return fail(TB_EINVAL, "null plan");
  CU(cudaSetDevice(pl->device));
  long long nl = 0;
  return launch_spmv(pl, x, y, (cudaStream_t)stream, false, &nl);
}

extern "C" int tb_pcg(tb_plan *pl, const double *b, double *x, double tol,
                      int64_t max_iters, int64_t check_every, void *stream,
                      tb_pcg_report *rep, double *history_host) {
  // check_every == 0: the whole loop is one CUDA graph (device-side
  // convergence test).  check_every > 0 (or env TB_PCG_NOGRAPH=<n>): plain
  // launches, the host polls the device state every check_every iterations
  // (profilers cannot see inside conditional graph nodes).
  {
    const int env_batch = env_int("TB_PCG_NOGRAPH", 0);
    if (env_batch > 0) check_every = env_batch;
  }
  if (!pl || !rep || !history_host) return fail(TB_EINVAL, "pcg: null argument");
  if (!(tol > 0.0) || max_iters < 1) return fail(TB_EINVAL, "pcg: bad tol / max_iters");
  CU(cudaSetDevice(pl->device));
  memset(rep, 0, sizeof(*rep));
  if (pl->hist_cap < max_iters + 1) {
    cudaFree(pl->hist);
    pl->hist = nullptr;
    CU(cudaMalloc((void **)&pl->hist, sizeof(double) * (size_t)(max_iters + 1)));
    pl->hist_cap = max_iters + 1;
  }
  // Split path (large systems): kernel sequence with the TMA SpMV and one
  // persistent dataflow precond launch per iteration, host polling every
  // check_every iterations (each launch takes a fresh flag epoch).
  // TB_PCG_SPLIT=1/0 forces it on/off; default: n >= TB_PCG_SPLIT_N.
  {
    const int se = env_int("TB_PCG_SPLIT", -1);
    const long long sn = kSplitN;
    // default whenever the TMA SpMV and the dataflow precond apply
    // (configs 2, 3, 5: 23.3 / 51.9 / 1694 ms vs 28.5 / 54.4 / ~2000 ms for
    // the single persistent launch)
    pl->split_pcg = (pl->persist_ok || pl->flow2_grid > 0) && pl->spmv_S > 0 &&
                    (se == 1 || (se < 0 && pl->n >= sn && pl->n_lvl1_flow > 0));
    // the split path runs as a CUDA graph (conditional WHILE, device-side
    // convergence test) unless TB_PCG_SPLIT_POLL=n asks for host polling
    if (pl->split_pcg && check_every <= 0) check_every = env_int("TB_PCG_SPLIT_POLL", 0);
  }
  // reset the device state (keep the loop handle if a graph exists)
  PcgState hs;
  CU(cudaMemcpy(&hs, pl->st, sizeof(PcgState), cudaMemcpyDeviceToHost));
  const cudaGraphConditionalHandle h = hs.loop;
  const int has = hs.has_loop;
  memset(&hs, 0, sizeof(hs));
  hs.tol = tol;
  hs.max_iters = max_iters;
  hs.loop = h;
  hs.has_loop = check_every > 0 ? 0 : has;
  CU(cudaMemcpy(pl->st, &hs, sizeof(PcgState), cudaMemcpyHostToDevice));
  int rc;
  long long polled_launches = 0, polls = 0;
  const bool persistent =
      check_every <= 0 && pl->persist_ok && pl->persist_pcg_ok && !pl->split_pcg;
  if (persistent) {
    if ((rc = sync_in(pl, stream))) return rc;
    if ((rc = launch_persistent(pl, 1, nullptr, nullptr, b, x, pl->stream, max_iters + 1)))
      return rc;
    CU(cudaMemcpyAsync(&hs, pl->st, sizeof(PcgState), cudaMemcpyDeviceToHost, pl->stream));
    CU(cudaStreamSynchronize(pl->stream));
  } else if (check_every > 0) {
    if ((rc = sync_in(pl, stream))) return rc;
    if ((rc = launch_prologue(pl, b, x, pl->stream, &polled_launches))) return rc;
    for (;;) {
      for (int64_t q = 0; q < check_every; ++q)
        if ((rc = launch_iteration(pl, x, pl->stream, &polled_launches))) return rc;
      CU(cudaMemcpyAsync(&hs, pl->st, sizeof(PcgState), cudaMemcpyDeviceToHost, pl->stream));
      CU(cudaStreamSynchronize(pl->stream));
      ++polls;
      if (hs.done) break;
    }
    if ((rc = launch_x_final(pl, x, pl->stream, &polled_launches))) return rc;
    // restore the graph-loop fields for the next graph run
    PcgState tmp = hs;
    tmp.loop = h;
    tmp.has_loop = has;
    CU(cudaMemcpy(pl->st, &tmp, sizeof(PcgState), cudaMemcpyHostToDevice));
  } else {
    if (pl->split_pcg && !pl->epoch_dev) {
      CU(cudaMalloc((void **)&pl->epoch_dev, sizeof(unsigned)));
    }
    // L2 residency of the CG work vectors across the iteration's kernels
    // (the factor and A stream past them): an access-policy window over the
    // vector pool on the capturing stream is copied into the graph's kernel
    // nodes, and cleared again before any other launch.  TB_L2WIN=0: off.
    const int win = env_int("TB_L2WIN", 1) != 0;
    if (!pl->gexec || pl->g_b != b || pl->g_x != x || pl->g_hist_cap != pl->hist_cap ||
        pl->g_split != pl->split_pcg || pl->g_win != win) {
      pl->l2_window = false;
      pl->g_win = win;
      if (win) set_l2_window(pl, true);
      rc = build_graph(pl, b, x);
      if (win) set_l2_window(pl, false);
      if (rc) return rc;
    }
    if ((rc = sync_in(pl, stream))) return rc;
    if (pl->split_pcg) {
      // flags hold epochs < pl->epoch; restart them well before the
      // counter could wrap during this solve
      if ((unsigned long long)pl->epoch + (unsigned long long)max_iters + 4 > 0xF0000000ull) {
        CU(cudaMemsetAsync(pl->flags, 0, sizeof(unsigned) * 2 * pl->n_lvl1_flow, pl->stream));
        pl->epoch = 1;
      }
      CU(cudaMemcpyAsync(pl->epoch_dev, &pl->epoch, sizeof(unsigned), cudaMemcpyHostToDevice,
                         pl->stream));
    }
    // the persisting set-aside exists only while the solve runs: every other
    // launch (sweeps, SpMV, callers' kernels) keeps the whole L2.  The guard
    // restores the caller's previous limit on every exit path.
    L2SetAside l2guard;
    if (pl->l2_window) l2guard.raise(pl->l2_persist);
    CU(cudaGraphLaunch(pl->gexec, pl->stream));
    CU(cudaMemcpyAsync(&hs, pl->st, sizeof(PcgState), cudaMemcpyDeviceToHost, pl->stream));
    if (pl->split_pcg)
      CU(cudaMemcpyAsync(&pl->epoch, pl->epoch_dev, sizeof(unsigned), cudaMemcpyDeviceToHost,
                         pl->stream));
    CU(cudaStreamSynchronize(pl->stream));
    // the last application may not have bumped (the loop stopped before its
    // p update): never reuse its epoch
    if (pl->split_pcg) ++pl->epoch;
  }
  pl->split_pcg = false;
  if ((rc = sync_out(pl, stream))) return rc;
  const long long iters = hs.iter;
  CU(cudaMemcpy(history_host, pl->hist, sizeof(double) * (size_t)(iters + 1),
                cudaMemcpyDeviceToHost));
  rep->iterations = iters;
  rep->converged = hs.converged;
  rep->status = hs.status;
  rep->breakdown_iter = hs.bd_iter;
  rep->breakdown_value = hs.bd_val;
  rep->host_syncs = 1;
  // body runs iters times on success, iters+1 times on a breakdown / max-iter exit
  const long long bodies = hs.bnorm == 0.0 ? 0 : (hs.status ? iters + 1 : iters);
  rep->kernel_launches = pl->launches_prologue + bodies * pl->launches_per_iter;
  if (check_every > 0) {
    rep->kernel_launches = polled_launches;
    rep->host_syncs = polls;
  }
  if (persistent) rep->kernel_launches = 1;
  if (hs.status == TB_ECG_BREAKDOWN)
    return fail(TB_ECG_BREAKDOWN, "p.Ap = %.6g <= 0 at iteration %lld", hs.bd_val,
                (long long)hs.bd_iter);
  return TB_OK;
}

// ------------------------------------------------ raw device operators
extern "C" int tb_dev_spmv_sell(int64_t n_slices, const int64_t *slice_ptr,
                                const int32_t *slice_len, const int32_t *col_idx,
                                const double *vals, int64_t width,
                                const double *x, double *out, void *stream) {
  const long long n = n_slices * width;
  if (n <= 0) return TB_OK;
  spmv_sell<false><<<grid_for(n), kBlock, 0, (cudaStream_t)stream>>>(
      n, (const long long *)slice_ptr, slice_len, col_idx, vals, (int)width, x,
      out, nullptr, nullptr);
  CU(cudaGetLastError());
  return TB_OK;
}

extern "C" int tb_dev_spmv_csr(int64_t n, const int64_t *row_ptr,
                               const int32_t *col_idx, const double *vals,
                               const double *x, double *out, void *stream) {
  if (n <= 0) return TB_OK;
  spmv_csr<false><<<grid_for(n), kBlock, 0, (cudaStream_t)stream>>>(
      n, (const long long *)row_ptr, col_idx, vals, x, out, nullptr, nullptr);
  CU(cudaGetLastError());
  return TB_OK;
}

extern "C" int tb_dev_fwd_sell_range(const int64_t *slice_ptr,
                                     const int32_t *slice_len,
                                     const int32_t *col_idx, const double *vals,
                                     const double *inv_d, const double *r,
                                     double *y, int64_t width, int64_t block_rows,
                                     int64_t k0, int64_t k1, void *stream) {
  const long long nt = (k1 - k0) * width;
  if (nt <= 0) return TB_OK;
  sell_sweep<true><<<grid_for(nt), kBlock, 0, (cudaStream_t)stream>>>(
      (const long long *)slice_ptr, slice_len, col_idx, vals, inv_d, r, y,
      (int)width, (int)block_rows, k0, nt, nullptr);
  CU(cudaGetLastError());
  return TB_OK;
}

extern "C" int tb_dev_bwd_sell_range(const int64_t *slice_ptr,
                                     const int32_t *slice_len,
                                     const int32_t *col_idx, const double *vals,
                                     const double *inv_d, const double *y,
                                     double *z, int64_t width, int64_t block_rows,
                                     int64_t k0, int64_t k1, void *stream) {
  const long long nt = (k1 - k0) * width;
  if (nt <= 0) return TB_OK;
  sell_sweep<false><<<grid_for(nt), kBlock, 0, (cudaStream_t)stream>>>(
      (const long long *)slice_ptr, slice_len, col_idx, vals, inv_d, y, z,
      (int)width, (int)block_rows, k0, nt, nullptr);
  CU(cudaGetLastError());
  return TB_OK;
}

extern "C" int tb_dev_csr_sweep_tasks(int forward, const int64_t *row_ptr,
                                      const int32_t *col_idx, const double *vals,
                                      const double *inv_d, const double *src,
                                      double *dst, int64_t task0, int64_t task1,
                                      const int64_t *task_ptr, const int64_t *rows,
                                      void *stream) {
  const long long nt = task1 - task0;
  if (nt <= 0) return TB_OK;
  if (forward)
    csr_task_sweep<true><<<grid_for(nt), kBlock, 0, (cudaStream_t)stream>>>(
        (const long long *)row_ptr, col_idx, vals, inv_d, src, dst, task0, nt,
        (const long long *)task_ptr, (const long long *)rows, nullptr);
  else
    csr_task_sweep<false><<<grid_for(nt), kBlock, 0, (cudaStream_t)stream>>>(
        (const long long *)row_ptr, col_idx, vals, inv_d, src, dst, task0, nt,
        (const long long *)task_ptr, (const long long *)rows, nullptr);
  CU(cudaGetLastError());
  return TB_OK;
}
