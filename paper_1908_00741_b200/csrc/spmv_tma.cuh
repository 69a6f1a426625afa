// SELL SpMV with TMA-staged matrix stream (sm_100a).
//
// K/numba_backend.py:26-37 spmv_sell, bitwise: out[row] = 0; then
// out[row] = out[row] + v * x[col] over the row's slots in stored order
// (__dmul_rn / __dadd_rn).
//
// The matrix stream (values + int32 columns, 12 B per slot, ~90 % of the
// SpMV's bytes) is moved by 1-D TMA bulk copies (cp.async.bulk, mbarrier
// complete_tx): a CHUNK = S consecutive slices, whose slots are one
// contiguous range of both arrays, lands in one of D shared-memory stages.
// CTAs are persistent (grid = co-resident CTAs) and walk the chunks
// round-robin, keeping D chunks in flight -- tens of KB per SM queued in the
// copy engine without spending a register on them, which is what a
// latency-bound thread-per-row SpMV lacks.  Warps then read columns / values
// from shared memory (lane = row of a slice: conflict-free), gather x (the
// vector is L2-resident for the configs up to ~126 MB) with KG gathers in
// flight per lane, and accumulate in slot order.
//
// Optional fused epilogue (DOT): this thread's partial of x . out (p . Ap).

#pragma once

#include "tma_util.cuh"

namespace spmv_tma {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kG = 8;   // gathers in flight per lane

struct Params {
  long long n;                 // rows (the last slice may hold rows >= n: skipped)
  long long n_slices;
  const long long *slice_ptr;  // element offsets, multiples of 32
  const int *slice_len;
  const int *col;
  const double *val;
  const double *x;
  double *out;
  int S;                 // slices per chunk
  int cap;               // slot capacity of a stage (>= the largest chunk, % 32 == 0)
  int D;                 // stages
  long long n_chunks;
};

__host__ __device__ inline size_t stage_bytes(int cap) { return (size_t)cap * 12; }
__host__ __device__ inline size_t smem_bytes(int cap, int D) {
  return (size_t)D * stage_bytes(cap) + (size_t)D * 8 + 16;
}

// Issue the bulk copies of chunk q into stage st (one thread).
__device__ __forceinline__ void issue(const Params &p, long long q, unsigned char *stage,
                                      int cap, unsigned long long *bar) {
  const long long s0 = q * p.S;
  const long long s1 = s0 + p.S < p.n_slices ? s0 + p.S : p.n_slices;
  const long long a = p.slice_ptr[s0], b = p.slice_ptr[s1];
  const unsigned cnt = (unsigned)(b - a);
  tma::mbar_arrive_expect_tx(bar, cnt * 12u);
  if (cnt) {
    // the matrix stream is read once: evict-first, so it does not flush the
    // gathered vector out of L2 (config 2 45.2 -> 42.5 us, config 3 582 ->
    // 551, config 4 406 -> 366, config 5 2257 -> 2223; profiles r03h)
    const unsigned long long pol = tma::policy_evict_first();
    tma::bulk_g2s_hint(stage, p.val + a, cnt * 8u, bar, pol);
    tma::bulk_g2s_hint(stage + (size_t)cap * 8, p.col + a, cnt * 4u, bar, pol);
  }
}

// One slice row (lane) of the stage: acc = 0; acc = acc + v * x[col].
// Two slices per call (the second may be absent: len1 = -1) so a lane keeps
// 2 * kG gathers in flight.
__device__ __forceinline__ void rows2(const double *sv, const int *sc, int off0, int len0,
                                      int off1, int len1, const double *x, double &acc0,
                                      double &acc1) {
  const int lm = len0 > len1 ? len0 : len1;
  for (int t0 = 0; t0 < lm; t0 += kG) {
    double v0[kG], x0[kG], v1[kG], x1[kG];
#pragma unroll
    for (int u = 0; u < kG; ++u) {
      const bool i0 = t0 + u < len0, i1 = t0 + u < len1;
      const int c0 = i0 ? sc[off0 + (t0 + u) * 32] : 0;
      const int c1 = i1 ? sc[off1 + (t0 + u) * 32] : 0;
      v0[u] = i0 ? sv[off0 + (t0 + u) * 32] : 0.0;
      v1[u] = i1 ? sv[off1 + (t0 + u) * 32] : 0.0;
      x0[u] = i0 ? __ldcg(x + c0) : 0.0;
      x1[u] = i1 ? __ldcg(x + c1) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kG; ++u) {
      if (t0 + u < len0) acc0 = __dadd_rn(acc0, __dmul_rn(v0[u], x0[u]));
      if (t0 + u < len1) acc1 = __dadd_rn(acc1, __dmul_rn(v1[u], x1[u]));
    }
  }
}

// Rows of chunk q from stage memory; returns the DOT partial.  Warp w takes
// slices w, w + kWarps, ... of the chunk, two at a time.
template <bool DOT>
__device__ __forceinline__ double compute(const Params &p, long long q,
                                          const unsigned char *stage, int cap) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double *sv = (const double *)stage;
  const int *sc = (const int *)(stage + (size_t)cap * 8);
  const long long s0 = q * p.S;
  const long long s1 = s0 + p.S < p.n_slices ? s0 + p.S : p.n_slices;
  const long long base = p.slice_ptr[s0];
  double part = 0.0;
  for (long long s = s0 + warp; s < s1; s += 2 * kWarps) {
    const long long t = s + kWarps;
    const bool two = t < s1;
    const int off0 = (int)(p.slice_ptr[s] - base) + lane, len0 = p.slice_len[s];
    const int off1 = two ? (int)(p.slice_ptr[t] - base) + lane : 0;
    const int len1 = two ? p.slice_len[t] : -1;
    double acc0 = 0.0, acc1 = 0.0;
    rows2(sv, sc, off0, len0, off1, len1, p.x, acc0, acc1);
    const long long r0 = s * 32 + lane;
    if (r0 < p.n) {
      p.out[r0] = acc0;
      if (DOT) part += __ldcg(p.x + r0) * acc0;
    }
    if (two) {
      const long long r1 = t * 32 + lane;
      if (r1 < p.n) {
        p.out[r1] = acc1;
        if (DOT) part += __ldcg(p.x + r1) * acc1;
      }
    }
  }
  return part;
}

// Whole SpMV by this CTA's chunks.  smem: D stages then D mbarriers.
// `phase` holds one parity bit per stage (the mbarrier's completed-phase
// count mod 2); persistent kernels call run() once per iteration with the
// same barriers, so the bits carry over between calls.
template <bool DOT>
__device__ __forceinline__ double run(const Params &p, unsigned char *smem, unsigned &phase) {
  unsigned long long *bars =
      (unsigned long long *)(smem + (size_t)p.D * stage_bytes(p.cap));
  const long long G = gridDim.x;
  long long nmine = p.n_chunks > blockIdx.x ? (p.n_chunks - 1 - blockIdx.x) / G + 1 : 0;
  if (threadIdx.x == 0) {
    tma::fence_proxy_async_smem();
    for (int i = 0; i < p.D && i < nmine; ++i)
      issue(p, blockIdx.x + i * G, smem + (size_t)i * stage_bytes(p.cap), p.cap, bars + i);
  }
  double part = 0.0;
  for (long long i = 0; i < nmine; ++i) {
    const int st = (int)(i % p.D);
    tma::mbar_wait(bars + st, (phase >> st) & 1u);
    phase ^= 1u << st;
    part += compute<DOT>(p, blockIdx.x + i * G, smem + (size_t)st * stage_bytes(p.cap), p.cap);
    __syncthreads();
    if (threadIdx.x == 0 && i + p.D < nmine) {
      tma::fence_proxy_async_smem();
      issue(p, blockIdx.x + (i + p.D) * G, smem + (size_t)st * stage_bytes(p.cap), p.cap,
            bars + st);
    }
  }
  return part;
}

__device__ __forceinline__ void init_bars(const Params &p, unsigned char *smem) {
  unsigned long long *bars =
      (unsigned long long *)(smem + (size_t)p.D * stage_bytes(p.cap));
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.D; ++i) tma::mbar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 2) spmv_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  init_bars(p, smem);
  unsigned phase = 0;
  run<false>(p, smem, phase);
}

}  // namespace spmv_tma
