// HBMC substitution sweep with a CTA-wide TMA operand ring (sm_100a).
//
// Same arithmetic as K/numba_backend.py:132-171, bitwise (products
// __dmul_rn, updates __dsub_rn, the reference's slot order, padding slots
// multiply the in-progress value).
//
// The lean kernel (sweep_lean.cuh) keeps one step's operands per thread in
// registers, so the bytes a lane chain has in flight are bounded by the
// register file.  Here the static operands never touch a register until
// they are consumed:
//   * a GROUP = kG consecutive level-1 blocks of one color, one per consumer
//     warp; the group's step-l slices are one contiguous range of the
//     step-major factor arrays (device.cu:upload_sell_step_major);
//   * a JOB = (group, step).  One producer thread streams jobs into a
//     D-stage shared-memory ring: the slice values and columns by two 1-D
//     bulk copies, the rhs rows and inv_d rows of the kG blocks by two 3-D
//     tensor copies (vector viewed as [block][step][lane], box = kG x 1 x
//     32), all completing on the stage's mbarrier.  Slice descriptors
//     (slice_ptr / slice_len of the group) are bulk-copied one group ahead.
//     The ring crosses group boundaries, so it never drains inside a launch;
//   * consumer warp i walks block i's lane chains from shared memory.  The
//     cross-color gathers of job q + A are issued (volatile predicated
//     loads into a rotating register set) before the chain of job q runs:
//     the only global latency left on the chain is hidden A steps deep;
//   * consumers release a stage with one mbarrier arrive per warp.
// CTAs are persistent over the color's groups (round-robin).

#pragma once

#include <cuda.h>

#include "tma_util.cuh"

namespace sweep_group {

constexpr int kG = 8;                    // consumer warps = level-1 blocks per group
constexpr int kThreads = (kG + 1) * 32;  // + the producer warp
constexpr int kNDesc = 4;                // descriptor buffers (groups)
constexpr int kNSet = 4;                 // rotating gather register sets

struct Params {
  const long long *slice_ptr;
  const int *slice_len;
  const int *col;
  const double *val;
  double *dst;
  int b_s, k0, k1;  // level-1 block range [k0, k1) of the color
  int cap;          // slot capacity of a stage (multiple of 32)
  int D;            // stages
  const int *done;  // solve-finished flag (kernel-sequence PCG), or null
};

__host__ __device__ inline size_t stage_bytes(int cap) { return (size_t)cap * 12 + kG * 512; }
__host__ __device__ inline size_t desc_bytes(int b_s) { return (size_t)kG * b_s * 12; }
__host__ __device__ inline size_t smem_bytes(int cap, int D, int b_s) {
  return (size_t)D * stage_bytes(cap) + kNDesc * desc_bytes(b_s) + (size_t)kG * b_s * 256 +
         (size_t)(2 * D + 2 * kNDesc) * 8 + 128;
}

__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tma::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tensor3_g2s(void *dst, const CUtensorMap *tm, int c0, int c1,
                                            int c2, unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(tma::smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(tma::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ double ld_gather_nc(const double *p, bool pred) {
  double v;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b64 %0, 0;\n"
      " @q ld.global.nc.f64 %0, [%1];\n}"
      : "=d"(v)
      : "l"(p), "r"((int)pred));
  return v;
}

// FWD: forward (L, steps ascending) / backward (U, steps descending).
// KC: slots per step held in a gather register set (longer slices finish
// with synchronous gathers).  A: steps the gathers run ahead (1..3).
template <bool FWD, int KC, int A>
__global__ void __launch_bounds__(kThreads, 1)
    sweep_kernel(const __grid_constant__ CUtensorMap tm_rhs,
                 const __grid_constant__ CUtensorMap tm_idg, const Params P) {
  extern __shared__ __align__(128) unsigned char smem[];
  static_assert(A >= 1 && A < kNSet, "gather distance");
  if (P.done && *(const volatile int *)P.done) return;
  const int b_s = P.b_s, D = P.D, cap = P.cap;
  const size_t sbytes = stage_bytes(cap);
  unsigned char *stages = smem;
  unsigned char *descs = smem + (size_t)D * sbytes;
  double *ys = (double *)(descs + kNDesc * desc_bytes(b_s));
  unsigned long long *full = (unsigned long long *)(ys + (size_t)kG * b_s * 32);
  unsigned long long *empty = full + D;
  unsigned long long *dfull = empty + D;
  unsigned long long *dempty = dfull + kNDesc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < D; ++i) {
      tma::mbar_init(full + i, 1);
      tma::mbar_init(empty + i, kG);
    }
    for (int i = 0; i < kNDesc; ++i) {
      tma::mbar_init(dfull + i, 1);
      tma::mbar_init(dempty + i, kG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int ng = (P.k1 - P.k0 + kG - 1) / kG;
  const int nmine = ng > (int)blockIdx.x ? (ng - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto sp_of = [&](int db) { return (const long long *)(descs + (size_t)db * desc_bytes(b_s)); };
  auto sl_of = [&](int db) {
    return (const int *)(descs + (size_t)db * desc_bytes(b_s) + (size_t)kG * b_s * 8);
  };
  auto kg0_of = [&](int t) { return P.k0 + ((int)blockIdx.x + t * (int)gridDim.x) * kG; };

  if (warp == kG) {
    // ------------------------------------------------------------ producer
    if (lane != 0) return;
    auto issue_desc = [&](int t) {
      const int kg0 = kg0_of(t);
      const int gn = P.k1 - kg0 < kG ? P.k1 - kg0 : kG;
      const int db = t % kNDesc;
      if (t >= kNDesc) tma::mbar_wait(dempty + db, (unsigned)((t / kNDesc - 1) & 1));
      const unsigned cnt = (unsigned)(gn * b_s);
      tma::mbar_arrive_expect_tx(dfull + db, cnt * 12u);
      tma::bulk_g2s((void *)sp_of(db), P.slice_ptr + (long long)kg0 * b_s, cnt * 8u, dfull + db);
      tma::bulk_g2s((void *)sl_of(db), P.slice_len + (long long)kg0 * b_s, cnt * 4u, dfull + db);
    };
    if (nmine > 0) issue_desc(0);
    int st = 0, pass = 0;
    for (int t = 0; t < nmine; ++t) {
      if (t + 1 < nmine) issue_desc(t + 1);
      const int db = t % kNDesc;
      tma::mbar_wait(dfull + db, (unsigned)((t / kNDesc) & 1));
      const long long *sp = sp_of(db);
      const int *sl = sl_of(db);
      const int kg0 = kg0_of(t);
      const int gn = P.k1 - kg0 < kG ? P.k1 - kg0 : kG;
      for (int s = 0; s < b_s; ++s) {
        const int l = FWD ? s : b_s - 1 - s;
        if (pass > 0) tma::mbar_wait(empty + st, (unsigned)((pass - 1) & 1));
        const long long a = sp[l];
        const long long e = sp[(gn - 1) * b_s + l] + (long long)sl[(gn - 1) * b_s + l] * 32;
        const unsigned cnt = (unsigned)(e - a);
        unsigned char *stg = stages + (size_t)st * sbytes;
        tma::mbar_arrive_expect_tx(full + st, cnt * 12u + kG * 512u);
        if (cnt) {
          tma::bulk_g2s(stg, P.val + a, cnt * 8u, full + st);
          tma::bulk_g2s(stg + (size_t)cap * 8, P.col + a, cnt * 4u, full + st);
        }
        tensor3_g2s(stg + (size_t)cap * 12, &tm_rhs, 0, l, kg0, full + st);
        tensor3_g2s(stg + (size_t)cap * 12 + kG * 256, &tm_idg, 0, l, kg0, full + st);
        if (++st == D) {
          st = 0;
          ++pass;
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  double *ysw = ys + (size_t)warp * b_s * 32;
  const unsigned uspan = (unsigned)(b_s * 32);
  int gst = 0;        // stage of the next job whose gathers are issued
  unsigned gph = 0;   // its full-barrier parity
  int cst = 0;        // stage of the next job whose chain runs
  double xg[kNSet][KC];

  // job (t, s): wait for its stage, issue its cross-color gathers into x
  auto issue = [&](int t, int s, double (&x)[KC]) {
    const int db = t % kNDesc;
    if (s == 0) tma::mbar_wait(dfull + db, (unsigned)((t / kNDesc) & 1));
    tma::mbar_wait(full + gst, gph);
    const int l = FWD ? s : b_s - 1 - s;
    const int kg0 = kg0_of(t);
    const bool active = kg0 + warp < P.k1;
    const long long *sp = sp_of(db);
    const int off = active ? (int)(sp[warp * b_s + l] - sp[l]) + lane : 0;
    const int len = active ? sl_of(db)[warp * b_s + l] : 0;
    const int blk0 = (kg0 + warp) * b_s * 32;
    const int *sc = (const int *)(stages + (size_t)gst * sbytes + (size_t)cap * 8) + off;
#pragma unroll
    for (int u = 0; u < KC; ++u) {
      const int c = u < len ? sc[u * 32] : blk0;
      x[u] = ld_gather_nc(P.dst + c, (unsigned)(c - blk0) >= uspan);
    }
    if (++gst == D) {
      gst = 0;
      gph ^= 1u;
    }
  };

  // job (t, s): the lane's row of step s from the stage + gathered x
  auto chain = [&](int t, int s, const double (&x)[KC]) {
    const int db = t % kNDesc;
    const int l = FWD ? s : b_s - 1 - s;
    const int kg0 = kg0_of(t);
    const bool active = kg0 + warp < P.k1;
    const long long *sp = sp_of(db);
    const int off = active ? (int)(sp[warp * b_s + l] - sp[l]) + lane : 0;
    const int len = active ? sl_of(db)[warp * b_s + l] : 0;
    const int blk0 = (kg0 + warp) * b_s * 32;
    const int row = blk0 + l * 32 + lane;
    const unsigned char *stg = stages + (size_t)cst * sbytes;
    const double *sv = (const double *)stg + off;
    const int *sc = (const int *)(stg + (size_t)cap * 8) + off;
    const double *srhs = (const double *)(stg + (size_t)cap * 12);
    double y = srhs[warp * 32 + lane];
    const double idg = srhs[kG * 32 + warp * 32 + lane];
    auto update = [&](int c, double v, double xc) {
      const unsigned rel = (unsigned)(c - blk0);
      const bool inblk = rel < uspan;
      const unsigned lp = inblk ? rel >> 5 : 0u;
      const double ysv = ysw[lp * 32 + lane];
      const double xin = c == row ? y : ysv;
      y = __dsub_rn(y, __dmul_rn(v, inblk ? xin : xc));
    };
#pragma unroll
    for (int u = 0; u < KC; ++u)
      if (u < len) update(sc[u * 32], sv[u * 32], x[u]);
    for (int u = KC; u < len; ++u) {  // longer than the register set: rare
      const int c = sc[u * 32];
      const bool cross = (unsigned)(c - blk0) >= uspan;
      update(c, sv[u * 32], cross ? __ldg(P.dst + c) : 0.0);
    }
    y = __dmul_rn(y, idg);
    ysw[l * 32 + lane] = y;
    if (active) P.dst[row] = y;
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(empty + cst);
      if (s == b_s - 1) mbar_arrive(dempty + db);
    }
    if (++cst == D) cst = 0;
  };

  if (nmine == 0) return;
#pragma unroll
  for (int a = 0; a < A; ++a) issue(0, a, xg[a]);  // b_s >= 4 > A
  for (int t = 0; t < nmine; ++t) {
    for (int s0 = 0; s0 < b_s; s0 += kNSet) {
#pragma unroll
      for (int d = 0; d < kNSet; ++d) {
        const int s = s0 + d;
        int sa = s + A, ta = t;
        if (sa >= b_s) {
          sa -= b_s;
          ++ta;
        }
        if (ta < nmine) issue(ta, sa, xg[(d + A) % kNSet]);
        chain(t, s, xg[d]);
      }
    }
  }
}

}  // namespace sweep_group
