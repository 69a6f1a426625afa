// HBMC substitution sweep, staged version (sm_100a).
//
// Same arithmetic as K/numba_backend.py:132-171 (and as sell_sweep in
// device.cu), restructured for the memory system:
//
//   * one WARP TASK = G = 32 / w consecutive level-1 blocks of one color
//     (w = 32: one level-1 block; w = 8: four).  Their SELL slices are one
//     contiguous range [slice_ptr[k*b_s], slice_ptr[(k+G)*b_s]) of the value
//     and column arrays and their rows one contiguous range of the rhs and
//     inv_d vectors, so the whole task is moved by four 1-D TMA bulk copies
//     (cp.async.bulk, mbarrier complete_tx) into a shared-memory stage.
//     Warps are persistent over the color's tasks and keep 2 stages, so the
//     DRAM stream of task i+1 overlaps the compute of task i.
//   * pass A (gather): every slot whose column lies outside the task's rows
//     -- i.e. an operand of an EARLIER color (forward) / LATER color
//     (backward), final before this phase started -- is gathered (kUnroll
//     gathers in flight per lane) and its product v*x is written back into
//     the stage in place of v.
//   * pass B (chain): each lane walks its b_s rows in order; per slot it
//     subtracts the precomputed product, or, for an in-block slot (same
//     lane, earlier step), v times the lane's earlier result, which lives in
//     the stage's rhs area (written over the consumed rhs); the padding slot
//     (col == own row, v == 0) multiplies the in-progress value exactly like
//     the reference.
//
// Every product is __dmul_rn and every update __dsub_rn in the reference's
// slot order, so the output is bitwise equal to the reference.

#pragma once

namespace sweep_tma {

constexpr int kWarps = 8;    // max warps per CTA
constexpr int kUnroll = 16;  // gathers in flight per lane in pass A

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

struct Params {
  const long long *slice_ptr;  // [n_slices+1] element offsets
  const int *col;              // SELL columns (int32)
  const double *val;           // SELL values
  const double *inv_d;
  const double *src;
  double *dst;
  int w, b_s, G;               // G = 32 / w level-1 blocks per warp task
  long long k0, k1;            // level-1 block range of this color
  long long n_tasks;
  int max_slots;               // max slots of one task (stage capacity, %4 == 0)
  const int *done;             // PcgState::done or null
};

// One stage: vals[max_slots] | cols[max_slots] | rhs[32*b_s] | inv_d[32*b_s]
__host__ __device__ inline size_t cols_off(int max_slots) { return (size_t)max_slots * 8; }
__host__ __device__ inline size_t rhs_off(int max_slots) {
  return cols_off(max_slots) + ((size_t)max_slots * 4 + 15) / 16 * 16;
}
__host__ __device__ inline size_t stage_bytes(int max_slots, int b_s) {
  return rhs_off(max_slots) + (size_t)2 * 32 * b_s * 8;
}
__host__ __device__ inline size_t offs_bytes(int b_s, int G) {
  return ((size_t)(G * b_s + 1) * 8 + 15) / 16 * 16;
}
// Per warp: 2 stages + 2 slice-offset tables + 2 mbarriers.
__host__ __device__ inline size_t warp_smem_bytes(int max_slots, int b_s, int G) {
  return 2 * (stage_bytes(max_slots, b_s) + offs_bytes(b_s, G)) + 16;
}

template <bool FWD>
__global__ void __launch_bounds__(kWarps * 32, 1) sweep_kernel(Params p) {
  if (p.done && *(const volatile int *)p.done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b_s = p.b_s, w = p.w, G = p.G;
  const size_t sb = stage_bytes(p.max_slots, b_s);
  const size_t ob = offs_bytes(b_s, G);
  unsigned char *base = smem_raw + (size_t)warp * warp_smem_bytes(p.max_slots, b_s, G);
  auto stage_ptr = [&](int st) { return base + (st ? sb : 0); };
  auto offs_ptr = [&](int st) { return (long long *)(base + 2 * sb + (st ? ob : 0)); };
  unsigned long long *bars = (unsigned long long *)(base + 2 * sb + 2 * ob);

  const int wpc = blockDim.x >> 5;  // warps per CTA (host-chosen, <= kWarps)
  const long long gwarp = (long long)blockIdx.x * wpc + warp;
  const long long nwarps = (long long)gridDim.x * wpc;
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  const int span = b_s * w;
  // Stage task `t` into stage `s`: the warp loads the task's slice offsets
  // (task-relative) into shared memory, lane 0 arms the stage's mbarrier and
  // issues the bulk copies (values, columns, rhs rows, inv_d rows).  Every
  // lane first fences its earlier generic-proxy writes of the stage (passes
  // A and B write into it) against the async-proxy writes of the copies.
  auto issue = [&](long long t, int s) {
    const long long kb = p.k0 + t * G;
    long long ke = kb + G;
    if (ke > p.k1) ke = p.k1;
    const long long first = kb * b_s, last = ke * b_s;  // slice range
    long long *offs = offs_ptr(s);
    const long long start = p.slice_ptr[first];
    for (long long q = first + lane; q <= last; q += 32) offs[q - first] = p.slice_ptr[q] - start;
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      const unsigned slots = (unsigned)offs[last - first];
      const unsigned rows = (unsigned)((ke - kb) * span);
      unsigned char *stg = stage_ptr(s);
      mbar_arrive_expect_tx(&bars[s], slots * 12u + rows * 16u);
      if (slots) {
        bulk_g2s(stg, p.val + start, slots * 8u, &bars[s]);
        bulk_g2s(stg + cols_off(p.max_slots), p.col + start, slots * 4u, &bars[s]);
      }
      bulk_g2s(stg + rhs_off(p.max_slots), p.src + kb * span, rows * 8u, &bars[s]);
      bulk_g2s(stg + rhs_off(p.max_slots) + (size_t)32 * b_s * 8, p.inv_d + kb * span,
               rows * 8u, &bars[s]);
    }
  };

  unsigned phase_bits = 0u;  // bit s = parity of stage s
  long long t = gwarp;
  if (t < p.n_tasks) issue(t, 0);
  if (t + nwarps < p.n_tasks) issue(t + nwarps, 1);
  int s = 0;
  const int g = lane / w, j = lane - (lane / w) * w;
  for (; t < p.n_tasks; t += nwarps, s ^= 1) {
    const long long kb = p.k0 + t * G;
    const long long warp_row0 = kb * span;
    long long ke = kb + G;
    if (ke > p.k1) ke = p.k1;
    const long long warp_row1 = ke * span;
    const long long kk = kb + g;
    const bool active = (kk < ke) && (g < G);
    mbar_wait(&bars[s], (phase_bits >> s) & 1u);
    phase_bits ^= 1u << s;
    unsigned char *stg = stage_ptr(s);
    double *vs = (double *)stg;
    const int *cs = (const int *)(stg + cols_off(p.max_slots));
    double *ys = (double *)(stg + rhs_off(p.max_slots));  // rhs in, results out
    const double *ids = ys + 32 * b_s;
    const long long *offs = offs_ptr(s);
    const int n_slots = (int)offs[(ke - kb) * b_s];
    // ---- pass A: gather + multiply every cross-phase operand
    for (int q0 = lane; q0 < n_slots; q0 += 32 * kUnroll) {
      int c[kUnroll];
      double x[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int q = q0 + 32 * u;
        c[u] = q < n_slots ? cs[q] : (int)warp_row0;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const bool cross = (long long)c[u] < warp_row0 || (long long)c[u] >= warp_row1;
        x[u] = cross ? __ldcg(p.dst + c[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int q = q0 + 32 * u;
        const bool cross = (long long)c[u] < warp_row0 || (long long)c[u] >= warp_row1;
        if (q < n_slots && cross) vs[q] = __dmul_rn(vs[q], x[u]);
      }
    }
    __syncwarp();
    // ---- pass B: the lane's b_s-step chain
    if (active) {
      const long long sl0 = (kk - kb) * b_s;  // first slice of this lane's block (task-local)
      const int rloc0 = (int)((kk - kb) * span) + j;
      for (int ll = 0; ll < b_s; ++ll) {
        const int l = FWD ? ll : b_s - 1 - ll;
        const int rloc = rloc0 + l * w;           // task-local row
        const int row = (int)(warp_row0 + rloc);
        const int off = (int)offs[sl0 + l];
        const int len = (int)((offs[sl0 + l + 1] - off) / w);
        double y = ys[rloc];
        for (int tt = 0; tt < len; ++tt) {
          const int q = off + tt * w + j;
          const int cc = cs[q];
          double prod;
          if ((long long)cc >= warp_row0 && (long long)cc < warp_row1) {
            const double xv = (cc == row) ? y : ys[cc - (int)warp_row0];
            prod = __dmul_rn(vs[q], xv);
          } else {
            prod = vs[q];
          }
          y = __dsub_rn(y, prod);
        }
        y = __dmul_rn(y, ids[rloc]);
        ys[rloc] = y;
        p.dst[row] = y;
      }
    }
    __syncwarp();
    if (t + 2 * nwarps < p.n_tasks) issue(t + 2 * nwarps, s);
  }
}

}  // namespace sweep_tma
