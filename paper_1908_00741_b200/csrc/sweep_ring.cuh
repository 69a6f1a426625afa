// HBMC substitution sweep for w = 32: per-warp TMA ring over steps (sm_100a).
//
// Same arithmetic as K/numba_backend.py:132-171, bitwise.  Mapping: one warp
// = one level-1 block at a time (lane m = constituent BMC block m); warps are
// persistent over the color's level-1 blocks.  A warp's work is the sequence
// of its blocks' b_s steps; one STEP is one SELL slice (32 rows, `len`
// column-major slots: 32*len values + 32*len columns, contiguous) plus the
// 32 rhs and inv_d entries of those rows (contiguous).  Lane 0 streams steps
// into a ring of R shared-memory stages with 1-D TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx), R steps ahead of the consumer, so
// no DRAM latency sits on the warp's critical path; the step's offsets are
// themselves loaded one step ahead.
//
// Per step, each lane:
//   1. gathers every cross-color operand of its row (earlier colors in the
//      forward sweep, later colors in the backward sweep -- final before the
//      phase started), up to kChunk loads in flight, and forms v*x;
//   2. runs the row's slot chain in stored order: y = y - prod, where an
//      in-block slot (same lane, earlier step) uses v * (lane's earlier
//      result, kept in a per-warp shared array) and the padding slot
//      (col == own row, v == 0) multiplies the in-progress value exactly as
//      the reference does;  y *= inv_d;  store.
// All products __dmul_rn, all updates __dsub_rn: bitwise equal to the
// reference's sequential substitution.

#pragma once

namespace sweep_ring {

constexpr int kMaxWarps = 16;  // warps per CTA (host picks <= this)
constexpr int kMaxRing = 8;    // ring depth (host picks <= this)
constexpr int kChunk = 8;      // gathers in flight per lane per chunk

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
      "RWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra RWAIT_%=;\n"
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

struct Params {
  const long long *slice_ptr;  // [n_slices+1]
  const int *slice_len;        // [n_slices]
  const int *col;
  const double *val;
  const double *inv_d;
  const double *src;
  double *dst;
  int b_s;
  int lmax;                    // max slice length in this color (stage capacity)
  int ring;                    // R
  long long k0, k1;            // level-1 blocks of this color
  const int *done;             // PcgState::done or null
};

// stage: vals[32*lmax] | cols[32*lmax] | rhs[32] | inv_d[32] | len (int, padded)
__host__ __device__ inline size_t st_cols(int lmax) { return (size_t)lmax * 32 * 8; }
__host__ __device__ inline size_t st_rhs(int lmax) { return st_cols(lmax) + (size_t)lmax * 32 * 4; }
__host__ __device__ inline size_t st_len(int lmax) { return st_rhs(lmax) + 2 * 32 * 8; }
__host__ __device__ inline size_t stage_bytes(int lmax) { return st_len(lmax) + 16; }
__host__ __device__ inline size_t warp_bytes(int lmax, int ring, int b_s) {
  return (size_t)ring * stage_bytes(lmax) + (size_t)32 * b_s * 8 + (size_t)kMaxRing * 8;
}

template <bool FWD>
__global__ void __launch_bounds__(kMaxWarps * 32, 1) sweep_kernel(Params p) {
  if (p.done && *(const volatile int *)p.done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b_s = p.b_s, lmax = p.lmax, R = p.ring;
  const size_t sb = stage_bytes(lmax);
  unsigned char *wbase = smem_raw + (size_t)warp * warp_bytes(lmax, R, b_s);
  double *ysm = (double *)(wbase + (size_t)R * sb);
  unsigned long long *bars = (unsigned long long *)(wbase + (size_t)R * sb + (size_t)32 * b_s * 8);

  const int wpc = blockDim.x >> 5;
  const long long gw = (long long)blockIdx.x * wpc + warp;
  const long long nw = (long long)gridDim.x * wpc;
  const long long nblk = p.k1 - p.k0;
  const long long my_blocks = gw < nblk ? (nblk - gw + nw - 1) / nw : 0;
  const long long n_steps = my_blocks * b_s;
  if (n_steps == 0) return;

  if (lane == 0) {
    for (int r = 0; r < R; ++r) mbar_init(&bars[r], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // slice id of the warp's step i
  auto slice_of = [&](long long i) {
    const long long m = i / b_s;
    const int ll = (int)(i - m * b_s);
    const long long k = p.k0 + gw + m * nw;
    return k * b_s + (FWD ? ll : b_s - 1 - ll);
  };
  // lane 0: stage step i (offset/len already known) into ring slot i % R
  auto issue = [&](long long i, long long off, int len) {
    const int s = (int)(i % R);
    unsigned char *stg = wbase + (size_t)s * sb;
    const long long sid = slice_of(i);
    *(int *)(stg + st_len(lmax)) = len;
    const unsigned nbytes = (unsigned)len * 384u + 512u;
    mbar_arrive_expect_tx(&bars[s], nbytes);
    if (len) {
      bulk_g2s(stg, p.val + off, (unsigned)len * 256u, &bars[s]);
      bulk_g2s(stg + st_cols(lmax), p.col + off, (unsigned)len * 128u, &bars[s]);
    }
    bulk_g2s(stg + st_rhs(lmax), p.src + sid * 32, 256u, &bars[s]);
    bulk_g2s(stg + st_rhs(lmax) + 256, p.inv_d + sid * 32, 256u, &bars[s]);
  };

  // prologue: R steps in flight, then the offsets of step R prefetched
  long long pf_off = 0;
  int pf_len = 0;
  if (lane == 0) {
    const long long npro = n_steps < R ? n_steps : R;
    for (long long i = 0; i < npro; ++i) {
      const long long sid = slice_of(i);
      issue(i, p.slice_ptr[sid], p.slice_len[sid]);
    }
    if (R < n_steps) {
      const long long sid = slice_of(R);
      pf_off = p.slice_ptr[sid];
      pf_len = p.slice_len[sid];
    }
  }

  const int span = b_s * 32;
  for (long long i = 0; i < n_steps; ++i) {
    const int s = (int)(i % R);
    const unsigned parity = (unsigned)((i / R) & 1);
    const long long m = i / b_s;
    const int ll = (int)(i - m * b_s);
    const int l = FWD ? ll : b_s - 1 - ll;
    const long long k = p.k0 + gw + m * nw;
    const long long blk_row0 = k * span;
    const long long row = blk_row0 + (long long)l * 32 + lane;
    mbar_wait(&bars[s], parity);
    const unsigned char *stg = wbase + (size_t)s * sb;
    const double *vs = (const double *)stg;
    const int *cs = (const int *)(stg + st_cols(lmax));
    const double *rs = (const double *)(stg + st_rhs(lmax));
    const int len = *(const int *)(stg + st_len(lmax));
    double y = rs[lane];
    for (int t0 = 0; t0 < len; t0 += kChunk) {
      int c[kChunk];
      double pr[kChunk];
#pragma unroll
      for (int u = 0; u < kChunk; ++u) {
        const int t = t0 + u;
        c[u] = t < len ? cs[t * 32 + lane] : (int)row;
      }
#pragma unroll
      for (int u = 0; u < kChunk; ++u) {
        const bool cross = (long long)c[u] < blk_row0 || (long long)c[u] >= blk_row0 + span;
        pr[u] = cross ? __ldg(p.dst + c[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kChunk; ++u) {
        const int t = t0 + u;
        if (t < len) {
          const double v = vs[t * 32 + lane];
          const bool cross = (long long)c[u] < blk_row0 || (long long)c[u] >= blk_row0 + span;
          double prod;
          if (cross) {
            prod = __dmul_rn(v, pr[u]);
          } else {
            const double xv = ((long long)c[u] == row) ? y : ysm[c[u] - blk_row0];
            prod = __dmul_rn(v, xv);
          }
          y = __dsub_rn(y, prod);
        }
      }
    }
    y = __dmul_rn(y, rs[32 + lane]);
    ysm[row - blk_row0] = y;
    p.dst[row] = y;
    __syncwarp();
    // refill the consumed slot with step i + R; prefetch offsets of i + R + 1
    if (lane == 0 && i + R < n_steps) {
      issue(i + R, pf_off, pf_len);
      if (i + R + 1 < n_steps) {
        const long long sid = slice_of(i + R + 1);
        pf_off = p.slice_ptr[sid];
        pf_len = p.slice_len[sid];
      }
    }
  }
}

}  // namespace sweep_ring
