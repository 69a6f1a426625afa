// HBMC substitution sweep, lean thread-per-lane version (sm_100a).
//
// Same arithmetic as K/numba_backend.py:132-171, bitwise.  One thread per
// (level-1 block k, lane j); the thread walks its b_s rows.  The walk is a
// chain of dependent steps, so the lane chain is built to keep DRAM traffic
// in flight while each step waits on its gathers, with a short instruction
// stream:
//   * all step descriptors (slice offset, length) are loaded up front into
//     the thread's column of shared memory;
//   * the first KC slots (columns + values), rhs and inv_d of step i+1 are
//     loaded while step i issues its gathers and runs its chain -- two
//     register buffers used ping-pong (the step loop is unrolled by two), so
//     no register copies; slots beyond KC (rare) are loaded synchronously;
//   * with W = 32 known at compile time every slot load is an immediate
//     offset from one base pointer per step;
//   * in-block operands (same lane, earlier step) are read back from the
//     thread's results in shared memory (branch-free, clamped index);
//   * 32-bit row / column / slot arithmetic (the host checks the ranges).
// Products __dmul_rn, updates __dsub_rn, slot order = the reference's; a
// padding slot (col == own row, v == 0) multiplies the in-progress value.
//
// lane_chain() is shared by the per-phase kernel below (CG = false: vectors
// read through the read-only path, valid because every phase is its own
// launch) and the persistent kernel of persist.cuh (CG = true: vectors that
// other CTAs wrote inside the same launch are read with ld.global.cg).

#pragma once


namespace sweep_lean {

template <int KC>
struct Buf {
  int c[KC];
  double v[KC];
  double rhs, idg;
};

template <bool CG>
__device__ __forceinline__ double ldv(const double *p) {
  return CG ? __ldcg(p) : __ldg(p);
}

// Streamed (read-once) factor entries of the per-phase kernels: read-only
// path with an L2 evict-first policy, so the stream does not flush the
// vectors the gathers read.
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int ld_stream(const int *p, unsigned long long pol) {
  int v;
  asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_stream(const double *p, unsigned long long pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// Predicated gather as a volatile load: the compiler keeps every gather of
// a step ahead of the step's first update instead of sinking each one into
// its slot's branch (which serialises the gathers behind the chain -- seen
// in the SASS of the KC = 24 kernel: LDG, DMUL, DADD, LDG, ...).  CG: L2
// only (vectors written by other CTAs inside the launch); else read-only.
template <bool CG>
__device__ __forceinline__ double ld_gather(const double *p, bool pred) {
  double v;
  if (CG)
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b64 %0, 0;\n"
        " @q ld.global.cg.f64 %0, [%1];\n}"
        : "=d"(v) : "l"(p), "r"((int)pred));
  else
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b64 %0, 0;\n"
        " @q ld.global.nc.f64 %0, [%1];\n}"
        : "=d"(v) : "l"(p), "r"((int)pred));
  return v;
}

// One lane's b_s-step walk.  W > 0: compile-time slice width; W == 0: w_rt.
// Shared memory: ys/offs/lens columns of this thread ([b_s][nt] each).
// dotv != nullptr: also accumulate dotv[row] * result into *dotacc (r . z
// fused into the backward sweep), rows in walk order.
template <bool FWD, int KC, int W, bool CG>
__device__ __forceinline__ void lane_chain(const long long *__restrict__ slice_ptr,
                                           const int *__restrict__ slice_len,
                                           const int *__restrict__ col,
                                           const double *__restrict__ val,
                                           const double *__restrict__ inv_d,
                                           const double *src, double *dst, int w_rt, int b_s,
                                           int k, int j, double *ys, int *offs, int *lens,
                                           const double *dotv = nullptr,
                                           double *dotacc = nullptr) {
  const int w = W > 0 ? W : w_rt;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int span = b_s * w;
  const int blk0 = k * span;
  const unsigned uspan = (unsigned)span;

  // walk step i is slice sid(i) = k*b_s + (FWD ? i : b_s-1-i)
  for (int i = 0; i < b_s; ++i) {
    const int sid = k * b_s + (FWD ? i : b_s - 1 - i);
    offs[i * nt + tid] = (int)slice_ptr[sid] + j;
    lens[i * nt + tid] = slice_len[sid];
  }

  // per-phase launches only (the persistent kernel is register-tight);
  // kNN precond 796 -> 779 us (profiles r03i)
  constexpr bool HINT = !CG;
  unsigned long long pol = 0;
  if (HINT) pol = policy_evict_first();
  auto load = [&](int i, Buf<KC> &b) {
    const int off = offs[i * nt + tid], len = lens[i * nt + tid];
    const int row = blk0 + (FWD ? i : b_s - 1 - i) * w + j;
    const int *cp = col + off;
    const double *vp = val + off;
#pragma unroll
    for (int u = 0; u < KC; ++u) {
      const bool in = u < len;
      if (HINT) {
        b.c[u] = in ? ld_stream(cp + u * w, pol) : row;
        b.v[u] = in ? ld_stream(vp + u * w, pol) : 0.0;
      } else {
        b.c[u] = in ? __ldg(cp + u * w) : row;
        b.v[u] = in ? __ldg(vp + u * w) : 0.0;
      }
    }
    b.rhs = ldv<CG>(src + row);
    b.idg = __ldg(inv_d + row);
  };

  auto step = [&](int i, const Buf<KC> &b) {
    const int l = FWD ? i : b_s - 1 - i;
    const int row = blk0 + l * w + j;
    const int len = lens[i * nt + tid];
    double x[KC];
#pragma unroll
    for (int u = 0; u < KC; ++u) {
      const bool inblk = (unsigned)(b.c[u] - blk0) < uspan;
      // KC <= 8 (every persistent kernel): ptxas already batches the
      // gathers, and the volatile form would cost spills at 128 registers
      x[u] = KC > 8 ? ld_gather<CG>(dst + b.c[u], !inblk) : inblk ? 0.0 : ldv<CG>(dst + b.c[u]);
    }
    double y = b.rhs;
    // branch-free slot update: the shared-memory read is clamped in range
    // and selected away for cross / padding slots
    auto update = [&](int cc, double vv, double xcross) {
      const unsigned rel = (unsigned)(cc - blk0);
      const bool inblk = rel < uspan;
      unsigned lp = W > 0 ? rel / (unsigned)W : rel / (unsigned)w;
      lp = lp < (unsigned)b_s ? lp : 0u;
      const double ysv = ys[(FWD ? (int)lp : b_s - 1 - (int)lp) * nt + tid];
      const double xin = cc == row ? y : ysv;
      const double xv = inblk ? xin : xcross;
      y = __dsub_rn(y, __dmul_rn(vv, xv));
    };
#pragma unroll
    for (int u = 0; u < KC; ++u)
      if (u < len) update(b.c[u], b.v[u], x[u]);
    if (len > KC) {  // long row: the remaining slots
      const int off = offs[i * nt + tid];
      if constexpr (KC > 8) {
        // chunks of 4 with every load of a chunk in flight together
        // (volatile loads keep ptxas from serialising them behind the chain)
        for (int t0 = KC; t0 < len; t0 += 4) {
          int cc[4];
          double vv[4], xc[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const bool in = t0 + u < len;
            const int *cp = col + off + (t0 + u) * w;
            int c;
            asm volatile(
                "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b32 %0, %3;\n"
                " @q ld.global.nc.u32 %0, [%1];\n}"
                : "=r"(c) : "l"(cp), "r"((int)in), "r"(row));
            cc[u] = c;
            vv[u] = ld_gather<false>(val + off + (t0 + u) * w, in);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            xc[u] = ld_gather<CG>(dst + cc[u], (unsigned)(cc[u] - blk0) >= uspan);
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (t0 + u < len) update(cc[u], vv[u], xc[u]);
        }
      } else {
        for (int t = KC; t < len; ++t) {
          const int cc = __ldg(col + off + t * w);
          const double vv = __ldg(val + off + t * w);
          const double xc = (unsigned)(cc - blk0) < uspan ? 0.0 : ldv<CG>(dst + cc);
          update(cc, vv, xc);
        }
      }
    }
    y = __dmul_rn(y, b.idg);
    ys[i * nt + tid] = y;
    dst[row] = y;
    if (dotv) *dotacc += ldv<CG>(dotv + row) * y;
  };

  // operands of step i+1 load while step i gathers and runs its chain: two
  // register buffers used ping-pong (the loop is unrolled by two)
  Buf<KC> A, B;
  load(0, A);
  int i = 0;
  for (; i + 1 < b_s; i += 2) {
    load(i + 1, B);
    step(i, A);
    if (i + 2 < b_s) load(i + 2, A);
    step(i + 1, B);
  }
  if (i < b_s) step(i, A);
}

template <bool FWD, int KC, int W>
__global__ void __launch_bounds__(256, 1)
    sweep_kernel(const long long *__restrict__ slice_ptr, const int *__restrict__ slice_len,
                 const int *__restrict__ col, const double *__restrict__ val,
                 const double *__restrict__ inv_d, const double *__restrict__ src,
                 double *__restrict__ dst, int w_rt, int b_s, int k0, int nthreads,
                 const int *done) {
  // shared: ys[b_s][T] doubles | offs[b_s][T] ints | lens[b_s][T] ints
  extern __shared__ __align__(16) double ys[];
  if (done && *(const volatile int *)done) return;
  const int w = W > 0 ? W : w_rt;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nthreads) return;
  int *offs = (int *)(ys + (size_t)b_s * blockDim.x);
  int *lens = offs + (size_t)b_s * blockDim.x;
  const int kq = g / w;
  lane_chain<FWD, KC, W, false>(slice_ptr, slice_len, col, val, inv_d, src, dst, w, b_s,
                                k0 + kq, g - kq * w, ys, offs, lens);
}

// Per-phase lean sweep with the partitioned solve's halo push fused in
// (tb_plan_sweep_phase_push, w = 32): after its walk a thread stores each of
// its b_s results that peers need straight into their vectors (remote
// stores over NVLink), then the last CTA out releases the phase's epoch into
// every peer's flag for this rank.
template <bool FWD, int KC>
__global__ void __launch_bounds__(256, 1)
    sweep_push_kernel(const long long *__restrict__ slice_ptr, const int *__restrict__ slice_len,
                      const int *__restrict__ col, const double *__restrict__ val,
                      const double *__restrict__ inv_d, const double *__restrict__ src,
                      double *__restrict__ dst, int b_s, int k0, int nthreads,
                      const tb_push_desc pd) {
  extern __shared__ __align__(16) double ys[];
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  int *offs = (int *)(ys + (size_t)b_s * blockDim.x);
  int *lens = offs + (size_t)b_s * blockDim.x;
  if (g < nthreads) {
    const int kq = g >> 5, j = g & 31;
    lane_chain<FWD, KC, 32, false>(slice_ptr, slice_len, col, val, inv_d, src, dst, 32, b_s,
                                   k0 + kq, j, ys, offs, lens);
    const long long blk0 = (long long)(k0 + kq) * b_s * 32;
    for (int i = 0; i < b_s; ++i) {
      const int l = FWD ? i : b_s - 1 - i;
      const long long rel = blk0 + l * 32 + j - pd.row0;
      if (rel < 0 || rel >= pd.nrows) continue;
      const double y = ys[i * blockDim.x + threadIdx.x];
      for (int q = pd.ptr[rel]; q < pd.ptr[rel + 1]; ++q) pd.peer_dst[pd.peer[q]][pd.off[q]] = y;
    }
  }
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(pd.done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) {
    if (threadIdx.x == 0) *pd.done_ctr = 0;
    __threadfence_system();
    if (threadIdx.x < pd.npeers)
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pd.peer_flag[threadIdx.x]),
                   "r"(pd.epoch)
                   : "memory");
  }
}

__host__ inline size_t smem_bytes(int b_s, int threads) { return (size_t)b_s * threads * 16; }

}  // namespace sweep_lean
