// HBMC substitution sweep, cp.async-pipelined thread-per-lane version.
//
// Same arithmetic as K/numba_backend.py:132-171, bitwise.  One thread per
// (level-1 block k, lane j) walking its b_s rows.  The walk is a chain of
// b_s dependent steps, so the kernel keeps D steps of operands in flight per
// thread without spending registers on them: each thread streams its steps'
// values, columns, rhs and inv_d into its own slots of a D-deep shared-memory
// ring with cp.async (LDGSTS; one commit group per step), D steps ahead of
// the step it computes.  The cross-color gathers of step i+1 are issued
// before step i's chain runs.  In-block operands (same lane, earlier step)
// come from the thread's results, kept in shared memory.
//
// Shared memory is struct-of-arrays over the CTA's threads (conflict free).
// Products __dmul_rn, updates __dsub_rn, slot order = the reference's.

#pragma once

namespace sweep_async {

constexpr int kThreads = 128;
constexpr int kMaxD = 8;

__device__ __forceinline__ unsigned s32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp4(void *s, const void *g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp8(void *s, const void *g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct Params {
  const long long *slice_ptr;
  const int *slice_len;
  const int *col;
  const double *val;
  const double *inv_d;
  const double *src;
  double *dst;
  int w, b_s, lmax, k0, nthreads;
  const int *done;
};

// per-CTA shared memory
//   ring[D]: vals[lmax][T] f64 | rhs[T] | invd[T] | cols[lmax][T] i32
//   ys[b_s][T] f64 | off[b_s][T] i32 | len[b_s][T] i32
__host__ __device__ inline size_t slot_bytes(int lmax) {
  return (size_t)kThreads * (lmax * 12 + 16);
}
__host__ __device__ inline size_t smem_bytes(int D, int lmax, int b_s) {
  return (size_t)D * slot_bytes(lmax) + (size_t)b_s * kThreads * 16;
}

template <bool FWD, int D>
__global__ void __launch_bounds__(kThreads) sweep_kernel(Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (p.done && *(const volatile int *)p.done) return;
  const int T = kThreads, tid = threadIdx.x;
  const int g = blockIdx.x * T + tid;
  const bool live = g < p.nthreads;
  const int w = p.w, b_s = p.b_s, lmax = p.lmax;
  const int kq = (live ? g : 0) / w;
  const int j = (live ? g : 0) - kq * w;
  const int k = p.k0 + kq;
  const int span = b_s * w;
  const int blk0 = k * span;
  const unsigned uspan = (unsigned)span;
  const size_t sb = slot_bytes(lmax);
  double *ys = (double *)(smem + (size_t)D * sb);
  int *offs = (int *)(ys + (size_t)b_s * T);
  int *lens = offs + (size_t)b_s * T;
  auto vals_of = [&](int d) { return (double *)(smem + (size_t)d * sb); };
  auto cols_of = [&](int d) { return (int *)(smem + (size_t)d * sb + (size_t)T * (lmax * 8 + 16)); };

  // step descriptors for the whole walk (one batch of loads)
  if (live)
    for (int i = 0; i < b_s; ++i) {
      const int l = FWD ? i : b_s - 1 - i;
      const int sid = k * b_s + l;
      offs[i * T + tid] = (int)p.slice_ptr[sid] + j;
      lens[i * T + tid] = p.slice_len[sid];
    }
  // cp.async the operands of walk step i into ring slot i % D
  auto issue = [&](int i) {
    if (live && i < b_s) {
      const int d = i % D;
      const int l = FWD ? i : b_s - 1 - i;
      const int row = blk0 + l * w + j;
      const int off = offs[i * T + tid], len = lens[i * T + tid];
      double *vs = vals_of(d);
      int *cs = cols_of(d);
      for (int t = 0; t < len; ++t) {
        cp8(vs + (size_t)t * T + tid, p.val + off + t * w);
        cp4(cs + (size_t)t * T + tid, p.col + off + t * w);
      }
      cp8(vs + (size_t)lmax * T + tid, p.src + row);
      cp8(vs + (size_t)(lmax + 1) * T + tid, p.inv_d + row);
    }
    commit();  // always commit: group i == walk step i
  };
#pragma unroll
  for (int i = 0; i < D; ++i) issue(i);

  constexpr int kG = 8;  // gathers held in registers per step
  double xg[kG];
  auto gather = [&](int i) {
    const int d = i % D;
    const int *cs = cols_of(d);
    const int len = (live && i < b_s) ? lens[i * T + tid] : 0;
#pragma unroll
    for (int t = 0; t < kG; ++t) {
      double xv = 0.0;
      if (t < len) {
        const int c = cs[(size_t)t * T + tid];
        if ((unsigned)(c - blk0) >= uspan) xv = __ldg(p.dst + c);
      }
      xg[t] = xv;
    }
  };

  wait_group<D - 1>();  // step 0 landed
  gather(0);
  for (int i = 0; i < b_s; ++i) {
    double xc[kG];
#pragma unroll
    for (int t = 0; t < kG; ++t) xc[t] = xg[t];
    // step i+1's operands, then its gathers, ahead of step i's chain
    if (i + 1 < b_s) {
      wait_group<D - 2 >= 0 ? D - 2 : 0>();
      gather(i + 1);
    }
    if (live) {
      const int d = i % D;
      const int l = FWD ? i : b_s - 1 - i;
      const int row = blk0 + l * w + j;
      const double *vs = vals_of(d);
      const int *cs = cols_of(d);
      const int len = lens[i * T + tid];
      double y = vs[(size_t)lmax * T + tid];
      auto update = [&](int t, double xcross) {
        const int c = cs[(size_t)t * T + tid];
        const double v = vs[(size_t)t * T + tid];
        double xv;
        if ((unsigned)(c - blk0) >= uspan) {
          xv = xcross;
        } else if (c == row) {
          xv = y;
        } else {
          const int lp = w == 32 ? (c - blk0) >> 5 : (c - blk0) / w;
          xv = ys[(size_t)(FWD ? lp : b_s - 1 - lp) * T + tid];
        }
        y = __dsub_rn(y, __dmul_rn(v, xv));
      };
#pragma unroll
      for (int t = 0; t < kG; ++t)
        if (t < len) update(t, xc[t]);
      for (int t = kG; t < len; ++t) update(t, __ldg(p.dst + cs[(size_t)t * T + tid]));
      y = __dmul_rn(y, vs[(size_t)(lmax + 1) * T + tid]);
      ys[(size_t)i * T + tid] = y;
      p.dst[row] = y;
    }
    issue(i + D);  // refill the slot just consumed (an empty group past the end)
  }
}

}  // namespace sweep_async
