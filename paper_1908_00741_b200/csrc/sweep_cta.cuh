// HBMC substitution sweep, two-pass CTA version (sm_100a).
//
// Same arithmetic as K/numba_backend.py:132-171, bitwise.  A CTA owns
// `bpc` consecutive level-1 blocks of one color (bpc * b_s * w rows, one
// thread per row), i.e. a contiguous row range and a contiguous range of
// SELL slices.
//
//   pass 1 (every thread = one row, all rows at once): load the row's rhs,
//     inv_d and all its SELL slots (column + value; coalesced across the w
//     lanes of a slice), gather every cross-color operand (final before this
//     phase), and stage per slot either the product v*x (cross), or v and the
//     in-block source step (same lane, other step), or v and a padding mark
//     (col == own row) in shared memory.  All global loads of the block are
//     in flight together: one DRAM round trip plus one gather round trip.
//   pass 2 (one thread per lane of each block): the b_s-step chain entirely
//     out of shared memory: y = rhs; y = y - prod (stored order);
//     y = y * inv_d; store.  In-block operands are the lane's own results of
//     earlier steps, written over the staged rhs.
//
// Products __dmul_rn, updates __dsub_rn, slot order = the reference's.

#pragma once

namespace sweep_cta {

constexpr int kCross = -1;  // staged value is the finished product v*x
constexpr int kPad = -2;    // padding slot: v * (in-progress value)

struct Params {
  const long long *slice_ptr;
  const int *slice_len;
  const int *col;
  const double *val;
  const double *inv_d;
  const double *src;
  double *dst;
  int w, b_s, bpc, lmax;
  int k0, k1;  // level-1 blocks of this color
  const int *done;
};

// shared memory: pv[lmax][R] doubles | ys[R] | id[R] | cd[lmax][R] shorts | len[R] shorts
__host__ __device__ inline size_t smem_bytes(int rows, int lmax) {
  return (size_t)rows * (lmax * 8 + 16) + (((size_t)rows * (lmax + 1) * 2 + 15) / 16) * 16;
}

template <bool FWD>
__global__ void __launch_bounds__(1024) sweep_kernel(Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (p.done && *(const volatile int *)p.done) return;
  const int w = p.w, b_s = p.b_s, lmax = p.lmax;
  const int span = b_s * w;
  const int R = p.bpc * span;  // rows of this CTA (== blockDim.x)
  double *pv = (double *)smem;
  double *ys = pv + (size_t)lmax * R;
  double *id = ys + R;
  short *cd = (short *)(id + R);
  short *ln = cd + (size_t)lmax * R;

  const int kfirst = p.k0 + blockIdx.x * p.bpc;
  const int r = threadIdx.x;
  const int kk = r / span;
  const int rr = r - kk * span;
  const int l = rr / w;
  const int j = rr - l * w;
  const int k = kfirst + kk;
  const int blk0 = k * span;
  const unsigned uspan = (unsigned)span;
  // ---------------- pass 1
  if (k < p.k1) {
    const int sid = k * b_s + l;
    const int grow = blk0 + rr;
    const int off = (int)p.slice_ptr[sid] + j;
    const int len = p.slice_len[sid];
    ys[r] = __ldg(p.src + grow);
    id[r] = __ldg(p.inv_d + grow);
    ln[r] = (short)len;
    for (int t0 = 0; t0 < len; t0 += 8) {
      int c[8];
      double v[8], x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool in = t0 + u < len;
        c[u] = in ? __ldg(p.col + off + (t0 + u) * w) : grow;
        v[u] = in ? __ldg(p.val + off + (t0 + u) * w) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool inblk = (unsigned)(c[u] - blk0) < uspan;
        x[u] = inblk ? 0.0 : __ldg(p.dst + c[u]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = t0 + u;
        if (t < len) {
          const bool inblk = (unsigned)(c[u] - blk0) < uspan;
          short code;
          double sv;
          if (!inblk) {
            code = kCross;
            sv = __dmul_rn(v[u], x[u]);
          } else if (c[u] == grow) {
            code = kPad;
            sv = v[u];
          } else {
            code = (short)((c[u] - blk0) / w);  // source step
            sv = v[u];
          }
          pv[(size_t)t * R + r] = sv;
          cd[(size_t)t * R + r] = code;
        }
      }
    }
  }
  __syncthreads();
  // ---------------- pass 2: one chain per lane (threads with l == 0)
  if (l == 0 && k < p.k1) {
    const int base = kk * span + j;
    for (int ii = 0; ii < b_s; ++ii) {
      const int ls = FWD ? ii : b_s - 1 - ii;
      const int rl = base + ls * w;
      double y = ys[rl];
      const int len = ln[rl];
      for (int t = 0; t < len; ++t) {
        const int code = cd[(size_t)t * R + rl];
        const double sv = pv[(size_t)t * R + rl];
        double prod;
        if (code == kCross)
          prod = sv;
        else if (code == kPad)
          prod = __dmul_rn(sv, y);
        else
          prod = __dmul_rn(sv, ys[base + code * w]);
        y = __dsub_rn(y, prod);
      }
      y = __dmul_rn(y, id[rl]);
      ys[rl] = y;
      p.dst[blk0 + ls * w + j] = y;
    }
  }
}

}  // namespace sweep_cta
