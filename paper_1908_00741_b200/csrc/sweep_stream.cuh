// HBMC preconditioner application, streamed dataflow version (sm_100a).
//
// z = (L L^T)^-1 r, both sweeps in one launch, bitwise the reference's
// K/numba_backend.py:132-171 (every product __dmul_rn, every update
// __dsub_rn, the slot order of the SELL rows; a padding slot -- col == own
// row, v == 0 -- multiplies the in-progress value).
//
// Schedule: the dataflow item sequence of persist.cuh (forward level-1
// blocks k ascending, then backward k descending; warp gw takes items gw,
// gw + W, ...; before an item the warp waits for the completion flags of the
// blocks its rows read, after it lane 0 publishes the item's flag).
//
// Data path: the lane chain of b_s dependent steps (lane j of block k walks
// rows k*b_s*32 + l*32 + j) is latency-bound when its operands arrive one
// step ahead in registers (the lean kernel: ~47 % of HBM bandwidth at config
// 2).  Here every warp streams the STATIC operands of its step sequence --
// the step's SELL slice (values + int32 columns, one contiguous range) and
// its 32 inv_d -- into a D-deep ring of shared-memory slots with warp-wide
// 16-byte cp.async.cg copies (no registers, L1 bypassed), D-1 steps ahead and
// across item boundaries.  The DYNAMIC operands -- the rhs (r, or the forward
// result y for the backward sweep) and the cross-color gathers of y / z --
// are loaded one step ahead into registers once the item's dependency flags
// are seen: the chain of step i then waits on nothing issued during step i.
// In-block operands (same lane, earlier step) come from the warp's results in
// shared memory.
//
// Per warp shared memory: D slots x (LC*32*12 + 256) B + b_s*32*8 B (results)
// + 64 B, LC = the factor's longest slice.

#pragma once

#include "persist.cuh"

namespace sweep_stream {

__device__ __forceinline__ unsigned s32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp16(void *s, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__host__ __device__ inline size_t slot_bytes(int lc) { return (size_t)lc * 384 + 256; }
__host__ __device__ inline size_t warp_bytes(int lc, int D, int b_s) {
  return (size_t)D * slot_bytes(lc) + (size_t)b_s * 256 + 64;
}

// Item q of warp gw: sequence index gw + q*W; forward k = seq for seq < n,
// backward k = 2n - 1 - seq after.
struct Item {
  bool valid, fwd;
  int k;
};
__device__ __forceinline__ Item item_of(int gw, int q, int W, int n) {
  const int seq = gw + q * W;
  Item it;
  it.valid = seq < 2 * n;
  it.fwd = seq < n;
  it.k = it.fwd ? seq : 2 * n - 1 - seq;
  return it;
}

template <int KG, int D>
__device__ __forceinline__ void run(const persist::Params &P, unsigned char *smem) {
  static_assert(D >= 2 && D <= 8, "ring depth");
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  const int W = gridDim.x * wpc;
  const int gw = blockIdx.x * wpc + wid;
  const int n = P.n_lvl1, b_s = P.b_s, LC = P.s_LC;
  const unsigned epoch = P.epoch_dev ? *P.epoch_dev : P.epoch;
  const double *src = P.pre_src;
  double *mid = P.y, *dst = P.pre_dst;
  const unsigned SB = (unsigned)slot_bytes(LC);
  unsigned char *wb = smem + (size_t)wid * warp_bytes(LC, D, b_s);
  const unsigned wb_s = s32(wb);   // shared-window address of the warp's ring
  double *ys = (double *)(wb + (size_t)D * SB);
  int *slen = (int *)(wb + (size_t)D * SB + (size_t)b_s * 256);

  // ---- issue side: descriptors (slice offset / length of every step) of
  // the item being issued (A) and the next one (B), lane l holding step l
  int iq = 0, ii = 0, islot = 0;
  int a_off = 0, b_off = 0, a_len = 0, b_len = 0;
  auto load_desc = [&](int q, int &off, int &len) {
    const Item it = item_of(gw, q, W, n);
    off = 0;
    len = 0;
    if (it.valid && lane < b_s) {
      const int l = it.fwd ? lane : b_s - 1 - lane;
      const int sid = it.k * b_s + l;
      off = (int)(it.fwd ? P.Lsp[sid] : P.Usp[sid]);
      len = it.fwd ? P.Lsl[sid] : P.Usl[sid];
    }
  };
  load_desc(0, a_off, a_len);
  load_desc(1, b_off, b_len);
  // stream the static operands of the next step into ring slot islot: the
  // slice's values (16 x len chunks of 16 B), columns (8 x len) and the 32
  // inv_d (16); one commit group per step (empty past the last item)
  auto issue = [&]() {
    const Item it = item_of(gw, iq, W, n);
    if (it.valid) {
      const int off = __shfl_sync(FULL, a_off, ii);
      const int len = __shfl_sync(FULL, a_len, ii);
      const int l = it.fwd ? ii : b_s - 1 - ii;
      const unsigned sl = wb_s + (unsigned)islot * SB;
      const char *gv = (const char *)((it.fwd ? P.Lval : P.Uval) + off);
      const char *gc = (const char *)((it.fwd ? P.Lcol : P.Ucol) + off);
      for (int c = lane; c < 16 * len; c += 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sl + c * 16),
                     "l"(gv + c * 16) : "memory");
      const unsigned slc = sl + (unsigned)LC * 256;
      for (int c = lane; c < 8 * len; c += 32)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(slc + c * 16),
                     "l"(gc + c * 16) : "memory");
      if (lane < 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         sl + (unsigned)LC * 384 + lane * 16),
                     "l"((const char *)(P.inv_d + (it.k * b_s + l) * 32) + lane * 16)
                     : "memory");
      if (lane == 0) slen[islot] = len;
    }
    commit();
    islot = islot + 1 == D ? 0 : islot + 1;
    if (++ii == b_s) {
      ii = 0;
      ++iq;
      a_off = b_off;
      a_len = b_len;
      load_desc(iq + 1, b_off, b_len);
    }
  };
#pragma unroll
  for (int d = 0; d < D; ++d) issue();

  // ---- compute side
  int cslot = 0;
  double xa[KG], xb[KG];
  for (int q = 0;; ++q) {
    const Item it = item_of(gw, q, W, n);
    if (!it.valid) break;
    const bool fwd = it.fwd;
    const int k = it.k;
    const int span = b_s * 32, blk0 = k * span;
    const unsigned uspan = (unsigned)span;
    const double *rhs_v = fwd ? src : mid;
    double *out = fwd ? mid : dst;
    if (fwd)
      persist::wait_flags(P, P.fflag, P.fdep, P.fdep_ptr[k], P.fdep_ptr[k + 1], epoch,
                          nullptr, P.s_ns);
    else
      persist::wait_flags(P, P.bflag, P.bdep, P.bdep_ptr[k], P.bdep_ptr[k + 1], epoch,
                          P.fflag + k, P.s_ns);
    // dynamic operands of walk step i in slot sl: rhs and cross-color gathers
    auto gather = [&](int i, int sl, double *x, double &rhs) {
      const int l = fwd ? i : b_s - 1 - i;
      rhs = __ldcg(rhs_v + blk0 + l * 32 + lane);
      const int *sc = (const int *)(wb + (size_t)sl * SB + (size_t)LC * 256);
      const int len = slen[sl];
#pragma unroll
      for (int u = 0; u < KG; ++u) {
        const int c = u < len ? sc[u * 32 + lane] : blk0;
        x[u] = (unsigned)(c - blk0) >= uspan ? __ldcg(out + c) : 0.0;
      }
    };
    // walk step i from slot sl with its gathers x (x_next: the next step's,
    // issued before this step's chain)
    auto step = [&](int i, int sl, const double *x, double rhs) {
      const int l = fwd ? i : b_s - 1 - i;
      const int row = blk0 + l * 32 + lane;
      const unsigned char *sp = wb + (size_t)sl * SB;
      const double *sv = (const double *)sp;
      const int *sc = (const int *)(sp + (size_t)LC * 256);
      const double idg = ((const double *)(sp + (size_t)LC * 384))[lane];
      const int len = slen[sl];
      double y = rhs;
      auto update = [&](int cc, double vv, double xcross) {
        const unsigned rel = (unsigned)(cc - blk0);
        const bool inblk = rel < uspan;
        unsigned lp = rel >> 5;
        lp = lp < (unsigned)b_s ? lp : 0u;
        const double ysv = ys[(fwd ? (int)lp : b_s - 1 - (int)lp) * 32 + lane];
        const double xin = cc == row ? y : ysv;
        y = __dsub_rn(y, __dmul_rn(vv, inblk ? xin : xcross));
      };
#pragma unroll
      for (int u = 0; u < KG; ++u)
        if (u < len) update(sc[u * 32 + lane], sv[u * 32 + lane], x[u]);
      for (int t = KG; t < len; ++t) {
        const int cc = sc[t * 32 + lane];
        const double xc = (unsigned)(cc - blk0) < uspan ? 0.0 : __ldcg(out + cc);
        update(cc, sv[t * 32 + lane], xc);
      }
      y = __dmul_rn(y, idg);
      ys[i * 32 + lane] = y;
      out[row] = y;
    };
    wait_group<D - 1>();
    __syncwarp();
    double ra = 0.0, rb = 0.0;
    gather(0, cslot, xa, ra);
    // two steps per trip, register buffers used ping-pong (no copies)
    int i = 0;
    for (; i + 1 < b_s; i += 2) {
      const int s1 = cslot + 1 == D ? 0 : cslot + 1;
      wait_group<D - 2>();
      __syncwarp();
      gather(i + 1, s1, xb, rb);
      step(i, cslot, xa, ra);
      __syncwarp();
      issue();
      cslot = s1;
      const int s2 = cslot + 1 == D ? 0 : cslot + 1;
      if (i + 2 < b_s) {
        wait_group<D - 2>();
        __syncwarp();
        gather(i + 2, s2, xa, ra);
      }
      step(i + 1, cslot, xb, rb);
      __syncwarp();
      issue();
      cslot = s2;
    }
    if (i < b_s) {   // odd b_s: the last step's gathers are in xa
      const int s1 = cslot + 1 == D ? 0 : cslot + 1;
      step(i, cslot, xa, ra);
      __syncwarp();
      issue();
      cslot = s1;
    }
    __syncwarp();
    if (lane == 0) persist::st_release((fwd ? P.fflag : P.bflag) + k, epoch);
  }
  wait_group<0>();
}

}  // namespace sweep_stream
