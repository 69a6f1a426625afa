// Dataflow HBMC preconditioner, one software pipeline per warp (sm_100a).
//
// Schedule and arithmetic are those of persist::sweep_pair_dataflow: one warp
// per item (a level-1 block of the forward or of the backward sweep), one
// lane per level-2 block walking its b_s rows, per-block completion flags
// instead of grid barriers; every product __dmul_rn, every update __dsub_rn,
// slots in stored order (K/numba_backend.py:132-171) -- bitwise the
// reference's z.  The lane chain is latency-bound (a few warps per
// scheduler, each a dependent instruction stream), so the kernel is built to
// keep the DRAM stream in flight without registers and the per-step
// instruction stream short:
//   * static operands through a per-warp shared-memory ring.  Every step the
//     warp issues the 16-byte cp.async.cg copies of the step D-1 ahead (its
//     slice's values and encoded columns, its inv_d row and -- forward items
//     -- its rhs row), across item boundaries, and consumes the oldest stage
//     with short shared-memory loads.  The copies hold no registers, so D-1
//     steps of the stream are in flight per warp (register ping-pong buffers
//     hold one), and 16 warps (4 CTAs) run per SM;
//   * pre-classified columns.  The plan keeps an encoded copy of the L / U
//     column arrays (encode_cols): a cross-block column stays the row index
//     (>= 0), an in-block column becomes the shared-memory slot of the walk
//     step that produced it, a padding slot (col == own row, v == 0) points at
//     a shared-memory zero.  One generic load per slot fetches the operand
//     from global (L2-coherent) or shared memory -- no range tests, clamps or
//     selects; the chain is DMUL + DADD per slot.  A padding slot is y - 0*y
//     in the reference: the identity except -0 -> +0 (and inf -> NaN);
//     padding is trailing and that map is idempotent, so it is applied once
//     after the row's slots when the last slot is a padding slot;
//   * slice lengths are warp-uniform: slots are guarded by uniform branches,
//     so a short row executes no dead slots;
//   * the item descriptors (slice offsets / lengths of the b_s steps, the
//     dependency list, the block index) of the NEXT item load while the
//     current one runs and live in lane registers (lane i holds step i's;
//     read with a shuffle): no pointer chase at item start;
//   * L2 eviction policies: the stream's copies are evict-first, the result
//     stores evict-last, so the vectors the gathers read stay in L2;
//   * flags are polled with ld.acquire (no fence that would drain the
//     warp's outstanding copies); a backward item's rhs (the forward result
//     of its own block, valid only after its flag) is prefetched one step
//     ahead in a register instead of through the ring.
// Item order (host-built, item_k): forward blocks k ascending, then the
// backward sweep color by color (descending) but ASCENDING k inside a color --
// blocks of one color are independent, and this way a backward item's own
// forward block finished ~n_lvl1 items ago instead of just now.
// Dependencies are one unified list per item over the flag array
// [forward flags | backward flags], fixed stride, -1 padded: a backward item
// lists its own forward block next to the later-color blocks its U rows read.
// Every dependency precedes its reader in the item order and each warp walks
// its items in order, so the lowest unfinished item can always run.  Backward
// items whose block no later item reads (the first color's) publish no flag
// and skip the release fence.
//
// Requirements (host-checked; otherwise the plan keeps persist.cuh's kernel
// or the per-phase kernels): w == 32, kStages <= b_s <= 32, <= 32
// dependencies per item, in-block entries only inside a lane's own level-2
// block.  Slices of up to 8 slots run the one-chunk-per-step instantiation
// (KC = 2 / 4 / 6 / 8), longer ones (27-point rows) the LONG one: a step is
// several 8-slot ring chunks.  What was tried and rejected on the way
// (profiles/README.md r02q-r03x): register ping-pong buffers, L2 prefetch of
// the stream (bulk and per line) and of the gathered operands, 3-4 CTAs/SM
// with spills, gathers issued one step ahead, lazy flag publication, a
// wavefront item order, dependency lists beyond 32 entries (kNN).

#pragma once

#include "persist.cuh"

namespace flow2 {

constexpr int kInBias = 1 << 30;  // in-block code = walk_step * (ys row stride) - kInBias

// Encoded columns of one factor (warp per slice, lane per row).  fwd: the
// walk step of in-block source row l' is l'; bwd: b_s-1-l'.  stride = doubles
// between consecutive walk steps' results in the kernel's shared memory.
__global__ void encode_cols(const long long *__restrict__ sp, const int *__restrict__ sl,
                            const int *__restrict__ col, int *__restrict__ out,
                            long long n_slices, int b_s, int fwd, int stride, int *bad) {
  const long long sid = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (sid >= n_slices) return;
  const int lane = threadIdx.x & 31;
  const long long k = sid / b_s;
  const long long row = sid * 32 + lane;
  const long long blk0 = k * b_s * 32;
  const long long off = sp[sid];
  const int len = sl[sid];
  for (int t = 0; t < len; ++t) {
    const long long q = off + (long long)t * 32 + lane;
    const long long c = col[q];
    int e;
    if (c == row) {
      e = b_s * stride - kInBias;  // padding: the zero row
    } else if (c >= blk0 && c < blk0 + (long long)b_s * 32) {
      const int ls = (int)((c - blk0) >> 5);
      if (((c - blk0) & 31) != lane) atomicAdd(bad, 1);  // must be the lane's own level-2 block
      e = (fwd ? ls : b_s - 1 - ls) * stride - kInBias;
    } else {
      e = (int)c;
    }
    out[q] = e;
  }
}

// Per item and walk step: {slice offset, slice length} (lane i of the item's
// warp loads entry i); item it < n is forward block item_k[it], else backward.
__global__ void build_item_meta(const long long *__restrict__ Lsp, const int *__restrict__ Lsl,
                                const long long *__restrict__ Usp, const int *__restrict__ Usl,
                                const int *__restrict__ item_k, int2 *__restrict__ im, int n,
                                int b_s) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= 2ll * n * b_s) return;
  const int it = (int)(g / b_s), i = (int)(g % b_s);
  const bool fwd = it < n;
  const long long sid = (long long)item_k[it] * b_s + (fwd ? i : b_s - 1 - i);
  im[g] = make_int2((int)(fwd ? Lsp : Usp)[sid], (fwd ? Lsl : Usl)[sid]);
}

template <int KC>
struct Buf {
  int e[KC];
  double v[KC];
  double rhs, idg;
};

// operand of one slot: generic load (global part L2-coherent), predicated
__device__ __forceinline__ double ld_operand(const char *addr, bool pred) {
  double v;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
      " @q ld.relaxed.gpu.f64 %0, [%1];\n}"
      : "=d"(v) : "l"(addr), "r"((int)pred) : "memory");
  return v;
}

// slots U.. of one row: nested warp-uniform branches, so a row of len slots
// runs len DMUL + DADD pairs and nothing else
template <int U, int KC>
__device__ __forceinline__ void chain(int len, double &y, bool &pad, const Buf<KC> &b,
                                      const double (&x)[KC], int pad_code) {
  if constexpr (U < KC) {
    if (len > U) {
      y = __dsub_rn(y, __dmul_rn(b.v[U], x[U]));
      pad = b.e[U] == pad_code;
      chain<U + 1, KC>(len, y, pad, b, x, pad_code);
    }
  }
}

struct Meta {
  int off, len;  // lane i < b_s: walk step i's slice offset (slots) and length
  int dep;       // lane q: q-th dependency (index into the flag array) or -1
  int k;         // the item's level-1 block; bit 31 set: no later item reads its result
                 // (backward items of the first color): no flag to publish
};

// ---------------------------------------------------------------- kernel
constexpr int kThreads = 128;
constexpr int kStages = 3;  // ring depth (4: fewer warps fit, slower at b_s = 16)

template <int KC>
__host__ __device__ constexpr int ring_stage_bytes() { return KC * 384 + 512; }

// 16-byte async copy with an L2 eviction policy (the operand stream is read
// once: evict-first keeps it from flushing the result vectors the gathers read)
__device__ __forceinline__ void cp_async16(unsigned dst, const void *src, bool pred,
                                           unsigned long long pol) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
      " @q cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %3;\n}" ::"r"(dst),
      "l"(src), "r"((int)pred), "l"(pol)
      : "memory");
}
// the same at a compile-time byte offset from both addresses (one address
// computation per slice instead of one per 512-byte round)
template <int OFF>
__device__ __forceinline__ void cp_async16_at(unsigned dst, const void *src, bool pred,
                                              unsigned long long pol) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n"
      " @q cp.async.cg.shared.global.L2::cache_hint [%0+%4], [%1+%4], 16, %3;\n}" ::"r"(dst),
      "l"(src), "r"((int)pred), "l"(pol), "n"(OFF)
      : "memory");
}
template <int R, int NR>
__device__ __forceinline__ void cp_rounds(unsigned dst, const char *src, int lane, int nchunk,
                                          unsigned long long pol) {
  if constexpr (R < NR) {
    cp_async16_at<R * 512>(dst, src, lane + 32 * R < nchunk, pol);
    cp_rounds<R + 1, NR>(dst, src, lane, nchunk, pol);
  }
}
__device__ __forceinline__ void st_result(double *p, double v, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

template <int KC, bool LONG>
__global__ void __launch_bounds__(kThreads)
    precond_kernel(const __grid_constant__ persist::Params P) {
  extern __shared__ __align__(128) unsigned char rsm[];
  constexpr unsigned full = 0xffffffffu;
  constexpr int D = kStages;
  constexpr int ST = ring_stage_bytes<KC>();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int NW = gridDim.x * (kThreads >> 5);
  const int gw = blockIdx.x * (kThreads >> 5) + wib;
  const int b_s = P.b_s, n = P.n_lvl1, total = 2 * n;
  const unsigned epoch = P.epoch_dev ? *P.epoch_dev : P.epoch;
  const int span = b_s * 32;
  unsigned *flags = P.fflag;
  const double *src = P.pre_src;
  double *mid = P.y, *out = P.pre_dst;
  // per warp: D stages, then ys[b_s + 1][32]
  const int wbytes = D * ST + (b_s + 1) * 256;
  unsigned char *wsm = rsm + (size_t)wib * wbytes;
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(wsm);
  double *ys = (double *)(wsm + D * ST) + lane;
  const int pad_code = b_s * 32 - kInBias;
  const char *ys_base = (const char *)ys + 8ll * kInBias;
  ys[b_s * 32] = 0.0;
  if (gw >= total) return;
  // L2 policies: the operand stream is read once (evict-first), the result
  // vectors are gathered from by later items (evict-last): config 3 519 ->
  // 487 us, config 2 91 -> 86 us, config 5 3823 -> 3746 us
  unsigned long long pol_stream, pol_result;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_result));

  auto load_meta = [&](int it) {
    Meta m;
    int2 ol = make_int2(0, 0);
    if (lane < b_s) ol = __ldg(P.item_meta + (size_t)it * b_s + lane);
    m.off = ol.x;
    m.len = ol.y;
    m.dep = lane < P.dep_stride ? __ldg(P.dep2 + (size_t)it * P.dep_stride + lane) : -1;
    m.k = __ldg(P.item_k + it);
    return m;
  };
  auto wait_deps = [&](const Meta &m) {
    if (m.dep >= 0) {
      const unsigned *f = flags + m.dep;
      if (persist::ld_acquire(f) < epoch) {
        const long long t0 = clock64();
        while (persist::ld_acquire(f) < epoch)
          if (P.watchdog > 0 && clock64() - t0 > P.watchdog) __trap();
      }
    }
    __syncwarp();
  };
  // A ring stage holds one CHUNK: up to KC slots of a step's slice (LONG:
  // slices longer than KC take several chunks; else a step is one chunk)
  // plus, with a step's first chunk, its inv_d row and -- forward -- rhs row.
  auto nchunks = [&](int len) { return LONG ? (len > KC ? (len + KC - 1) / KC : 1) : 1; };
  // copies of chunk c of walk step i of item (fwd, m) into ring stage st
  auto copy_chunk = [&](bool fwd, const Meta &m, int i, int c, int st) {
    const int off = __shfl_sync(full, m.off, i) + (LONG ? c * KC * 32 : 0);
    int len = __shfl_sync(full, m.len, i);
    if (LONG) {
      len -= c * KC;
      len = len > KC ? KC : len;
    }
    const unsigned sb = ring_s + st * ST;
    const char *vp = (const char *)((fwd ? P.Lval : P.Uval) + off);
    const char *cp = (const char *)((fwd ? P.Lce : P.Uce) + off);
    // 16-byte chunk lane + 32 r of the slice's values (16 per slot) and
    // columns (8 per slot)
    cp_rounds<0, (KC * 16 + 31) / 32>(sb + lane * 16, vp + lane * 16, lane, len * 16, pol_stream);
    cp_rounds<0, (KC * 8 + 31) / 32>(sb + KC * 256 + lane * 16, cp + lane * 16, lane, len * 8,
                                     pol_stream);
    if (!LONG || c == 0) {
      // lanes 0-15: inv_d row; lanes 16-31: rhs row (forward: an input);
      // 32-bit row index (n_pad < 2^31)
      const int r0 = (m.k & 0x7fffffff) * span + (fwd ? i : b_s - 1 - i) * 32 + (lane & 15) * 2;
      const double *q = (lane < 16 ? P.inv_d : src) + r0;
      cp_async16(sb + KC * 384 + lane * 16, q, lane < 16 || fwd, pol_stream);
    }
  };

  Meta cur = load_meta(gw), nx;
  nx.off = nx.len = nx.k = 0;
  nx.dep = -1;
  bool fwd = gw < n, fwdn = false, has_n = false;
  // issue cursor: chunk ic of walk step is of the current (inx = false) or
  // the next item; it runs D-1 chunks ahead of the consumer (an item has at
  // least b_s >= D-1 chunks, so it never leaves the next item)
  int is = 0, ic = 0, sti = 0;
  bool inx = false;
  auto issue_next = [&]() {
    const bool valid = is < b_s && (!inx || has_n);
    if (valid) {
      const Meta &m = inx ? nx : cur;
      copy_chunk(inx ? fwdn : fwd, m, is, ic, sti);
      if (LONG) {
        const int len = __shfl_sync(full, m.len, is);
        ic = ic + 1 < nchunks(len) ? ic + 1 : 0;
      }
      if (ic == 0) {
        ++is;
        if (is == b_s && !inx) {
          inx = true;
          is = 0;
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    sti = sti + 1 == D ? 0 : sti + 1;
  };
  // prologue: the first D-1 chunks of the warp's first item
#pragma unroll
  for (int t = 0; t < D - 1; ++t) {
    if constexpr (LONG) {
      issue_next();
    } else {
      copy_chunk(fwd, cur, t, 0, t);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  }
  int st = 0;  // stage of the chunk about to be consumed
  for (int it = gw; it < total; it += NW) {
    const int k = cur.k & 0x7fffffff;
    const int itn = it + NW;
    has_n = itn < total;
    fwdn = itn < n;
    if (has_n) nx = load_meta(itn);
    wait_deps(cur);
    double *dst = fwd ? mid : out;
    double rhs_reg = 0.0;
    if (!fwd) rhs_reg = __ldcg(mid + (size_t)k * span + (b_s - 1) * 32 + lane);
    // one walk step; NEXT: its ring copies belong to the next item (the last
    // D-1 steps of an item, one-chunk steps) -- known at compile time so the
    // common case carries no per-step source selection
    auto run_step = [&](int i, auto next_tag) {
      constexpr bool NEXT = decltype(next_tag)::value;
      const int len = __shfl_sync(full, cur.len, i);
      const int row = k * span + (fwd ? i : b_s - 1 - i) * 32 + lane;
      const int nch = nchunks(len);
      double y = 0.0, idg = 0.0, rhs_next = 0.0;
      bool pad = false;
      for (int c = 0; c < nch; ++c) {
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 2) : "memory");
        __syncwarp();
        if constexpr (LONG) {
          issue_next();  // into the stage consumed one chunk ago
        } else {
          // one chunk per step: stream step i + D - 1 (this item's or the
          // next one's) into the stage consumed last step
          const int t = i + D - 1;
          int sn = st + D - 1;
          sn = sn >= D ? sn - D : sn;
          if constexpr (!NEXT)
            copy_chunk(fwd, cur, t, 0, sn);
          else if (has_n)
            copy_chunk(fwdn, nx, t - b_s, 0, sn);
          asm volatile("cp.async.commit_group;" ::: "memory");
        }
        int clen = len;
        if (LONG) {
          clen -= c * KC;
          clen = clen > KC ? KC : clen;
        }
        const unsigned char *sb = wsm + st * ST;
        const int *se = (const int *)(sb + KC * 256) + lane;
        const double *sv = (const double *)sb + lane;
        Buf<KC> b;
        double x[KC];
#pragma unroll
        for (int u0 = 0; u0 < KC; u0 += 2) {
          if (u0 == 0 || clen > u0) {  // warp-uniform
#pragma unroll
            for (int u = u0; u < u0 + 2 && u < KC; ++u) {
              b.e[u] = se[u * 32];
              const char *base = b.e[u] >= 0 ? (const char *)dst : ys_base;
              x[u] = ld_operand(base + 8ll * b.e[u], u < clen);
            }
          }
        }
        if (!LONG || c == 0) {
          if (!fwd && i + 1 < b_s) rhs_next = __ldcg(mid + row - 32);
        }
#pragma unroll
        for (int u0 = 0; u0 < KC; u0 += 2) {
          if (u0 == 0 || clen > u0) {
#pragma unroll
            for (int u = u0; u < u0 + 2 && u < KC; ++u) b.v[u] = sv[u * 32];
          }
        }
        if (!LONG || c == 0) {
          idg = *((const double *)(sb + KC * 384) + lane);
          y = fwd ? *((const double *)(sb + KC * 384 + 256) + lane) : rhs_reg;
        }
        chain<0, KC>(clen, y, pad, b, x, pad_code);
        st = st + 1 == D ? 0 : st + 1;
      }
      if (pad) y = __dsub_rn(y, __dmul_rn(0.0, y));
      y = __dmul_rn(y, idg);
      ys[i * 32] = y;
      st_result(dst + row, y, pol_result);
      rhs_reg = rhs_next;
    };
    if constexpr (LONG) {
      for (int i = 0; i < b_s; ++i) run_step(i, std::false_type{});
    } else {
      int i = 0;
      for (; i < b_s - (D - 1); ++i) run_step(i, std::false_type{});
      for (; i < b_s; ++i) run_step(i, std::true_type{});
    }
    __syncwarp();
    if (lane == 0 && cur.k >= 0) persist::st_release(flags + (fwd ? k : n + k), epoch);
    // the issue cursor is inside the next item by now: it becomes current
    cur = nx;
    fwd = fwdn;
    inx = false;
    if (!has_n) is = b_s;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

template <int KC>
__host__ inline size_t smem_bytes(int b_s) {
  return (size_t)(kThreads / 32) *
         ((size_t)kStages * ring_stage_bytes<KC>() + (size_t)(b_s + 1) * 256);
}

}  // namespace flow2
