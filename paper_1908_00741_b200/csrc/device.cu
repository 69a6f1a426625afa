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

#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "tb_internal.h"

using tb::fail;

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

// ------------------------------------------------------------ SpMV
// K/numba_backend.py:26-37: out = 0; out += v * x[col] per slot in stored
// order.  Optional fused epilogue: pap = p . (A p) and alpha = rz / pap.
template <bool DOT>
__global__ void __launch_bounds__(kBlock)
    spmv_sell(long long n, const long long *__restrict__ slice_ptr,
              const int *__restrict__ slice_len, const int *__restrict__ col,
              const double *__restrict__ val, int w,
              const double *__restrict__ x, double *__restrict__ out,
              double *partials, PcgState *st) {
  if (DOT && st->done) return;
  double part = 0.0;
  for (long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (long long)gridDim.x * blockDim.x) {
    const long long s = row / w;
    const int j = (int)(row - s * w);
    long long off = slice_ptr[s] + j;
    const int len = slice_len[s];
    double acc = 0.0;
    for (int t = 0; t < len; ++t, off += w)
      acc = __dadd_rn(acc, __dmul_rn(val[off], x[col[off]]));
    out[row] = acc;
    if (DOT) part += x[row] * acc;
  }
  if (DOT)
    grid_reduce(part, partials, &st->counter[0], [st](double pap) {
      const long long j = st->iter + 1;
      st->pap = pap;
      if (pap <= 0.0) {  // src/solver.py:176-177
        st->status = TB_ECG_BREAKDOWN;
        st->bd_iter = j;
        st->bd_val = pap;
        stop_loop(st);
        return;
      }
      st->alpha = st->rz / pap;
    });
}

// K/numba_backend.py:16-23 spmv_csr (thread per row).
template <bool DOT>
__global__ void __launch_bounds__(kBlock)
    spmv_csr(long long n, const long long *__restrict__ rp,
             const int *__restrict__ col, const double *__restrict__ val,
             const double *__restrict__ x, double *__restrict__ out,
             double *partials, PcgState *st) {
  if (DOT && st->done) return;
  double part = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (long long p = rp[i]; p < rp[i + 1]; ++p)
      acc = __dadd_rn(acc, __dmul_rn(val[p], x[col[p]]));
    out[i] = acc;
    if (DOT) part += x[i] * acc;
  }
  if (DOT)
    grid_reduce(part, partials, &st->counter[0], [st](double pap) {
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
    });
}

// ------------------------------------------------------------ CG vectors
// x = 0; r = b; bnorm = ||b|| (src/solver.py:159-167).
__global__ void __launch_bounds__(kBlock)
    cg_init(long long n, const double *__restrict__ b, double *__restrict__ x,
            double *__restrict__ r, double *partials, PcgState *st,
            double *hist) {
  double part = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    part += bi * bi;
  }
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

// x += alpha p; r -= alpha ap; rel = ||r|| / ||b|| (src/solver.py:178-186).
__global__ void __launch_bounds__(kBlock)
    cg_update_xr(long long n, const double *__restrict__ p,
                 const double *__restrict__ ap, double *__restrict__ x,
                 double *__restrict__ r, double *partials, PcgState *st,
                 double *hist) {
  if (st->done) return;
  const double alpha = st->alpha;
  double part = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(alpha, ap[i]));
    r[i] = ri;
    part += ri * ri;
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

// rz_new = r . z; beta = rz_new / rz; rz = rz_new (src/solver.py:190-192).
// FIRST: the prologue's rz = r . z and p = z.
template <bool FIRST>
__global__ void __launch_bounds__(kBlock)
    cg_rz(long long n, const double *__restrict__ r,
          const double *__restrict__ z, double *__restrict__ p,
          double *partials, PcgState *st) {
  if (st->done) return;
  double part = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double zi = z[i];
    part += r[i] * zi;
    if (FIRST) p[i] = zi;
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
__global__ void __launch_bounds__(kBlock)
    cg_update_p(long long n, const double *__restrict__ z,
                double *__restrict__ p, const PcgState *st) {
  if (st->done) return;
  const double beta = st->beta;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

// ------------------------------------------------------------ helpers
inline unsigned grid_for(long long n, int per_block = kBlock) {
  long long g = (n + per_block - 1) / per_block;
  if (g < 1) g = 1;
  return (unsigned)g;
}

inline unsigned reduce_grid(long long n) {
  // Fixed for a given n: up to 4 CTAs per SM-ish worth of work, capped.
  long long g = (n + kBlock * 4 - 1) / (kBlock * 4);
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
  // task sweeps
  DevCsr Lc, Uc, Ac;
  DevSched fs, bs;
  double *inv_d = nullptr;
  // internal vectors and PCG state
  double *r = nullptr, *y = nullptr, *z = nullptr, *p = nullptr, *ap = nullptr;
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
};

namespace {

// Launch one substitution sweep (all phases) on `s`.  Returns kernel count.
int launch_forward(tb_plan *pl, const double *src, double *dst, cudaStream_t s,
                   const PcgState *st, long long *nl) {
  if (pl->precond_kind == TB_PRECOND_HBMC) {
    for (long long c = 0; c < pl->n_c; ++c) {
      const long long k0 = pl->color_lvl1[c], k1 = pl->color_lvl1[c + 1];
      const long long nt = (k1 - k0) * pl->w;
      if (nt <= 0) continue;
      sell_sweep<true><<<grid_for(nt), kBlock, 0, s>>>(
          pl->L.slice_ptr, pl->L.slice_len, pl->L.col, pl->L.val, pl->inv_d,
          src, dst, (int)pl->w, (int)pl->b_s, k0, nt, st);
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
      sell_sweep<false><<<grid_for(nt), kBlock, 0, s>>>(
          pl->U.slice_ptr, pl->U.slice_len, pl->U.col, pl->U.val, pl->inv_d,
          src, dst, (int)pl->w, (int)pl->b_s, k0, nt, st);
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

int launch_spmv(tb_plan *pl, const double *x, double *out, cudaStream_t s,
                bool dot, long long *nl) {
  const long long n = pl->n;
  if (n <= 0) return TB_OK;
  if (pl->spmv_format == TB_SPMV_NONE)
    return fail(TB_EINVAL, "plan has no matrix A (preconditioner-only plan)");
  if (pl->spmv_format == TB_SPMV_SELL) {
    if (dot)
      spmv_sell<true><<<reduce_grid(n), kBlock, 0, s>>>(
          n, pl->A.slice_ptr, pl->A.slice_len, pl->A.col, pl->A.val,
          (int)pl->A.width, x, out, pl->partials, pl->st);
    else
      spmv_sell<false><<<grid_for(n), kBlock, 0, s>>>(
          n, pl->A.slice_ptr, pl->A.slice_len, pl->A.col, pl->A.val,
          (int)pl->A.width, x, out, nullptr, nullptr);
  } else {
    if (dot)
      spmv_csr<true><<<reduce_grid(n), kBlock, 0, s>>>(
          n, pl->Ac.rp, pl->Ac.col, pl->Ac.val, x, out, pl->partials, pl->st);
    else
      spmv_csr<false><<<grid_for(n), kBlock, 0, s>>>(
          n, pl->Ac.rp, pl->Ac.col, pl->Ac.val, x, out, nullptr, nullptr);
  }
  ++*nl;
  CU(cudaGetLastError());
  return TB_OK;
}

// One CG iteration (src/solver.py:174-193) as a kernel sequence.
int launch_iteration(tb_plan *pl, double *x, cudaStream_t s, long long *nl) {
  const long long n = pl->n;
  const unsigned rg = reduce_grid(n);
  int rc;
  if ((rc = launch_spmv(pl, pl->p, pl->ap, s, true, nl))) return rc;
  cg_update_xr<<<rg, kBlock, 0, s>>>(n, pl->p, pl->ap, x, pl->r, pl->partials,
                                     pl->st, pl->hist);
  ++*nl;
  if ((rc = launch_forward(pl, pl->r, pl->y, s, pl->st, nl))) return rc;
  if ((rc = launch_backward(pl, pl->y, pl->z, s, pl->st, nl))) return rc;
  cg_rz<false><<<rg, kBlock, 0, s>>>(n, pl->r, pl->z, pl->p, pl->partials, pl->st);
  cg_update_p<<<grid_for(n), kBlock, 0, s>>>(n, pl->z, pl->p, pl->st);
  *nl += 2;
  CU(cudaGetLastError());
  return TB_OK;
}

int launch_prologue(tb_plan *pl, const double *b, double *x, cudaStream_t s,
                    long long *nl) {
  const long long n = pl->n;
  const unsigned rg = reduce_grid(n);
  int rc;
  cg_init<<<rg, kBlock, 0, s>>>(n, b, x, pl->r, pl->partials, pl->st, pl->hist);
  ++*nl;
  if ((rc = launch_forward(pl, pl->r, pl->y, s, pl->st, nl))) return rc;
  if ((rc = launch_backward(pl, pl->y, pl->z, s, pl->st, nl))) return rc;
  cg_rz<true><<<rg, kBlock, 0, s>>>(n, pl->r, pl->z, pl->p, pl->partials, pl->st);
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
  CU(cudaStreamBeginCaptureToGraph(pl->stream, g, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  int rc = launch_prologue(pl, b, x, pl->stream, &nl);
  cudaGraph_t captured;
  cudaError_t ce = cudaStreamEndCapture(pl->stream, &captured);
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
  if (rc) return rc;
  CU(ce);
  pl->launches_per_iter = nl;
  CU(cudaGraphInstantiate(&pl->gexec, g, 0));
  pl->g_b = b;
  pl->g_x = x;
  pl->g_hist_cap = pl->hist_cap;
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
    if ((rc = upload_sell(pl->L, d->L_sell))) return bail(rc);
    if ((rc = upload_sell(pl->U, d->U_sell))) return bail(rc);
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
  } else {
    if ((rc = upload_csr(pl->Ac, d->A_csr))) return bail(rc);
  }
  if ((rc = upload(&pl->inv_d, d->inv_d, d->n))) return bail(rc);
  const long long nv = d->n > 0 ? d->n : 1;
  if ((rc = upload<double>(&pl->r, nullptr, nv))) return bail(rc);
  if ((rc = upload<double>(&pl->y, nullptr, nv))) return bail(rc);
  if ((rc = upload<double>(&pl->z, nullptr, nv))) return bail(rc);
  if ((rc = upload<double>(&pl->p, nullptr, nv))) return bail(rc);
  if ((rc = upload<double>(&pl->ap, nullptr, nv))) return bail(rc);
  if ((rc = upload<double>(&pl->partials, nullptr, kMaxPartials))) return bail(rc);
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
  cudaFree(pl->r);
  cudaFree(pl->y);
  cudaFree(pl->z);
  cudaFree(pl->p);
  cudaFree(pl->ap);
  cudaFree(pl->partials);
  cudaFree(pl->st);
  cudaFree(pl->hist);
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
  long long nl = 0;
  int rc = launch_forward(pl, r, pl->y, (cudaStream_t)stream, nullptr, &nl);
  if (rc) return rc;
  return launch_backward(pl, pl->y, z, (cudaStream_t)stream, nullptr, &nl);
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
  (void)check_every;  // the loop is device-resident: no host polling
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
  // reset the device state (keep the loop handle if a graph exists)
  PcgState hs;
  CU(cudaMemcpy(&hs, pl->st, sizeof(PcgState), cudaMemcpyDeviceToHost));
  const cudaGraphConditionalHandle h = hs.loop;
  const int has = hs.has_loop;
  memset(&hs, 0, sizeof(hs));
  hs.tol = tol;
  hs.max_iters = max_iters;
  hs.loop = h;
  hs.has_loop = has;
  CU(cudaMemcpy(pl->st, &hs, sizeof(PcgState), cudaMemcpyHostToDevice));
  if (!pl->gexec || pl->g_b != b || pl->g_x != x || pl->g_hist_cap != pl->hist_cap) {
    int rc = build_graph(pl, b, x);
    if (rc) return rc;
  }
  int rc = sync_in(pl, stream);
  if (rc) return rc;
  CU(cudaGraphLaunch(pl->gexec, pl->stream));
  CU(cudaMemcpyAsync(&hs, pl->st, sizeof(PcgState), cudaMemcpyDeviceToHost, pl->stream));
  CU(cudaStreamSynchronize(pl->stream));
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
