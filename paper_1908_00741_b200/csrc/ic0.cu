// IC(0) factorization on the B200 in the HBMC schedule.
//
// K/numba_backend.py:40-79 (ic0_factor), bitwise: for every row i, for each
// strictly-lower entry (i, j) in ascending j,
//     s = a_ij; s = s - l_ik * l_jk  for k in row i (before j) ∩ row j, ascending
//     l_ij = s * inv_d[j]
// then s = a_ii (1 + shift); s = s - l_ik^2 over the row; pivot s <= 0 is a
// breakdown; d_i = sqrt(s); inv_d_i = 1 / d_i.  Every operation is a
// separately rounded __dmul_rn / __dsub_rn / __dsqrt_rn / __ddiv_rn, so the
// factor is bitwise the reference's.
//
// Dependency structure = the forward sweep's: in HBMC order every
// strictly-lower column of row i is either the same lane of the same level-1
// block at an earlier step, or a row of an earlier color (the structural
// fact of SURVEY §8(a), checked by src/ordering.py:328-346).  So one launch
// per color, thread per (level-1 block, lane) walking its b_s rows in order,
// computes every row after all rows it reads: earlier colors finished in
// earlier launches, earlier steps of the same lane by the same thread.
// The kernel checks that precondition per entry (a violation fails the call
// with TB_EINVAL instead of computing from unfinished rows).
// A non-positive pivot records min(row) with atomicMin; a row's dependents
// all have larger indices, so the minimum is the row the sequential
// reference stops at, and its pivot is exact.

#include <cuda_runtime.h>

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

__global__ void __launch_bounds__(128)
    ic0_phase(const long long *__restrict__ lrp, const int *__restrict__ lci, double *lv,
              const double *__restrict__ adiag, double *d, double *inv_d, int w, int b_s,
              long long k0, long long nthreads, unsigned long long *bad_row, double *pivots,
              unsigned *bad_structure) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nthreads) return;
  const long long k = k0 + g / w;
  const int j = (int)(g % w);
  const long long span = (long long)b_s * w;
  for (int l = 0; l < b_s; ++l) {
    const long long i = (k * b_s + l) * w + j;
    const long long lo = lrp[i], hi = lrp[i + 1];
    for (long long p = lo; p < hi; ++p) {
      const int jc = lci[p];
      // the schedule's precondition: same block => same lane, earlier step;
      // else an earlier color (its level-1 blocks all precede k0)
      const long long kj = jc / span;
      const bool ok = kj == k ? ((jc % w) == j && jc < i) : kj < k0;
      if (!ok) {
        atomicOr(bad_structure, 1u);
        return;
      }
      double s = lv[p];
      long long p1 = lo, p2 = lrp[jc];
      const long long e2 = lrp[jc + 1];
      while (p1 < p && p2 < e2) {
        const int c1 = lci[p1], c2 = lci[p2];
        if (c1 == c2) {
          s = __dsub_rn(s, __dmul_rn(lv[p1], lv[p2]));
          ++p1;
          ++p2;
        } else if (c1 < c2) {
          ++p1;
        } else {
          ++p2;
        }
      }
      lv[p] = __dmul_rn(s, inv_d[jc]);
    }
    double s = adiag[i];
    for (long long p = lo; p < hi; ++p) s = __dsub_rn(s, __dmul_rn(lv[p], lv[p]));
    if (s <= 0.0) {
      const unsigned long long prev = atomicMin(bad_row, (unsigned long long)i);
      pivots[i] = s;
      (void)prev;
    }
    const double di = __dsqrt_rn(s);
    d[i] = di;
    inv_d[i] = __ddiv_rn(1.0, di);
  }
}

}  // namespace

extern "C" int tb_dev_ic0_hbmc(int64_t n, const int64_t *lrp, const int32_t *lci,
                               double *lvals, const double *adiag, double *d, double *inv_d,
                               int64_t w, int64_t b_s, int64_t n_c,
                               const int64_t *color_lvl1_ranges, double *pivot_ws,
                               int64_t *bad_row, double *bad_pivot, void *stream) {
  *bad_row = -1;
  *bad_pivot = 0.0;
  if (n < 0 || w < 1 || b_s < 1 || n_c < 0 || (n_c > 0 && !color_lvl1_ranges))
    return fail(TB_EINVAL, "dev_ic0_hbmc: bad arguments");
  if (n_c > 0 && color_lvl1_ranges[n_c] * b_s * w != n)
    return fail(TB_EINVAL, "dev_ic0_hbmc: color ranges do not cover n");
  if (n > 0x7fffffffLL) return fail(TB_EINVAL, "dev_ic0_hbmc: n exceeds int32 columns");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long *flag = nullptr;   // [0] = min bad row, [1] = structure error
  CU(cudaMallocAsync((void **)&flag, 2 * sizeof(unsigned long long), s));
  CU(cudaMemsetAsync(flag, 0xff, sizeof(unsigned long long), s));
  CU(cudaMemsetAsync(flag + 1, 0, sizeof(unsigned long long), s));
  for (int64_t c = 0; c < n_c; ++c) {
    const long long k0 = color_lvl1_ranges[c], k1 = color_lvl1_ranges[c + 1];
    const long long nt = (k1 - k0) * w;
    if (nt <= 0) continue;
    ic0_phase<<<(unsigned)((nt + 127) / 128), 128, 0, s>>>(
        (const long long *)lrp, lci, lvals, adiag, d, inv_d, (int)w, (int)b_s, k0, nt, flag,
        pivot_ws, (unsigned *)(flag + 1));
    CU(cudaGetLastError());
  }
  unsigned long long hf[2] = {~0ULL, 0};
  CU(cudaMemcpyAsync(hf, flag, sizeof(hf), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  CU(cudaFreeAsync(flag, s));
  if (hf[1])
    return fail(TB_EINVAL, "dev_ic0_hbmc: matrix lacks the HBMC dependency structure "
                "(a strictly-lower entry is neither same-lane-earlier-step nor an earlier color)");
  const unsigned long long h = hf[0];
  if (h != ~0ULL) {
    *bad_row = (int64_t)h;
    CU(cudaMemcpy(bad_pivot, pivot_ws + h, sizeof(double), cudaMemcpyDeviceToHost));
    return fail(TB_EIC_BREAKDOWN, "non-positive pivot %.6g at row %lld", *bad_pivot,
                (long long)h);
  }
  return TB_OK;
}
