// Device kernels of the row-partitioned HBMC ICCG.
//
// Per rank the sweeps and the SpMV are the single-device plan kernels run on
// the local HBMC system (paper_1908_00741_b200/partition.py); this file adds
// the glue the partitioned iteration of src/solver.py:157-193 needs:
//   * tb_dev_gather   pack the owned entries a peer's halo needs into the
//                     contiguous send buffer of one exchange step;
//   * tb_dev_dot      <u, v> over the rank's owned rows into a device scalar
//                     slot (all-reduced across ranks by the caller);
//   * tb_dev_cg_xr    alpha = s[num] / s[den]; x += alpha p; r -= alpha ap;
//                     s[rr] = <r, r> (local part);
//   * tb_dev_cg_p     beta = s[num] / s[den]; p = z + beta p.
// Scalars stay on the device: alpha / beta are formed inside the kernels
// from the all-reduced slots, so the only host read per iteration is the
// residual norm for the convergence test.
//
// Reductions are two-pass with a grid that depends only on n: per-CTA sums
// in a fixed order, then one CTA sums the partials in index order -- a
// rank's partial dot is bitwise reproducible run to run.  All fp64, HBM
// streaming: 16 B/row (dot), 48 B/row (x/r update), 24 B/row (p update).

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

constexpr int kT = 256;
constexpr int kMaxGrid = 1184;   // 8 CTAs x 148 SMs; ws holds this many partials

int grid_of(long long n) {
  long long g = (n + 4LL * kT - 1) / (4LL * kT);
  if (g < 1) g = 1;
  return (int)(g < kMaxGrid ? g : kMaxGrid);
}

__device__ __forceinline__ double cta_sum(double v) {
  __shared__ double sh[kT / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < kT / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

__global__ void __launch_bounds__(kT) gather_kernel(long long n, const int *__restrict__ idx,
                                                    const double *__restrict__ src,
                                                    double *__restrict__ dst) {
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < n;
       i += (long long)gridDim.x * kT)
    dst[i] = src[idx[i]];
}

__global__ void __launch_bounds__(kT) dot_kernel(long long n, const double *__restrict__ u,
                                                 const double *__restrict__ v,
                                                 double *__restrict__ ws) {
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < n;
       i += (long long)gridDim.x * kT)
    acc += u[i] * v[i];
  const double s = cta_sum(acc);
  if (threadIdx.x == 0) ws[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kT) xr_kernel(long long n, const double *__restrict__ scal,
                                                int num, int den, const double *__restrict__ p,
                                                const double *__restrict__ ap,
                                                double *__restrict__ x, double *__restrict__ r,
                                                double *__restrict__ ws) {
  const double alpha = scal[num] / scal[den];
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < n;
       i += (long long)gridDim.x * kT) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(alpha, ap[i]));
    r[i] = ri;
    acc += ri * ri;
  }
  const double s = cta_sum(acc);
  if (threadIdx.x == 0) ws[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kT) p_kernel(long long n, const double *__restrict__ scal,
                                               int num, int den, const double *__restrict__ z,
                                               double *__restrict__ p) {
  const double beta = scal[num] / scal[den];
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < n;
       i += (long long)gridDim.x * kT)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

// second pass: one CTA sums ws[0..m) in index order into scal[slot]
__global__ void __launch_bounds__(kT) finish_kernel(int m, const double *__restrict__ ws,
                                                    double *__restrict__ scal, int slot) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < m; i += kT) acc += ws[i];
  const double s = cta_sum(acc);
  if (threadIdx.x == 0) scal[slot] = s;
}

}  // namespace

extern "C" int tb_dev_gather(int64_t n, const int32_t *idx, const double *src, double *dst,
                             void *stream) {
  if (n < 0) return fail(TB_EINVAL, "dev_gather: n < 0");
  if (n == 0) return TB_OK;
  gather_kernel<<<grid_of(n), kT, 0, (cudaStream_t)stream>>>(n, idx, src, dst);
  CU(cudaGetLastError());
  return TB_OK;
}

extern "C" int tb_dev_dot(int64_t n, const double *u, const double *v, double *scal,
                          int32_t slot, double *ws, void *stream) {
  if (n < 0 || slot < 0) return fail(TB_EINVAL, "dev_dot: bad arguments");
  const int g = grid_of(n);
  dot_kernel<<<g, kT, 0, (cudaStream_t)stream>>>(n, u, v, ws);
  finish_kernel<<<1, kT, 0, (cudaStream_t)stream>>>(g, ws, scal, slot);
  CU(cudaGetLastError());
  return TB_OK;
}

extern "C" int tb_dev_cg_xr(int64_t n, double *scal, int32_t num, int32_t den, const double *p,
                            const double *ap, double *x, double *r, int32_t rr_slot,
                            double *ws, void *stream) {
  if (n < 0 || num < 0 || den < 0 || rr_slot < 0)
    return fail(TB_EINVAL, "dev_cg_xr: bad arguments");
  const int g = grid_of(n);
  xr_kernel<<<g, kT, 0, (cudaStream_t)stream>>>(n, scal, num, den, p, ap, x, r, ws);
  finish_kernel<<<1, kT, 0, (cudaStream_t)stream>>>(g, ws, scal, rr_slot);
  CU(cudaGetLastError());
  return TB_OK;
}

extern "C" int tb_dev_cg_p(int64_t n, const double *scal, int32_t num, int32_t den,
                           const double *z, double *p, void *stream) {
  if (n < 0 || num < 0 || den < 0) return fail(TB_EINVAL, "dev_cg_p: bad arguments");
  if (n == 0) return TB_OK;
  p_kernel<<<grid_of(n), kT, 0, (cudaStream_t)stream>>>(n, scal, num, den, z, p);
  CU(cudaGetLastError());
  return TB_OK;
}
