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
#include <cstdlib>

#include <cstring>

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

// ===================================================================== P2P
// NVLink halo exchange without NCCL (north star: "exchanges
// halo entries per color by NVLink P2P stores").  The sender's push kernel
// gathers its owned entries and STORES them straight into the receiver's
// halo slice through a peer pointer (CUDA IPC mapping of the receiver's
// vector), then the CTA that finishes last publishes the step's epoch in the
// receiver's flag word with a system-scope release.  The receiver runs a
// one-thread wait kernel (system-scope acquire, watchdog) on its stream
// before the next color phase.  Epochs only grow and every exchange step
// writes its own halo slots (steps of one sweep cover different colors; the
// CG all-reduces separate iterations), so one flag per (receiver, sender)
// compared with >= is enough.

namespace {

__global__ void __launch_bounds__(kT) push_kernel(long long n, const int *__restrict__ idx,
                                                  const double *__restrict__ src,
                                                  double *dst_remote, unsigned *flag_remote,
                                                  unsigned epoch, unsigned *done_ctr) {
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < n;
       i += (long long)gridDim.x * kT)
    dst_remote[i] = src[idx[i]];
  // last CTA out publishes the flag after every CTA's stores are visible
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(done_ctr, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    *done_ctr = 0;
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag_remote), "r"(epoch) : "memory");
  }
}

__global__ void wait_kernel(const unsigned *flags, int count, int skip, unsigned epoch,
                            long long watchdog) {
  for (int q = 0; q < count; ++q) {
    if (q == skip) continue;
    const long long t0 = clock64();
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + q) : "memory");
      if ((int)(v - epoch) >= 0) break;
      if (watchdog > 0 && clock64() - t0 > watchdog) __trap();
    }
  }
}

}  // namespace

// p = z + beta p with the SpMV's halo push fused in: rows a peer needs are
// stored into its p vector right after they are formed; the last CTA out
// releases the epoch into every peer's flag for this rank.
__global__ void __launch_bounds__(kT) p_push_kernel(long long n, const double *__restrict__ scal,
                                                    int num, int den,
                                                    const double *__restrict__ z,
                                                    double *__restrict__ p, const tb_push_desc pd) {
  const double beta = scal[num] / scal[den];
  for (long long i = (long long)blockIdx.x * kT + threadIdx.x; i < n;
       i += (long long)gridDim.x * kT) {
    const double pi = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
    p[i] = pi;
    const long long rel = i - pd.row0;
    if (rel >= 0 && rel < pd.nrows)
      for (int q = pd.ptr[rel]; q < pd.ptr[rel + 1]; ++q) pd.peer_dst[pd.peer[q]][pd.off[q]] = pi;
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

extern "C" int tb_dev_cg_p_push(int64_t n, const double *scal, int32_t num, int32_t den,
                                const double *z, double *p, const tb_push_desc *pd,
                                void *stream) {
  if (n < 0 || num < 0 || den < 0 || !pd || !pd->done_ctr || pd->npeers < 0 ||
      pd->npeers > TB_MAX_PEERS)
    return fail(TB_EINVAL, "dev_cg_p_push: bad arguments");
  int g = grid_of(n);
  if (g > 592) g = 592;
  p_push_kernel<<<g, kT, 0, (cudaStream_t)stream>>>(n, scal, num, den, z, p, *pd);
  CU(cudaGetLastError());
  return TB_OK;
}

extern "C" int tb_p2p_alloc(int64_t bytes, void **ptr, void *handle64) {
  *ptr = nullptr;
  if (bytes <= 0) return fail(TB_EINVAL, "p2p_alloc: bytes <= 0");
  CU(cudaMalloc(ptr, (size_t)bytes));
  CU(cudaMemset(*ptr, 0, (size_t)bytes));
  if (handle64) {
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, *ptr));
    memcpy(handle64, &h, sizeof(h) < 64 ? sizeof(h) : 64);
  }
  return TB_OK;
}

extern "C" int tb_p2p_free(void *ptr) {
  if (ptr) CU(cudaFree(ptr));
  return TB_OK;
}

extern "C" int tb_p2p_open(const void *handle64, void **ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  CU(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return TB_OK;
}

extern "C" int tb_p2p_close(void *ptr) {
  if (ptr) CU(cudaIpcCloseMemHandle(ptr));
  return TB_OK;
}

extern "C" int tb_p2p_push(int64_t n, const int32_t *idx, const double *src, double *dst_remote,
                           uint32_t *flag_remote, uint32_t epoch, uint32_t *done_ctr,
                           void *stream) {
  if (n < 0 || !flag_remote || !done_ctr) return fail(TB_EINVAL, "p2p_push: bad arguments");
  int g = grid_of(n);
  if (g > 264) g = 264;
  push_kernel<<<g, kT, 0, (cudaStream_t)stream>>>(n, idx, src, dst_remote, flag_remote, epoch,
                                                  done_ctr);
  CU(cudaGetLastError());
  return TB_OK;
}

extern "C" int tb_p2p_wait(const uint32_t *flags, int32_t count, int32_t skip, uint32_t epoch,
                           void *stream) {
  if (count <= 0) return TB_OK;
  // watchdog as in device.cu: TB_WATCHDOG_MS (default 2000; the peer wait gets
  // twice that), 0 disables the trap
  static const long long wd = [] {
    const char *e = getenv("TB_WATCHDOG_MS");
    return (long long)(e && *e ? atoi(e) : 2000) * 2 * 1900000LL;
  }();
  wait_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(flags, count, skip, epoch, wd);
  CU(cudaGetLastError());
  return TB_OK;
}
