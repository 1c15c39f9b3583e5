// Building blocks of the sharded (one process per GPU) solve, SURVEY.md §8(e).
//
// Rank g owns a spatially coherent group of subdomains and the DOFs whose
// base owner (decomp.py:29-44 `base_owner`) is in that group.  Its local
// context (capi.cu) holds the group's subdomain graphs over the rank's local DOF
// set (owned + ghosts, ascending global order, so every per-subdomain kernel
// sees exactly the single-GPU layout).  Between the stream-ordered calls below
// the host issues the collectives (torch.distributed / NCCL): halo exchange of
// p and r, an all-gather of the per-subdomain (R0 r)_i and s_i, a reverse
// exchange of the individual (subdomain, DOF) prolongation terms, and scalar
// all-reduces for the Krylov dot products.
//
// Vector kernels here are HBM-bound fp64 streams; dot products use a fixed
// two-stage reduction (deterministic for a given n).
#include <cmath>

#include "../../include/ddmgnn_b200.h"
#include "ddmgnn_internal.h"

namespace ddmgnn {

namespace {

constexpr int kT = 256;
constexpr int kMaxBlocks = 148 * 8;

int nblocks(long long n) {
  long long b = (n + kT - 1) / kT;
  if (b > kMaxBlocks) b = kMaxBlocks;
  return b < 1 ? 1 : static_cast<int>(b);
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[kT / 32];
  v = wsum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    t = wsum(t);
  }
  return t;  // valid in thread 0
}

__global__ void gather_kernel(long long n, const double* __restrict__ src,
                              const int* __restrict__ idx, double* __restrict__ dst) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[i] = src[idx[i]];
}

__global__ void scatter_kernel(long long n, const double* __restrict__ src,
                               const int* __restrict__ idx, double* __restrict__ dst) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[idx[i]] = src[i];
}

// partial[b] = sum over the block's grid-stride elements of x*y
__global__ void dot_partial_kernel(long long n, const double* __restrict__ x,
                                   const double* __restrict__ y, double* __restrict__ part) {
  double acc = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    acc += x[i] * y[i];
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// partial[b] = sum over the block's grid-stride elements of x*(y - w)  (flexible CG)
__global__ void dot_diff_partial_kernel(long long n, const double* __restrict__ x,
                                        const double* __restrict__ y,
                                        const double* __restrict__ w, double* __restrict__ part) {
  double acc = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    acc += x[i] * __dsub_rn(y[i], w[i]);
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void sum_partials_kernel(int nb, const double* __restrict__ part,
                                    double* __restrict__ out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += part[i];
  acc = block_sum(acc);
  if (threadIdx.x == 0) out[0] = acc;
}

// u += alpha p; r -= alpha q (numpy rounding, sparse.py:112-113); partial r.r
__global__ void axpy2_kernel(long long n, double alpha, const double* __restrict__ p,
                             const double* __restrict__ q, double* __restrict__ u,
                             double* __restrict__ r, double* __restrict__ part) {
  double acc = 0.0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    u[i] = __dadd_rn(u[i], __dmul_rn(alpha, p[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
    r[i] = ri;
    acc += ri * ri;
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// p = z + beta p (sparse.py:126)
__global__ void xpby_kernel(long long n, const double* __restrict__ z, double beta,
                            double* __restrict__ p) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}

}  // namespace

}  // namespace ddmgnn

using namespace ddmgnn;

static int cuda_status(cudaError_t e) { return report_cuda(e, "sharded vector kernel"); }

extern "C" int ddmgnn_gather(const double* src, const int32_t* idx, int64_t n, double* dst,
                             void* stream) {
  if (n <= 0) return 0;
  gather_kernel<<<nblocks(n), kT, 0, static_cast<cudaStream_t>(stream)>>>(n, src, idx, dst);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_scatter(const double* src, const int32_t* idx, int64_t n, double* dst,
                              void* stream) {
  if (n <= 0) return 0;
  scatter_kernel<<<nblocks(n), kT, 0, static_cast<cudaStream_t>(stream)>>>(n, src, idx, dst);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_dot(int64_t n, const double* x, const double* y, double* work,
                          double* out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = nblocks(n);
  dot_partial_kernel<<<nb, kT, 0, s>>>(n, x, y, work);
  sum_partials_kernel<<<1, kT, 0, s>>>(nb, work, out);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_dot_diff(int64_t n, const double* x, const double* y, const double* w,
                               double* work, double* out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = nblocks(n);
  dot_diff_partial_kernel<<<nb, kT, 0, s>>>(n, x, y, w, work);
  sum_partials_kernel<<<1, kT, 0, s>>>(nb, work, out);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_axpy2(int64_t n, double alpha, const double* p, const double* q,
                            double* u, double* r, double* work, double* rr_out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = nblocks(n);
  axpy2_kernel<<<nb, kT, 0, s>>>(n, alpha, p, q, u, r, work);
  sum_partials_kernel<<<1, kT, 0, s>>>(nb, work, rr_out);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_xpby(int64_t n, const double* z, double beta, double* p, void* stream) {
  if (n <= 0) return 0;
  xpby_kernel<<<nblocks(n), kT, 0, static_cast<cudaStream_t>(stream)>>>(n, z, beta, p);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_dense_gemv(int64_t k, const double* a, const double* x, double* y,
                                 void* stream) {
  if (k <= 0) return 0;
  return cuda_status(launch_coarse_gemv(static_cast<int>(k), a, x, y, nullptr,
                                        static_cast<cudaStream_t>(stream)));
}

extern "C" int ddmgnn_prolong(int64_t n, int two_level, const int32_t* tptr,
                              const int32_t* tent, const double* pou, const double* y,
                              const double* scale, const double* zloc, double* z,
                              void* stream) {
  if (n <= 0) return 0;
  return cuda_status(launch_prolong(static_cast<int>(n), two_level, tptr,
                                    reinterpret_cast<const int2*>(tent), pou, y, scale, zloc, z,
                                    nullptr, nullptr, nullptr, 0, nullptr,
                                    static_cast<cudaStream_t>(stream)));
}

// ---------------------------------------------------------------- device-side scalars
// Distributed PCG with its scalars on the device (no host round trip per dot):
// st[] = {rho, pq, alpha, rr, nb, tol, rz, beta, iter, status, max_iter, rzo}; the
// all-reduces of pq, rr, rz operate on st[1], st[3], st[6] in place, and the
// updates below become no-ops once status != 0 (converged / not SPD / non-finite),
// so the host only polls the status every few iterations.
namespace ddmgnn {
namespace {
enum { kRho, kPq, kAlpha, kRr, kNb, kTol, kRz, kBeta, kIter, kStatus, kMaxIter, kRzo };

__global__ void pcg_scalars_kernel(int op, double* st, double* hist) {
  if (st[kStatus] != 0.0) return;
  if (op == 0) {  // alpha = rho / <p, Ap> (sparse.py:108-111)
    if (st[kPq] <= 0.0) st[kStatus] = 3.0;
    else st[kAlpha] = st[kRho] / st[kPq];
  } else if (op == 1) {  // relative residual, history, stopping test (sparse.py:114-121)
    const double rel = sqrt(st[kRr]) / st[kNb];
    const int it = static_cast<int>(st[kIter]) + 1;
    st[kIter] = it;
    if (!isfinite(rel)) {
      st[kStatus] = 4.0;
      return;
    }
    hist[it] = rel;
    if (rel < st[kTol]) st[kStatus] = 1.0;
    else if (it >= static_cast<int>(st[kMaxIter])) st[kStatus] = 2.0;
  } else if (op == 2) {  // beta = rho' / rho, rho = rho' (sparse.py:123-125)
    st[kBeta] = st[kRz] / st[kRho];
    st[kRho] = st[kRz];
  } else {  // flexible CG: beta = <r, z - z_old> / rho, rho = rho'
    st[kBeta] = st[kRzo] / st[kRho];
    st[kRho] = st[kRz];
  }
}

__global__ void axpy2_dev_kernel(long long n, const double* __restrict__ st,
                                 const double* __restrict__ p, const double* __restrict__ q,
                                 double* __restrict__ u, double* __restrict__ r,
                                 double* __restrict__ part) {
  double acc = 0.0;
  if (st[kStatus] == 0.0) {
    const double alpha = st[kAlpha];
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
      u[i] = __dadd_rn(u[i], __dmul_rn(alpha, p[i]));
      const double ri = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
      r[i] = ri;
      acc += ri * ri;
    }
  }
  acc = block_sum(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void xpby_dev_kernel(long long n, const double* __restrict__ z,
                                const double* __restrict__ st, double* __restrict__ p) {
  if (st[kStatus] != 0.0) return;
  const double beta = st[kBeta];
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, p[i]));
}
}  // namespace
}  // namespace ddmgnn

extern "C" int ddmgnn_pcg_scalars(int op, double* st, double* hist, void* stream) {
  if (op < 0 || op > 3) return kValueError;
  pcg_scalars_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(op, st, hist);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_axpy2_dev(int64_t n, const double* st, const double* p, const double* q,
                                double* u, double* r, double* work, double* rr_out,
                                void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = nblocks(n);
  axpy2_dev_kernel<<<nb, kT, 0, s>>>(n, st, p, q, u, r, work);
  sum_partials_kernel<<<1, kT, 0, s>>>(nb, work, rr_out);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_xpby_dev(int64_t n, const double* z, const double* st, double* p,
                               void* stream) {
  if (n <= 0) return 0;
  xpby_dev_kernel<<<nblocks(n), kT, 0, static_cast<cudaStream_t>(stream)>>>(n, z, st, p);
  return cuda_status(cudaGetLastError());
}
