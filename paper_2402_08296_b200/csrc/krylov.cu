// Krylov-loop and gluing kernels for sm_100a (all fp64, HBM-bound).
//
// Replaces, per PCG iteration of pkg/src/ddmgnn/sparse.py:76-127:
//   q = A p (:107) + <p, q> (:108) + alpha (:111)          -> spmv_kernel<true> (SELL-32)
//   u += alpha p, r -= alpha q (:112-113) + ||r|| (:114)    -> update_kernel
//   p = z + beta p (:126)                                   -> pupdate_kernel
// and the two-level gluing of hybrid.py:117,133-135:
//   y = (R0 A R0^T)^-1 (R0 r)        -> coarse_gemv_kernel (dense inverse, fp64)
//   z_j = sum_{i ∋ j, asc} pou_j y_i + sum_{i ∋ j, asc} s_i sol_i[j]
//                                    -> prolong_kernel (gather over the transpose map,
//                                       fused with <r, z> for rho, sparse.py:123)
// Elementwise updates use explicit __dmul_rn/__dadd_rn so they round exactly like
// numpy (no FMA contraction); the per-DOF gluing and the SpMV row sums run in the
// reference's sequential order, so given equal inputs they are bit-identical to
// scipy.  Dot products use a deterministic two-stage tree reduction (fixed grid,
// fixed order), which differs from BLAS ddot only by summation order.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "ddmgnn_internal.h"

namespace ddmgnn {

constexpr int kMaxRedBlocks = 148 * 8;

int reduce_blocks(int n) {
  int b = (n + kRedThreads - 1) / kRedThreads;
  if (b > kMaxRedBlocks) b = kMaxRedBlocks;
  return b < 1 ? 1 : b;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum; result valid in thread 0.  blockDim.x must be a multiple of 32.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV]) {
  __shared__ double sh[NV][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int t = 0; t < NV; ++t) v[t] = warp_sum_d(v[t]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int t = 0; t < NV; ++t) sh[t][warp] = v[t];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int t = 0; t < NV; ++t) {
      double x = lane < nw ? sh[t][lane] : 0.0;
      v[t] = warp_sum_d(x);
    }
  }
}

// Deterministic grid reduction: every block deposits its partial; the last block to
// arrive sums all partials in block order.  Returns true in thread 0 of that block,
// with the totals in v.
template <int NV>
__device__ bool grid_sum(double (&v)[NV], double* partials, unsigned int* ticket) {
  __shared__ bool am_last;
  block_sum<NV>(v);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int t = 0; t < NV; ++t) partials[static_cast<size_t>(blockIdx.x) * NV + t] = v[t];
    __threadfence();
    const unsigned int prev = atomicAdd(ticket, 1u);
    am_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) acc[t] = 0.0;
  for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += blockDim.x) {
#pragma unroll
    for (int t = 0; t < NV; ++t) acc[t] += __ldcg(&partials[static_cast<size_t>(b) * NV + t]);
  }
  block_sum<NV>(acc);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int t = 0; t < NV; ++t) v[t] = acc[t];
    *ticket = 0u;
    return true;
  }
  return false;
}

// ------------------------------------------------------------------ SpMV
// SELL-32 SpMV (sliced ELL built once from the CSR in set_matrix): thread per row,
// slice = 32 consecutive rows = one warp, entry (e, lane) of slice q at
// off[q] + 32 e + lane, so every col/val load of the warp is one coalesced
// 128 B / 256 B request.  Padding entries have col = -1.  Each row is summed
// sequentially in ascending column order (scipy csr_matvec order), so y is
// bit-identical to the reference's A @ x.  Loads are issued eight entries ahead
// of the dependent adds (memory-level parallelism for the HBM-bound stream).
constexpr int kSpmvRows = 256;

template <bool PQ>
__global__ void __launch_bounds__(kSpmvRows) spmv_kernel(SellMatrix m, const double* __restrict__ x,
                                                         double* __restrict__ y, double* partials,
                                                         PcgState* st) {
  if (PQ && st->status != kRunning) return;
  double pq = 0.0;
  // grid-stride over rows with a grid of at most 8 blocks per SM: the fused <p, Ap>
  // reduction then has <= 1184 block partials instead of one per 256 rows
  for (int row = blockIdx.x * kSpmvRows + threadIdx.x; row < m.n; row += gridDim.x * kSpmvRows) {
    const int q = row >> 5;
    const int off = __ldg(&m.off[q]);
    const int w = (__ldg(&m.off[q + 1]) - off) >> 5;
    const int* __restrict__ cp = m.col + off + (row & 31);
    const double* __restrict__ vp = m.val + off + (row & 31);
    double acc = 0.0;
    // FEM rows are short (7 entries at config C): issue up to 8 col/val loads, then
    // all their x gathers, then the ordered sum — two dependent memory round trips
    // per 8 entries instead of one per entry.
    for (int e0 = 0; e0 < w; e0 += 8) {
      int c[8];
      double v[8], xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool in = e0 + u < w;
        c[u] = in ? __ldcs(cp + 32 * (e0 + u)) : -1;
        v[u] = in ? __ldcs(vp + 32 * (e0 + u)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = c[u] >= 0 ? __ldg(&x[c[u]]) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (c[u] >= 0) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
    }
    y[row] = acc;
    if (PQ) pq += x[row] * acc;
  }
  if (PQ) {
    double v[1] = {pq};
    if (grid_sum<1>(v, partials, &st->tickets[0])) {
      st->pq = v[0];
      if (v[0] <= 0.0) {  // sparse.py:109-110
        st->status = kNotSpd;
      } else {
        st->alpha = st->rho / v[0];  // sparse.py:111
      }
    }
  }
}

static int spmv_blocks(int n) {
  return std::max(1, std::min((n + kSpmvRows - 1) / kSpmvRows, kMaxRedBlocks));
}

cudaError_t launch_spmv(const SellMatrix& m, const double* x, double* y, cudaStream_t s) {
  if (m.n <= 0) return cudaSuccess;
  spmv_kernel<false><<<spmv_blocks(m.n), kSpmvRows, 0, s>>>(m, x, y, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_spmv_pq(const SellMatrix& m, const double* p, double* q, double* partials,
                           PcgState* st, cudaStream_t s) {
  spmv_kernel<true><<<spmv_blocks(m.n), kSpmvRows, 0, s>>>(m, p, q, partials, st);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ BLAS-1
// Vector kernels stream 16-byte (double2) loads, several per thread in flight,
// when the vectors are 16-byte aligned (the context's own buffers always are).
__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

__global__ void __launch_bounds__(kRedThreads) update_kernel(int n, double* __restrict__ u,
                                                             double* __restrict__ r,
                                                             const double* __restrict__ p,
                                                             const double* __restrict__ q,
                                                             double* partials, PcgState* st,
                                                             double* hist, int identity) {
  if (st->status != kRunning) return;
  const double alpha = st->alpha;
  // plain flexible CG (z = r): beta = <r', r' - r> / rho needs <r', r>
  const bool flex_id = identity && st->flexible;
  double rr = 0.0, rro = 0.0;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  int j_scalar = 0;
  if (aligned16(u) && aligned16(r) && aligned16(p) && aligned16(q)) {
    const int n2 = n >> 1;
    double2* u2 = reinterpret_cast<double2*>(u);
    double2* r2 = reinterpret_cast<double2*>(r);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* q2 = reinterpret_cast<const double2*>(q);
    for (int i = tid; i < n2; i += stride) {
      const double2 uo = u2[i], ro = r2[i], pp = __ldg(p2 + i), qq = __ldg(q2 + i);
      double2 un, rn;
      un.x = __dadd_rn(uo.x, __dmul_rn(alpha, pp.x));  // sparse.py:112
      un.y = __dadd_rn(uo.y, __dmul_rn(alpha, pp.y));
      rn.x = __dsub_rn(ro.x, __dmul_rn(alpha, qq.x));  // sparse.py:113
      rn.y = __dsub_rn(ro.y, __dmul_rn(alpha, qq.y));
      u2[i] = un;
      r2[i] = rn;
      rr += rn.x * rn.x;
      rr += rn.y * rn.y;
      if (flex_id) {
        rro += rn.x * __dsub_rn(rn.x, ro.x);
        rro += rn.y * __dsub_rn(rn.y, ro.y);
      }
    }
    j_scalar = 2 * n2;
  }
  for (int j = j_scalar + tid; j < n; j += stride) {
    u[j] = __dadd_rn(u[j], __dmul_rn(alpha, p[j]));  // sparse.py:112
    const double r_old = r[j];
    const double rj = __dsub_rn(r_old, __dmul_rn(alpha, q[j]));  // sparse.py:113
    r[j] = rj;
    rr += rj * rj;
    if (flex_id) rro += rj * __dsub_rn(rj, r_old);
  }
  double v[2] = {rr, rro};
  if (grid_sum<2>(v, partials, &st->tickets[1])) {
    const double rel = sqrt(v[0]) / st->nb;  // sparse.py:114
    st->rr = v[0];
    if (!isfinite(rel)) {  // sparse.py:115-116
      st->status = kNonFiniteResidual;
      return;
    }
    const int it = st->iter + 1;
    hist[it] = rel;  // sparse.py:117
    st->iter = it;
    if (rel < st->tol) {  // sparse.py:119-121
      st->status = kConverged;
    } else if (it >= st->max_iter) {
      st->status = kMaxIter;
    } else if (identity) {  // plain CG: z = r, rho' = r.r (sparse.py:122-125)
      st->rzo = v[1];
      st->beta = (st->flexible ? v[1] : v[0]) / st->rho;
      st->rho = v[0];
    }
  }
}

cudaError_t launch_update(int n, double* u, double* r, const double* p, const double* q,
                          double* partials, PcgState* st, double* hist, int identity_precond,
                          cudaStream_t s) {
  update_kernel<<<reduce_blocks(n), kRedThreads, 0, s>>>(n, u, r, p, q, partials, st, hist,
                                                         identity_precond);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kRedThreads) pupdate_kernel(int n, double* __restrict__ p,
                                                              const double* __restrict__ z,
                                                              const PcgState* st) {
  if (st->status != kRunning) return;
  const double beta = st->beta;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  int j_scalar = 0;
  if (aligned16(p) && aligned16(z)) {
    const int n2 = n >> 1;
    double2* p2 = reinterpret_cast<double2*>(p);
    const double2* z2 = reinterpret_cast<const double2*>(z);
    for (int i = tid; i < n2; i += stride) {
      const double2 pp = p2[i], zz = __ldg(z2 + i);
      p2[i] = make_double2(__dadd_rn(zz.x, __dmul_rn(beta, pp.x)),  // sparse.py:126
                           __dadd_rn(zz.y, __dmul_rn(beta, pp.y)));
    }
    j_scalar = 2 * n2;
  }
  for (int j = j_scalar + tid; j < n; j += stride)
    p[j] = __dadd_rn(z[j], __dmul_rn(beta, p[j]));  // sparse.py:126
}

cudaError_t launch_pupdate(int n, double* p, const double* z, PcgState* st, cudaStream_t s) {
  pupdate_kernel<<<reduce_blocks(n), kRedThreads, 0, s>>>(n, p, z, st);
  return cudaGetLastError();
}

// r = b - A u0 (Au0 may be null for u0 = 0), ||b||, hist[0] (sparse.py:92-97)
__global__ void __launch_bounds__(kRedThreads) init_kernel(int n, const double* __restrict__ b,
                                                           const double* __restrict__ au0,
                                                           double* __restrict__ r,
                                                           double* partials, PcgState* st,
                                                           double* hist) {
  double bb = 0.0, rr = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double bj = b[j];
    const double rj = au0 ? __dsub_rn(bj, au0[j]) : bj;
    r[j] = rj;
    bb += bj * bj;
    rr += rj * rj;
  }
  double v[2] = {bb, rr};
  if (grid_sum<2>(v, partials, &st->tickets[2])) {
    const double nb = sqrt(v[0]);
    st->nb = nb;
    st->rr = v[1];
    st->iter = 0;
    hist[0] = nb == 0.0 ? 0.0 : sqrt(v[1]) / nb;
  }
}

cudaError_t launch_pcg_init(int n, const double* b, double* r, double* partials, PcgState* st,
                            double* hist, cudaStream_t s) {
  // r may already hold A u0 (then it is read as au0 and overwritten in place)
  init_kernel<<<reduce_blocks(n), kRedThreads, 0, s>>>(n, b, nullptr, r, partials, st, hist);
  return cudaGetLastError();
}

cudaError_t launch_pcg_init_u0(int n, const double* b, const double* au0, double* r,
                               double* partials, PcgState* st, double* hist, cudaStream_t s) {
  init_kernel<<<reduce_blocks(n), kRedThreads, 0, s>>>(n, b, au0, r, partials, st, hist);
  return cudaGetLastError();
}

// p = z, rho = <r, z>  (sparse.py:102-103)
__global__ void __launch_bounds__(kRedThreads) rz_init_kernel(int n, const double* __restrict__ r,
                                                              const double* __restrict__ z,
                                                              double* __restrict__ p,
                                                              double* partials, PcgState* st) {
  double rz = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double zj = z[j];
    p[j] = zj;
    rz += r[j] * zj;
  }
  double v[1] = {rz};
  if (grid_sum<1>(v, partials, &st->tickets[3])) {
    st->rho = v[0];
    st->rz = v[0];
  }
}

cudaError_t launch_rz_init(int n, const double* r, const double* z, double* p, double* partials,
                           PcgState* st, cudaStream_t s) {
  rz_init_kernel<<<reduce_blocks(n), kRedThreads, 0, s>>>(n, r, z, p, partials, st);
  return cudaGetLastError();
}

// rho' = <r, z>, beta = rho'/rho, rho = rho'  (sparse.py:123-125), for host-side
// preconditioner callbacks
// (flexible: beta = <r, z - zold> / rho)
__global__ void __launch_bounds__(kRedThreads) rz_beta_kernel(int n, const double* __restrict__ r,
                                                              const double* __restrict__ z,
                                                              const double* __restrict__ zold,
                                                              double* partials, PcgState* st) {
  if (st->status != kRunning) return;
  const bool flex = st->flexible && zold != nullptr;
  double rz = 0.0, rzo = 0.0;
  // same element-to-thread map and per-thread order as update_kernel's ||r||^2, so
  // that PCG with the identity operator reproduces CG bit for bit (test_sparse.py:60-66)
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  int j_scalar = 0;
  if (aligned16(r) && aligned16(z) && (zold == nullptr || aligned16(zold))) {
    const int n2 = n >> 1;
    const double2* r2 = reinterpret_cast<const double2*>(r);
    const double2* z2 = reinterpret_cast<const double2*>(z);
    const double2* o2 = reinterpret_cast<const double2*>(zold);
    for (int i = tid; i < n2; i += stride) {
      const double2 rr = r2[i], zz = z2[i];
      rz += rr.x * zz.x;
      rz += rr.y * zz.y;
      if (flex) {
        const double2 oo = o2[i];
        rzo += rr.x * __dsub_rn(zz.x, oo.x);
        rzo += rr.y * __dsub_rn(zz.y, oo.y);
      }
    }
    j_scalar = 2 * n2;
  }
  for (int j = j_scalar + tid; j < n; j += stride) {
    const double rj = r[j], zj = z[j];
    rz += rj * zj;
    if (flex) rzo += rj * __dsub_rn(zj, zold[j]);
  }
  double v[2] = {rz, rzo};
  if (grid_sum<2>(v, partials, &st->tickets[5])) {
    st->rz = v[0];
    st->rzo = v[1];
    st->beta = (flex ? v[1] : v[0]) / st->rho;
    st->rho = v[0];
  }
}

cudaError_t launch_rz_beta(int n, const double* r, const double* z, const double* zold,
                           double* partials, PcgState* st, cudaStream_t s) {
  rz_beta_kernel<<<reduce_blocks(n), kRedThreads, 0, s>>>(n, r, z, zold, partials, st);
  return cudaGetLastError();
}

__global__ void copy_kernel(int n, const double* __restrict__ a, double* __restrict__ b) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    b[j] = a[j];
}

cudaError_t launch_copy(int n, const double* src, double* dst, cudaStream_t s) {
  copy_kernel<<<reduce_blocks(n), kRedThreads, 0, s>>>(n, src, dst);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ coarse level
// y = inv(R0 A R0^T) x (fp64, row-major inverse with leading dimension ld), 128
// threads (4 warps) per row and two rows per block so ~K/2 blocks keep the 8 K^2
// byte stream in flight; with an even ld (the context pads its copy) every thread
// issues its 16-byte row loads back to back.  Fixed reduction order.  Replaces
// the dense LU solve of sparse.py:163 (coarse matrix factorised at setup).
constexpr int kGemvRowThreads = 64;   // two warps per row, four rows per block
constexpr int kGemvRows = 256 / kGemvRowThreads;
__global__ void __launch_bounds__(256) coarse_gemv_kernel(int K, int ld,
                                                          const double* __restrict__ inv,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ y,
                                                          const int* skip) {
  if (skip != nullptr && *skip != kRunning) return;
  __shared__ double part[kGemvRows][kGemvRowThreads / 32];
  const int sub = threadIdx.x / kGemvRowThreads;  // which of the block's rows
  const int t = threadIdx.x % kGemvRowThreads;
  const int row = blockIdx.x * kGemvRows + sub;
  double acc = 0.0;
  if (row < K) {
    // thread t takes column pairs (2j, 2j+1), j = t, t + 64, ... in this order
    // whatever the alignment (16-byte loads when possible), so the result does not
    // depend on ld or on where the matrix lives (sharded solve: bit-identical z);
    // eight pairs per thread are in flight before the first FMA
    const double* rp = inv + static_cast<size_t>(row) * ld;
    const int k2 = K >> 1;
    const bool vec = (ld & 1) == 0 && aligned16(inv) && aligned16(x);
    for (int j0 = t; j0 < k2; j0 += 8 * kGemvRowThreads) {
      double2 a[8], b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u * kGemvRowThreads;
        if (j < k2) {
          if (vec) {
            a[u] = __ldcs(reinterpret_cast<const double2*>(rp) + j);
            b[u] = __ldg(reinterpret_cast<const double2*>(x) + j);
          } else {
            a[u] = make_double2(__ldcs(rp + 2 * j), __ldcs(rp + 2 * j + 1));
            b[u] = make_double2(__ldg(x + 2 * j), __ldg(x + 2 * j + 1));
          }
        } else {
          a[u] = b[u] = make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j0 + u * kGemvRowThreads < k2) {
          acc = fma(a[u].x, b[u].x, acc);
          acc = fma(a[u].y, b[u].y, acc);
        }
    }
    if ((K & 1) && t == 0) acc = fma(__ldcs(rp + K - 1), __ldg(x + K - 1), acc);
  }
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) part[sub][t >> 5] = acc;
  __syncthreads();
  if (t == 0 && row < K) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kGemvRowThreads / 32; ++w) s += part[sub][w];
    y[row] = s;
  }
}

cudaError_t launch_coarse_gemv(int K, int ld, const double* inv, const double* x, double* y,
                               const int* skip, cudaStream_t s) {
  coarse_gemv_kernel<<<(K + kGemvRows - 1) / kGemvRows, 256, 0, s>>>(K, ld, inv, x, y, skip);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ exact local solves
// DDM-LU comparator (asm.py:84-113, the reference's build_asm / apply_asm): local
// solves y_i = A_i^-1 r_i with dense inverses factorised once at setup (cuSOLVER),
// CTA per subdomain: r_i staged in shared memory, warp per row of A_i^-1 (fp64,
// coalesced row reads — an 8 sum_i k_i^2 byte HBM stream), (R0 r)_i for the coarse
// right-hand side alongside.
__global__ void __launch_bounds__(256) asm_local_kernel(const int* __restrict__ sub_ptr,
                                                        const int* __restrict__ idx,
                                                        const long long* __restrict__ off,
                                                        const double* __restrict__ ainv,
                                                        const double* __restrict__ pou,
                                                        const double* __restrict__ r,
                                                        double* __restrict__ yloc,
                                                        double* __restrict__ r0r,
                                                        double* __restrict__ scale,
                                                        const int* skip) {
  if (skip != nullptr && *skip != kRunning) return;
  extern __shared__ double rs[];
  __shared__ double part[8];
  const int sub = blockIdx.x;
  const int pos0 = sub_ptr[sub], k = sub_ptr[sub + 1] - pos0;
  double acc = 0.0;
  for (int n = threadIdx.x; n < k; n += blockDim.x) {
    const int g = idx[pos0 + n];
    const double v = r[g];
    rs[n] = v;
    acc = fma(pou[g], v, acc);
  }
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) t += part[w];
    r0r[sub] = t;
    scale[sub] = 1.0;  // every local solve contributes (asm.py:110-111)
  }
  const double* a = ainv + off[sub];
  const int lane = threadIdx.x & 31;
  for (int row = threadIdx.x >> 5; row < k; row += blockDim.x >> 5) {
    const double* ar = a + static_cast<long long>(row) * k;
    double y = 0.0;
    for (int m = lane; m < k; m += 32) y = fma(__ldcs(&ar[m]), rs[m], y);
    y = warp_sum_d(y);
    if (lane == 0) yloc[pos0 + row] = y;
  }
}

cudaError_t launch_asm_local(int K, int k_max, const int* sub_ptr, const int* idx,
                             const long long* off, const double* ainv, const double* pou,
                             const double* r, double* yloc, double* r0r, double* scale,
                             const int* skip, cudaStream_t s) {
  const size_t smem = sizeof(double) * static_cast<size_t>(k_max);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(asm_local_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  asm_local_kernel<<<K, 256, smem, s>>>(sub_ptr, idx, off, ainv, pou, r, yloc, r0r, scale, skip);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ prolongation
// z_j of DOF j (hybrid.py:117,133-135 / asm.py:108-113) over the transpose map.
// two_level bit 0: add the coarse correction; bit 1: ASM order (local terms first).
__device__ __forceinline__ double glue_dof(int j, int two_level, const int* __restrict__ tptr,
                                           const int2* __restrict__ tent,
                                           const double* __restrict__ pou,
                                           const double* __restrict__ y,
                                           const double* __restrict__ scale,
                                           const double* __restrict__ zloc) {
  const int b = tptr[j], e = tptr[j + 1];
  double acc = 0.0;
  if (two_level & 2) {
    // ASM order (asm.py:108-113): local sum first, coarse correction added last
    for (int t = b; t < e; ++t) acc = __dadd_rn(acc, zloc[tent[t].x]);
    if (two_level & 1) {
      const double w = pou[j];
      double c = 0.0;
      for (int t = b; t < e; ++t) c = __dadd_rn(c, __dmul_rn(w, y[tent[t].y]));
      acc = __dadd_rn(acc, c);
    }
  } else {
    if (two_level) {  // z = r0.T @ y  (CSC matvec order: ascending subdomain)
      const double w = pou[j];
      for (int t = b; t < e; ++t) acc = __dadd_rn(acc, __dmul_rn(w, y[tent[t].y]));
    }
    for (int t = b; t < e; ++t) {  // z[idx_i] += s_i * sol_i, ascending i (hybrid.py:134-135)
      const int2 pe = tent[t];
      if (scale[pe.y] != 0.0) acc = __dadd_rn(acc, zloc[pe.x]);
    }
  }
  return acc;
}


// mode 0: plain apply.  mode 1: PCG — also <r, z> -> rho', beta (sparse.py:123-125).
__global__ void __launch_bounds__(kRedThreads) prolong_kernel(
    int n, int two_level, const int* __restrict__ tptr, const int2* __restrict__ tent,
    const double* __restrict__ pou, const double* __restrict__ y,
    const double* __restrict__ scale, const double* __restrict__ zloc, double* z,
    const double* __restrict__ r, double* partials, PcgState* st, int mode,
    const int* skip) {
  if (skip != nullptr && *skip != kRunning) return;
  const bool flex = mode == 1 && st->flexible;
  double rz = 0.0, rzo = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double acc = glue_dof(j, two_level, tptr, tent, pou, y, scale, zloc);
    if (mode == 1) {
      const double rj = r[j];
      rz += rj * acc;
      // flexible CG: z still holds z_old here (z is updated in place)
      if (flex) rzo += rj * __dsub_rn(acc, z[j]);
    }
    z[j] = acc;
  }
  if (mode == 1) {
    double v[2] = {rz, rzo};
    if (grid_sum<2>(v, partials, &st->tickets[4])) {
      st->rz = v[0];
      st->rzo = v[1];
      st->beta = (flex ? v[1] : v[0]) / st->rho;  // sparse.py:124 (or Polak-Ribiere)
      st->rho = v[0];
    }
  }
}

cudaError_t launch_prolong(int n, int two_level, const int* tptr, const int2* tent,
                           const double* pou, const double* y, const double* scale,
                           const double* zloc, double* z, const double* r, double* partials,
                           PcgState* st, int mode, const int* skip, cudaStream_t s) {
  prolong_kernel<<<reduce_blocks(n), kRedThreads, 0, s>>>(n, two_level, tptr, tent, pou, y,
                                                          scale, zloc, z, r, partials, st, mode,
                                                          skip);
  return cudaGetLastError();
}


// ------------------------------------------------------------------ fused PCG tail
// Everything of one PCG iteration after the local solves (sparse.py:122-126 with
// hybrid.py:117,133-135) in ONE cooperative launch, two grid-wide barriers:
//   1. y = inv(R0 A R0^T) (R0 r)   (coarse GEMV, block per row, 16-byte loads)
//   2. z_j = glue (transpose map), <r, z> (+ <r, z - z_old>): block partials
//   3. every block sums the partials in block order (identical bits everywhere),
//      beta = rho'/rho (or Polak-Ribiere), p_j = z_j + beta p_j with z_j kept in
//      registers (up to kGlueRegs DOFs per thread; beyond that z is re-read).
// z is stored only when something reads it later (flexible CG's z_old, or the
// register budget).  Replaces coarse_gemv_kernel + prolong_kernel (mode 1) +
// pupdate_kernel: two launches and the z round trip through HBM.
constexpr int kGlueRegs = 8;

struct GlueArgs {
  int n, two_level, K, ld;
  const int* tptr;
  const int2* tent;
  const double *pou, *inv, *r0r, *scale, *zloc, *r;
  double *y, *z, *p, *partials;
  PcgState* st;
};

__global__ void __launch_bounds__(kRedThreads) pcg_glue_kernel(GlueArgs a) {
  namespace cg = cooperative_groups;
  PcgState* st = a.st;
  if (st->status != kRunning) return;  // same value in every block: no barrier is skipped
  cg::grid_group grid = cg::this_grid();
  const double rho = st->rho;          // read before block 0 replaces it
  const bool flex = st->flexible != 0;
  __shared__ double red[2][kRedThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // 1. coarse GEMV
  if (a.two_level & 1) {
    const int K = a.K;
    for (int row = blockIdx.x; row < K; row += gridDim.x) {
      const double* rp = a.inv + static_cast<size_t>(row) * a.ld;
      double acc = 0.0;
      if ((K & 1) == 0 && (a.ld & 1) == 0) {  // rows 16-byte aligned
        const double2* rp2 = reinterpret_cast<const double2*>(rp);
        const double2* x2 = reinterpret_cast<const double2*>(a.r0r);
        for (int j = threadIdx.x; j < K / 2; j += blockDim.x) {
          const double2 m = __ldcs(rp2 + j), x = __ldg(x2 + j);
          acc = fma(m.x, x.x, acc);
          acc = fma(m.y, x.y, acc);
        }
      } else {
        for (int j = threadIdx.x; j < K; j += blockDim.x) acc = fma(__ldcs(rp + j), __ldg(a.r0r + j), acc);
      }
      acc = warp_sum_d(acc);
      if (lane == 0) red[0][warp] = acc;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (blockDim.x >> 5); ++w) t += red[0][w];
        a.y[row] = t;
      }
      __syncthreads();
    }
    grid.sync();
  }
  // 2. gluing + <r, z>
  const int stride = gridDim.x * blockDim.x;
  const int j0 = blockIdx.x * blockDim.x + threadIdx.x;
  const bool in_regs = (a.n + stride - 1) / stride <= kGlueRegs;
  const bool store_z = flex || !in_regs;
  double zr[kGlueRegs];
  double rz = 0.0, rzo = 0.0;
#pragma unroll
  for (int m = 0; m < kGlueRegs; ++m) zr[m] = 0.0;
  {
    int m = 0;
    for (int j = j0; j < a.n; j += stride, ++m) {
      const double zj = glue_dof(j, a.two_level, a.tptr, a.tent, a.pou, a.y, a.scale, a.zloc);
      const double rj = a.r[j];
      rz += rj * zj;
      if (flex) rzo += rj * __dsub_rn(zj, a.z[j]);  // z still holds z_old
#pragma unroll
      for (int q = 0; q < kGlueRegs; ++q)
        if (q == m) zr[q] = zj;
      if (store_z) a.z[j] = zj;
    }
  }
  rz = warp_sum_d(rz);
  rzo = warp_sum_d(rzo);
  if (lane == 0) {
    red[0][warp] = rz;
    red[1][warp] = rzo;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) {
      t0 += red[0][w];
      t1 += red[1][w];
    }
    a.partials[2 * blockIdx.x] = t0;
    a.partials[2 * blockIdx.x + 1] = t1;
  }
  grid.sync();
  // 3. totals in block order (every block the same), beta, p update
  __shared__ double tot[2];
  if (warp == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) {
      t0 += __ldcg(&a.partials[2 * b]);
      t1 += __ldcg(&a.partials[2 * b + 1]);
    }
    t0 = warp_sum_d(t0);
    t1 = warp_sum_d(t1);
    if (lane == 0) {
      tot[0] = t0;
      tot[1] = t1;
    }
  }
  __syncthreads();
  const double beta = (flex ? tot[1] : tot[0]) / rho;  // sparse.py:124 (or Polak-Ribiere)
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->rz = tot[0];
    st->rzo = tot[1];
    st->beta = beta;
    st->rho = tot[0];  // sparse.py:125
  }
  {
    int m = 0;
    for (int j = j0; j < a.n; j += stride, ++m) {
      double zj = 0.0;
      if (in_regs) {
#pragma unroll
        for (int q = 0; q < kGlueRegs; ++q)
          if (q == m) zj = zr[q];
      } else {
        zj = a.z[j];
      }
      a.p[j] = __dadd_rn(zj, __dmul_rn(beta, a.p[j]));  // sparse.py:126
    }
  }
}

cudaError_t launch_pcg_glue(int n, int two_level, int K, int ld, const double* inv, const double* r0r,
                            double* y, const int* tptr, const int2* tent, const double* pou,
                            const double* scale, const double* zloc, double* z, const double* r,
                            double* p, double* partials, PcgState* st, cudaStream_t s) {
  static int max_blocks = 0;
  if (max_blocks == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_glue_kernel, kRedThreads, 0);
    max_blocks = std::max(1, std::min(kMaxRedBlocks, sms * per_sm));
  }
  GlueArgs a{n, two_level, K, ld, tptr, tent, pou, inv, r0r, scale, zloc, r, y, z, p, partials, st};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::min(max_blocks, std::max(reduce_blocks(n), two_level & 1 ? K : 1)));
  cfg.blockDim = dim3(kRedThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, pcg_glue_kernel, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace ddmgnn
