// IC(0) comparator (the reference's ic0 / Ic0Preconditioner, sparse.py:170-227;
// CLI method "ic0", cli.py:65-66) on the GPU.
//
// Factorisation: host port of sparse.py:184-227 (row by row on the lower pattern,
// zero fill, the reference's breakdown errors), done once at setup.  Apply:
// z = L^-T (L^-1 r) with two sync-free triangular-solve kernels: thread per row,
// rows handed out in chunks by an atomic ticket in solve order (so every row a
// thread waits on belongs to a chunk some running block already holds — no
// deadlock), each row spinning on the ready flags of the rows it depends on.
// Flags carry a solve epoch kept on the device, so the kernels are replayable
// inside the PCG's CUDA graph without resets.
#include <cmath>
#include <string>
#include <vector>

#include "ddmgnn_internal.h"

namespace ddmgnn {

int ic0_factor(int n, const int* rp, const int* ci, const double* v, std::vector<int>* lp,
               std::vector<int>* lc, std::vector<double>* lv, std::string* err) {
  lp->assign(n + 1, 0);
  lc->clear();
  lv->clear();
  std::vector<double> row_val(n, 0.0);
  std::vector<char> in_row(n, 0);
  for (int i = 0; i < n; ++i) {
    const int s = rp[i], e = rp[i + 1];
    int m = 0;  // lower-triangle entries of row i (cols <= i, ascending)
    while (s + m < e && ci[s + m] <= i) ++m;
    if (m == 0 || ci[s + m - 1] != i) {
      *err = "IC(0) breakdown: missing diagonal in row " + std::to_string(i);
      return kRuntimeError;
    }
    const int base = static_cast<int>(lc->size());
    for (int t = 0; t < m - 1; ++t) {
      const int j = ci[s + t];
      double acc = v[s + t];
      for (int q = (*lp)[j]; q < (*lp)[j + 1] - 1; ++q) {  // row j without its diagonal
        const int jc = (*lc)[q];
        if (in_row[jc]) acc -= row_val[jc] * (*lv)[q];
      }
      const double lij = acc / (*lv)[(*lp)[j + 1] - 1];
      row_val[j] = lij;
      in_row[j] = 1;
      lc->push_back(j);
      lv->push_back(lij);
    }
    double dot = 0.0;
    for (int t = base; t < static_cast<int>(lv->size()); ++t) dot += (*lv)[t] * (*lv)[t];
    const double diag = v[s + m - 1] - dot;
    for (int t = base; t < static_cast<int>(lc->size()); ++t) in_row[(*lc)[t]] = 0;
    if (!(diag > 0.0)) {
      *err = "IC(0) breakdown: nonpositive pivot at row " + std::to_string(i);
      return kRuntimeError;
    }
    lc->push_back(i);
    lv->push_back(std::sqrt(diag));
    (*lp)[i + 1] = static_cast<int>(lc->size());
  }
  return kOk;
}

namespace {

constexpr int kTriChunk = 128;

// st[0] = epoch, st[1] = lower ticket, st[2] = upper ticket
__global__ void tri_begin_kernel(int* st) {
  st[0] += 1;
  st[1] = 0;
  st[2] = 0;
}

// L y = b, L lower CSR with the diagonal last in each row
__global__ void __launch_bounds__(kTriChunk) tri_lower_kernel(int n, const int* __restrict__ rp,
                                                              const int* __restrict__ ci,
                                                              const double* __restrict__ v,
                                                              const double* __restrict__ b,
                                                              double* y, int* ready, int* st,
                                                              const int* skip) {
  if (skip != nullptr && *skip != kRunning) return;
  __shared__ int chunk;
  if (threadIdx.x == 0) chunk = atomicAdd(&st[1], 1);
  __syncthreads();
  const int epoch = *reinterpret_cast<volatile int*>(&st[0]);
  const int row = chunk * kTriChunk + threadIdx.x;
  if (row >= n) return;
  const int s = rp[row], e = rp[row + 1];
  double acc = b[row];
  for (int t = s; t < e - 1; ++t) {
    const int j = ci[t];
    while (*reinterpret_cast<volatile int*>(&ready[j]) != epoch) {
    }
    acc -= v[t] * *reinterpret_cast<volatile double*>(&y[j]);
  }
  *reinterpret_cast<volatile double*>(&y[row]) = acc / v[e - 1];
  __threadfence();
  *reinterpret_cast<volatile int*>(&ready[row]) = epoch;
}

// U z = y, U = L^T upper CSR with the diagonal first in each row; rows handed out
// from the last one down
__global__ void __launch_bounds__(kTriChunk) tri_upper_kernel(int n, const int* __restrict__ rp,
                                                              const int* __restrict__ ci,
                                                              const double* __restrict__ v,
                                                              const double* __restrict__ b,
                                                              double* z, int* ready, int* st,
                                                              const int* skip) {
  if (skip != nullptr && *skip != kRunning) return;
  __shared__ int chunk;
  if (threadIdx.x == 0) chunk = atomicAdd(&st[2], 1);
  __syncthreads();
  const int epoch = *reinterpret_cast<volatile int*>(&st[0]);
  const int row = n - 1 - (chunk * kTriChunk + threadIdx.x);
  if (row < 0) return;
  const int s = rp[row], e = rp[row + 1];
  double acc = b[row];
  for (int t = e - 1; t > s; --t) {
    const int j = ci[t];
    while (*reinterpret_cast<volatile int*>(&ready[j]) != epoch) {
    }
    acc -= v[t] * *reinterpret_cast<volatile double*>(&z[j]);
  }
  *reinterpret_cast<volatile double*>(&z[row]) = acc / v[s];
  __threadfence();
  *reinterpret_cast<volatile int*>(&ready[row]) = epoch;
}

}  // namespace

cudaError_t launch_ic0_apply(const Ic0Device& f, const double* r, double* tmp, double* z,
                             const int* skip, cudaStream_t s) {
  const int blocks = (f.n + kTriChunk - 1) / kTriChunk;
  tri_begin_kernel<<<1, 1, 0, s>>>(f.state);
  tri_lower_kernel<<<blocks, kTriChunk, 0, s>>>(f.n, f.lp, f.lc, f.lv, r, tmp, f.ready_l, f.state,
                                                 skip);
  tri_upper_kernel<<<blocks, kTriChunk, 0, s>>>(f.n, f.up, f.uc, f.uv, tmp, z, f.ready_u, f.state,
                                                 skip);
  return cudaGetLastError();
}

}  // namespace ddmgnn
