// One latent dimension of the fused GNN kernels per translation unit (compiled
// with -DGNN_D=<d>; -DGNN_BIG selects the flat path for oversized subdomains):
// each unit owns its own 64 KB constant bank, and the units compile in parallel.
#include <algorithm>

#include "ddmgnn_internal.h"

#ifndef GNN_D
#error "compile with -DGNN_D=<latent dimension>"
#endif

namespace ddmgnn {
static __constant__ float c_w[kConstFloats];
}

#include "gnn_impl.cuh"

#define DDM_CAT2(a, b) a##b
#define DDM_CAT(a, b) DDM_CAT2(a, b)
#ifdef GNN_BIG
#define DDM_NAME(x) DDM_CAT(DDM_CAT(x, _big_d), GNN_D)
#else
#define DDM_NAME(x) DDM_CAT(DDM_CAT(x, _d), GNN_D)
#endif

namespace ddmgnn {

cudaError_t DDM_NAME(gnn_upload)(const float* dev_bank, cudaStream_t s) {
  return cudaMemcpyToSymbolAsync(c_w, dev_bank, sizeof(float) * kConstFloats, 0,
                                 cudaMemcpyDeviceToDevice, s);
}

#ifndef GNN_BIG

cudaError_t DDM_NAME(gnn_configure)() {
  return cudaFuncSetAttribute(gnn_kernel<GNN_D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kGnnSmemMax);
}

// One CTA per subdomain over n_ctas subdomains (order[a.order_begin ...]); k_max =
// largest subdomain of the launch, smem = dynamic shared memory chosen by the host.
cudaError_t DDM_NAME(gnn_launch)(int n_ctas, int k_max, size_t smem, const GnnArgs& a,
                                 cudaStream_t s) {
  // tensor-core groups are 4 warps (one per TMEM lane quarter): multiples of 128
  constexpr int gran = GNN_TC_Q ? 128 : 32;
  int threads = ((k_max + gran - 1) / gran) * gran;
  constexpr int cap = gnn_cta_threads<GNN_D>();
  if (threads > cap) threads = cap / gran * gran;
  if (threads < 128) threads = 128;
  // small subdomains: two CTAs per SM when their shared memory fits (registers:
  // 2 x 448 threads x 72 fit the 64K file) — each CTA's warps fill the other's
  // barrier bubbles.  DDMGNN_TWO_CTA=0 (read when the context is built) disables.
  constexpr int half = cap / 2 / 32 * 32;
  if (!GNN_TC_Q && a.two_cta && threads > half &&
      2 * (smem + sizeof(GnnShared) + 1024) <= 228u * 1024u)
    threads = half;
  gnn_kernel<GNN_D><<<n_ctas, threads, smem, s>>>(a);
  return cudaGetLastError();
}

#else

cudaError_t DDM_NAME(gnn_configure)() {
  return cudaFuncSetAttribute(gnn_cluster_kernel<GNN_D>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, kGnnSmemMax);
}

namespace {
using QFn = void (*)(GnnArgs);
using UFn = void (*)(GnnArgs, int, int);
template <int L>
constexpr QFn qfn() {
  if constexpr (L < Cfg<GNN_D>::LMAX) return gnn_flat_q<GNN_D, L * Cfg<GNN_D>::STRIDE>;
  else return nullptr;
}
template <int L>
constexpr UFn ufn() {
  if constexpr (L < Cfg<GNN_D>::LMAX) return gnn_flat_u<GNN_D, L * Cfg<GNN_D>::STRIDE>;
  else return nullptr;
}
}  // namespace

// Oversized subdomains order[a.order_begin ...]: the first n_flat = n_subs -
// sum(a.cluster_count) (too large for an 8-CTA cluster) through the flat path —
// restriction (first chunk), then per layer one launch per phase over all
// a.n_bslices slices — then one cluster launch per cluster size 2, 4, 8 over
// a.csubs (shared memory and threads per CTA planned per class by the host).
cudaError_t DDM_NAME(gnn_launch)(int n_subs, int /*k_max*/, size_t /*smem*/, const GnnArgs& a,
                                 cudaStream_t s) {
  static const QFn qk[10] = {qfn<0>(), qfn<1>(), qfn<2>(), qfn<3>(), qfn<4>(),
                             qfn<5>(), qfn<6>(), qfn<7>(), qfn<8>(), qfn<9>()};
  static const UFn uk[10] = {ufn<0>(), ufn<1>(), ufn<2>(), ufn<3>(), ufn<4>(),
                             ufn<5>(), ufn<6>(), ufn<7>(), ufn<8>(), ufn<9>()};
  const int n_cl = a.cluster_count[0] + a.cluster_count[1] + a.cluster_count[2];
  const int n_flat = n_subs - n_cl;
  if (n_flat > 0 && a.n_bslices > 0) {
    if (a.first) gnn_flat_prologue<GNN_D><<<n_flat, kGnnThreads, 0, s>>>(a);
    for (int l = 0; l < a.nl; ++l) {
      const int blocks = (a.n_bslices + kFlatWarps - 1) / kFlatWarps;  // table padded
      qk[l]<<<blocks, 32 * kFlatWarps, 0, s>>>(a);
      uk[l]<<<blocks, 32 * kFlatWarps, 0, s>>>(a, a.layer0 + l, a.last && l == a.nl - 1);
    }
  }
  int off = 0;
  for (int j = 0; j < 3; ++j) {
    const int cnt = a.cluster_count[j];
    if (cnt <= 0) continue;
    const unsigned cs = 2u << j;
    GnnArgs m = a;
    m.csubs = a.csubs + off;
    off += cnt;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cnt * cs);
    cfg.blockDim = dim3(std::min(a.cluster_threads[j], gnn_cta_threads<GNN_D>()));
    cfg.dynamicSmemBytes = a.cluster_smem[j];
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, gnn_cluster_kernel<GNN_D>, m);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

#endif

}  // namespace ddmgnn
