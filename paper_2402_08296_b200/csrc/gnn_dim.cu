// One latent dimension of the fused GNN kernels per translation unit (compiled
// with -DGNN_D=<d>; -DGNN_BIG selects the oversized-subdomain kernel): each unit
// owns its own 64 KB constant bank, and the units compile in parallel.
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
#define DDM_KERNEL gnn_big_kernel
#define DDM_NAME(x) DDM_CAT(DDM_CAT(x, _big_d), GNN_D)
#else
#define DDM_KERNEL gnn_kernel
#define DDM_NAME(x) DDM_CAT(DDM_CAT(x, _d), GNN_D)
#endif

namespace ddmgnn {

cudaError_t DDM_NAME(gnn_configure)() {
  return cudaFuncSetAttribute(DDM_KERNEL<GNN_D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kGnnSmemMax);
}

cudaError_t DDM_NAME(gnn_upload)(const float* dev_bank, cudaStream_t s) {
  return cudaMemcpyToSymbolAsync(c_w, dev_bank, sizeof(float) * kConstFloats, 0,
                                 cudaMemcpyDeviceToDevice, s);
}

// One launch over n_ctas subdomains (order[a.order_begin ...]); k_max = largest
// subdomain of the launch, smem = dynamic shared memory chosen by the host.
cudaError_t DDM_NAME(gnn_launch)(int n_ctas, int k_max, size_t smem, const GnnArgs& a,
                                 cudaStream_t s) {
#ifdef GNN_BIG
  const int cap = kGnnThreads, npt = 1;
#else
  const int cap = kGnnThreads / kGnnNpt, npt = kGnnNpt;
#endif
  int threads = ((k_max + 32 * npt - 1) / (32 * npt)) * 32;
  if (threads > cap) threads = cap;
  if (threads < 64) threads = 64;
  DDM_KERNEL<GNN_D><<<n_ctas, threads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ddmgnn
