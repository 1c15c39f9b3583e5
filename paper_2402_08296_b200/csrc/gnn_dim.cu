// One latent dimension of the fused GNN kernel per translation unit (compiled
// with -DGNN_D=<d>): each unit owns its own 64 KB constant bank, and the units
// compile in parallel.
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

namespace ddmgnn {

cudaError_t DDM_CAT(gnn_configure_d, GNN_D)() {
  return cudaFuncSetAttribute(gnn_kernel<GNN_D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kGnnSmemMax);
}

cudaError_t DDM_CAT(gnn_upload_d, GNN_D)(const float* dev_bank, cudaStream_t s) {
  return cudaMemcpyToSymbolAsync(c_w, dev_bank, sizeof(float) * kConstFloats, 0,
                                 cudaMemcpyDeviceToDevice, s);
}

// One launch over n_ctas subdomains; k_max = largest subdomain, smem = dynamic
// shared memory chosen by the host (gnn_plan_smem).
cudaError_t DDM_CAT(gnn_launch_d, GNN_D)(int n_ctas, int k_max, size_t smem, const GnnArgs& a,
                                         cudaStream_t s) {
  int threads = ((k_max + 31) / 32) * 32;
  if (threads > kGnnThreads) threads = kGnnThreads;
  if (threads < 64) threads = 64;
  gnn_kernel<GNN_D><<<n_ctas, threads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace ddmgnn
