// Dispatch over the compiled latent dimensions of the fused GNN kernel
// (gnn_dim.cu, one object per dimension; kernel body in gnn_impl.cuh).
#include "ddmgnn_internal.h"
#include "gnn_cfg.h"

#ifndef DDM_GNN_DIMS
#define DDM_GNN_DIMS(X) X(3) X(4) X(10)
#endif

namespace ddmgnn {

#define X(DD)                                                                    \
  cudaError_t gnn_configure_d##DD();                                             \
  cudaError_t gnn_upload_d##DD(const float* dev_bank, cudaStream_t s);           \
  cudaError_t gnn_launch_d##DD(bool smem_variant, int n_ctas, int k_max,         \
                               const GnnArgs& a, cudaStream_t s);
DDM_GNN_DIMS(X)
#undef X

int gnn_supported_dim(int d) {
  switch (d) {
#define X(DD) case DD: return 1;
    DDM_GNN_DIMS(X)
#undef X
    default: return 0;
  }
}
int gnn_lmax(int d) {
  switch (d) {
#define X(DD) case DD: return Cfg<DD>::LMAX;
    DDM_GNN_DIMS(X)
#undef X
    default: return 0;
  }
}
int gnn_stride(int d) {
  switch (d) {
#define X(DD) case DD: return Cfg<DD>::STRIDE;
    DDM_GNN_DIMS(X)
#undef X
    default: return 0;
  }
}
int gnn_smem_node_bytes(int d) {
  switch (d) {
#define X(DD) case DD: return Cfg<DD>::SMEM_NODE_BYTES;
    DDM_GNN_DIMS(X)
#undef X
    default: return 0;
  }
}
int gnn_bank_offsets(int d, int* o) {
  switch (d) {
#define X(DD) case DD: cfg_offsets<DD>(o); return 1;
    DDM_GNN_DIMS(X)
#undef X
    default: return 0;
  }
}
int gnn_smem_max_nodes(int d) {
  const int nb = gnn_smem_node_bytes(d);
  return nb ? (227 * 1024 - 1024) / nb : 0;
}

cudaError_t gnn_configure_device() {
#define X(DD)                                   \
  {                                             \
    cudaError_t e = gnn_configure_d##DD();      \
    if (e != cudaSuccess) return e;             \
  }
  DDM_GNN_DIMS(X)
#undef X
  return cudaSuccess;
}

cudaError_t upload_bank(int d, const float* dev_bank, cudaStream_t s) {
  switch (d) {
#define X(DD) case DD: return gnn_upload_d##DD(dev_bank, s);
    DDM_GNN_DIMS(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gnn(int d, bool smem_variant, int n_ctas, int k_max, const GnnArgs& a,
                       cudaStream_t s) {
  if (n_ctas <= 0) return cudaSuccess;
  switch (d) {
#define X(DD) case DD: return gnn_launch_d##DD(smem_variant, n_ctas, k_max, a, s);
    DDM_GNN_DIMS(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ddmgnn
