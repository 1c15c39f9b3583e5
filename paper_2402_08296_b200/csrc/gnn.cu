// Dispatch over the compiled latent dimensions of the fused GNN kernel
// (gnn_dim.cu, one object per dimension; kernel body in gnn_impl.cuh).
#include "ddmgnn_internal.h"
#include "gnn_cfg.h"

#ifndef DDM_GNN_DIMS
#ifdef GNN_ONE_DIM  // experiment builds: one latent width only (make GNN_DIMS=<d>)
#define DDM_ONE_DIM(X, d) X(d)
#define DDM_GNN_DIMS(X) DDM_ONE_DIM(X, GNN_ONE_DIM)
#else
#define DDM_GNN_DIMS(X) X(3) X(4) X(5) X(10) X(20)
#endif
#endif

namespace ddmgnn {

#define X(DD)                                                                        \
  cudaError_t gnn_configure_d##DD();                                                 \
  cudaError_t gnn_upload_d##DD(const float* dev_bank, cudaStream_t s);               \
  cudaError_t gnn_launch_d##DD(int n_ctas, int k_max, size_t smem, const GnnArgs& a,  \
                               cudaStream_t s);                                      \
  cudaError_t gnn_configure_big_d##DD();                                             \
  cudaError_t gnn_upload_big_d##DD(const float* dev_bank, cudaStream_t s);           \
  cudaError_t gnn_launch_big_d##DD(int n_ctas, int k_max, size_t smem, const GnnArgs& a, \
                                   cudaStream_t s);
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
int gnn_edge_relu_plain() { return GNN_EDGE_RELU_MAX ? 1 : 0; }

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
  return nb ? kGnnSmemMax / nb : 0;
}

cudaError_t gnn_configure_device() {
#define X(DD)                                   \
  {                                             \
    cudaError_t e = gnn_configure_d##DD();      \
    if (e != cudaSuccess) return e;             \
    e = gnn_configure_big_d##DD();              \
    if (e != cudaSuccess) return e;             \
  }
  DDM_GNN_DIMS(X)
#undef X
  return cudaSuccess;
}

cudaError_t upload_bank(int d, const float* dev_bank, cudaStream_t s) {
  switch (d) {
#define X(DD)                                                  \
  case DD: {                                                   \
    cudaError_t e = gnn_upload_d##DD(dev_bank, s);             \
    return e != cudaSuccess ? e : gnn_upload_big_d##DD(dev_bank, s); \
  }
    DDM_GNN_DIMS(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

// Shared-memory plan of the CTA path for subdomains of up to k_max nodes: returns
// the dynamic smem bytes; *cap0 = the largest k whose node state (Q and h rows
// 0..k incl. the dummy rows, c) fits — larger subdomains take the flat path.
size_t gnn_plan_smem(int d, int k_max, int* cap0) {
  const int node0 = gnn_smem_node_bytes(d);  // h + Q + c
  const size_t m0 = static_cast<size_t>(k_max + 1) * node0 + kTcSmemBytes;
  const size_t smem = m0 <= static_cast<size_t>(kGnnSmemMax) ? m0 : kGnnSmemMax;
  *cap0 = node0 ? static_cast<int>((smem - kTcSmemBytes) / node0) - 1 : 0;
  // restriction scratch (k doubles) aliases Q: guaranteed since QS >= 2
  return smem;
}

// Launch the GNN over all subdomains of `order` (LPT, descending size): the first
// n_big (k > cap0) go through the flat node-parallel path on the side stream
// `side`, concurrently with gnn_kernel over the rest on `s` (fork/join by events,
// graph-capturable).
cudaError_t launch_gnn(int d, int n_ctas, int n_big, int k_max_small, size_t smem,
                       const GnnArgs& a, cudaStream_t s, cudaStream_t side, cudaEvent_t fork,
                       cudaEvent_t join) {
  if (n_ctas <= 0) return cudaSuccess;
  cudaError_t e;
  if (n_big > 0) {
    if ((e = cudaEventRecord(fork, s)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(side, fork, 0)) != cudaSuccess) return e;
    switch (d) {
#define X(DD) case DD: e = gnn_launch_big_d##DD(n_big, 0, smem, a, side); break;
      DDM_GNN_DIMS(X)
#undef X
      default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    if ((e = cudaEventRecord(join, side)) != cudaSuccess) return e;
  }
  if (n_ctas > n_big) {
    GnnArgs m = a;
    m.order_begin = a.order_begin + n_big;
    switch (d) {
#define X(DD) case DD: e = gnn_launch_d##DD(n_ctas - n_big, k_max_small, smem, m, s); break;
      DDM_GNN_DIMS(X)
#undef X
      default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
  }
  if (n_big > 0) return cudaStreamWaitEvent(s, join, 0);
  return cudaSuccess;
}

}  // namespace ddmgnn
