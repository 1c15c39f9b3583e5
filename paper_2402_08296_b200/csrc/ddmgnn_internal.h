// Internal declarations shared by the DDM-GNN B200 library translation units.
//
// Device data layout (all resident in HBM, built once per preconditioner):
//
//   K subdomains, V = sum_i k_i batched subdomain nodes, N global DOFs.
//   sub_ptr[K+1]  int32  batched offset of subdomain i (ascending i)
//   idx[V]        int32  global DOF of every batched node (ascending per subdomain,
//                        the reference's local node order, decomp.py:215)
//   Local graphs in SELL-32 ("sliced ELL", slice = 32 consecutive local nodes =
//   one warp): slice q of subdomain i holds w_q = max degree in the slice; record
//   (e, lane) of the slice lives at edges[slice_off[slice_base[i]+q] + 32*e + lane].
//   A record is float2 {|d|, bits(dst_local)}: the reference's edge_len
//   (dss.py:185, computed in fp64 then rounded to fp32) and the local destination.
//   Records of one node are in ascending dst order, i.e. the reference's
//   lexsorted (src, dst) edge order (dss.py:181).  The relative position
//   edge_vec = coords[dst] - coords[src] (dss.py:184) is folded into the per-node
//   projections, so per node the kernel reads
//   xy[V]         float2 fp32(coords - centre of the node's subdomain)
//   deg[V]        uint16 out-degree of every batched node
//   tptr[N+1], tent[V] (int2: batched position, subdomain) — transpose map used
//                 by the gather-based prolongation, ascending subdomain per DOF
//                 (the reference's gluing order, hybrid.py:133-135)
//   pou[N]        fp64   1/multiplicity  (decomp.py:184-189)
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace ddmgnn {

enum Status : int {
  kOk = 0,
  kValueError = 1,    // Python ValueError
  kRuntimeError = 2,  // Python RuntimeError
  kCudaError = 3,
  kStateError = 4,    // API misuse (missing set_* call)
};

// PCG / apply device status word values
enum DevStatus : int {
  kRunning = 0,
  kConverged = 1,
  kMaxIter = 2,
  kNotSpd = 3,
  kNonFiniteResidual = 4,
  kPrecondError = 5,
  kStagingTimeout = 6,  // ddmgnn_apply_host: an input chunk never arrived (apply word only)
};

#ifndef GNN_THREADS
#define GNN_THREADS 896
#endif
constexpr int kGnnThreads = GNN_THREADS;  // GNN CTA size (28 warps/SM; measured best of 640-1024)
constexpr int kConstFloats = 16384;  // 64 KB constant bank
constexpr int kFlatWarps = 8;        // slices (warps) per CTA of the flat path
#ifndef GNN_EDGE_RELU_MAX
// edge-loop relu as max(x, 0) on the ALU pipe (1) or 2 relu(x) = x + |x| on the FMA
// pipe (0); the bank's message weights carry the matching factor (layout.cpp)
#define GNN_EDGE_RELU_MAX 1
#endif
#ifndef GNN_EDGE_SHIFT
// edge loop as sum_e max(Q_t + |d| WL, -P) + width P (= sum_e relu(P + Q_t + |d| WL)):
// 2 instead of 3 packed FMA-pipe ops per pair and edge (gnn_impl.cuh slice_u)
#define GNN_EDGE_SHIFT 1
#endif
#ifndef GNN_EDGE_PREFETCH
#define GNN_EDGE_PREFETCH 1  // L1 prefetch of a slice's edge records before its P mat-vec
#endif
#ifndef GNN_DATAFLOW
// CTA path: layers as a dataflow over slices (per-slice phase flags in shared
// memory, dependencies within the subdomain's slice reach) instead of two CTA
// barriers per layer (gnn_impl.cuh cta_layer_df)
#define GNN_DATAFLOW 1
#endif
#ifndef GNN_DF_SLEEP
#define GNN_DF_SLEEP 20  // ns between polls of a dataflow wait
#endif
#ifndef GNN_DF_PAIRS
#define GNN_DF_PAIRS 1  // phase-A items are pairs of adjacent slices (shared weight loads)
#endif
constexpr int kDfMaxSlices = 64;  // per-slice flags in GnnShared (k <= 2048)
constexpr int kDfMaxReach = 15;   // 2 R + 2 <= 32 flags polled by one warp
#if GNN_EDGE_SHIFT && !GNN_EDGE_RELU_MAX
#error "GNN_EDGE_SHIFT sums relu(x) (not 2 relu(x)): it needs GNN_EDGE_RELU_MAX=1"
#endif
#ifndef GNN_Q2
#define GNN_Q2 1  // phase A two slices per warp (shared weight loads; 2.4% faster)
#endif
#ifndef GNN_TC_Q
#define GNN_TC_Q 0  // phase-A projection on tcgen05 (3xTF32) instead of FFMA2
#endif
// shared memory reserved at the start of the CTA path's dynamic smem for the
// tensor-core B operand (WQ^T hi/lo, 2 x 32 x 16 fp32)
constexpr int kTcSmemBytes = GNN_TC_Q == 2 ? 14336 : (GNN_TC_Q ? 4096 : 0);
constexpr int kGnnSmemMax = 227 * 1024 - 2048;  // dynamic smem cap (static smem < 2 KB)

struct DeviceLayout {
  int n = 0, K = 0, V = 0, S = 0, k_max = 0;
  long long E = 0, E_pad = 0;
  int *sub_ptr = nullptr, *idx = nullptr, *order = nullptr;
  int *slice_base = nullptr, *slice_off = nullptr;
  int* reach = nullptr;  // per subdomain: max |slice(dst) - slice(src)| over its edges
  uint16_t* deg = nullptr;
  float2* edges = nullptr;
  float2* xy = nullptr;
  int* tptr = nullptr;
  int2* tent = nullptr;
  double* pou = nullptr;
  std::vector<int> h_sub_ptr;  // host copies of the small arrays
  std::vector<int> h_order;    // LPT order (descending k, ascending id)
};

struct HostLayout {
  int n = 0, K = 0, V = 0, S = 0, k_max = 0;
  long long E = 0, E_pad = 0;
  std::vector<int> sub_ptr, idx, order, slice_base, slice_off;
  std::vector<int> reach;  // per subdomain: max |slice(dst) - slice(src)| over its edges
  std::vector<uint16_t> deg;
  std::vector<float> edges;  // 2 floats per record
  std::vector<float> xy;     // 2 floats per batched node
  std::vector<int> tptr;
  std::vector<int> tent;  // 2 ints per entry
  std::vector<double> pou;
};

// layout.cpp
int build_host_layout(int n, const int64_t* indptr, const int32_t* indices, const double* coords,
                      int K, const int64_t* sub_ptr, const int64_t* sub_idx, HostLayout* out,
                      std::string* err);

// model packing (layout.cpp)
struct PackedModel {
  int k_bar = 0, d = 0, lmax = 0, stride = 0, dec_off = 0;
  float alpha = 0.f;
  int h0_finite = 0;        // every weight of layer 1's bank slot is finite (h0 skip allowed)
  std::vector<float> bank;  // n_chunks * 16384 floats: chunk c = layers [c*lmax, ...)
  int n_chunks() const { return lmax ? (k_bar + lmax - 1) / lmax : 0; }
};
int gnn_supported_dim(int d);
int gnn_lmax(int d);
int gnn_stride(int d);
// 1 when the kernels sum relu(x) over edges, 0 when they sum 2 relu(x) (GNN_EDGE_RELU_MAX)
int gnn_edge_relu_plain();
int gnn_smem_node_bytes(int d);
int pack_model(int k_bar, int d, double alpha, const double* params, long long n_params,
               PackedModel* out, std::string* err);

// kernels (gnn.cu)
struct GnnArgs {
  const int* sub_ptr;
  const int* idx;
  const int* order;
  const int* slice_base;
  const int* slice_off;
  const int* reach;  // per subdomain slice reach (dataflow layer schedule; null = barriers)
  const uint16_t* deg;
  const float2* edges;
  const float2* xy;
  const double* pou;
  const double* r;
  double* r0r;
  double* scale;
  double* zloc;
  float* hbuf;  // V * HS  (multi-chunk models)
  float* cbuf;  // V       (multi-chunk models)
  float* qbuf;  // V * QS  (global-memory variant)
  int* bad_layer;
  int* out_bad;
  int* status;       // apply error word (atomicMax kPrecondError)
  const int* skip;   // PCG status word: kernels are no-ops when *skip != 0 (may be null)
  float alpha;
  int layer0;        // 1-based index of the first layer of this chunk
  int nl;            // layers in this chunk
  int first, last;   // chunk flags
  int order_begin;   // CTA b handles subdomain order[order_begin + b]
  int cap0;          // largest subdomain of the shared-memory CTA path (gnn_plan_smem)
  const int2* bslices;  // flat path: (subdomain, slice) of every slice of a big subdomain
  int n_bslices;
  const int* csubs;     // cluster path: subdomains of one cluster-size class
  int two_cta;           // CTA path: allow two CTAs per SM for small subdomains
  int h0_skip;           // first chunk: layer 1 starts from h = 0 and its weights are finite
  int cluster_count[3];  // subdomains per cluster size 2, 4, 8 (csubs laid out in that order)
  int cluster_smem[3];   // dynamic shared memory per CTA of each cluster-size class
  int cluster_threads[3];  // threads per CTA (448 when two CTAs fit an SM, else kGnnThreads)
  // staged input (ddmgnn_apply_host): r arrives in chunks; subdomain i may start once
  // ready[sub_stage[i]] >= epoch (flags written by the copy stream).  null = no wait.
  const unsigned int* ready;
  const int* sub_stage;
  unsigned int epoch;
};
int gnn_smem_max_nodes(int d);
// WQ WP B1 WL WU BP1 WP2 BP2 STRIDE D2P DP DEC_W1 DEC_B1 DEC_W2 DEC_B2 LMAX (gnn_cfg.h)
int gnn_bank_offsets(int d, int* o);
cudaError_t gnn_configure_device();
cudaError_t upload_bank(int d, const float* dev_bank, cudaStream_t s);  // D2D into the constant bank
size_t gnn_plan_smem(int d, int k_max, int* cap0);
cudaError_t launch_gnn(int d, int n_ctas, int n_big, int k_max_small, size_t smem,
                       const GnnArgs& a, cudaStream_t s, cudaStream_t side, cudaEvent_t fork,
                       cudaEvent_t join);

// capi.cu: record a CUDA failure as the thread's last error; returns the status code
int report_cuda(cudaError_t e, const char* what);

// krylov.cu
struct PcgState {
  double rho, pq, alpha, beta, rr, nb, rz, tol;
  int iter, max_iter, status, pad;
  unsigned int tickets[8];
  // flexible CG (opt-in, not in the reference): beta = <r, z - z_old> / rho
  double rzo;    // last <r, z - z_old>
  int flexible;  // 0 = the reference's beta = rho'/rho (sparse.py:124), 1 = Polak-Ribiere
  int pad2;
};
constexpr int kRedThreads = 256;
int reduce_blocks(int n);
cudaError_t launch_coarse_gemv(int K, int ld, const double* inv, const double* x, double* y,
                               const int* skip, cudaStream_t s);
cudaError_t launch_asm_local(int K, int k_max, const int* sub_ptr, const int* idx,
                             const long long* off, const double* ainv, const double* pou,
                             const double* r, double* yloc, double* r0r, double* scale,
                             const int* skip, cudaStream_t s);
cudaError_t launch_prolong(int n, int two_level, const int* tptr, const int2* tent,
                           const double* pou, const double* y, const double* scale,
                           const double* zloc, double* z, const double* r, double* partials,
                           PcgState* st, int mode, const int* skip, cudaStream_t s);
// Fused PCG tail after the local solves: coarse GEMV (two_level bit 0), gluing,
// <r, z>, beta and p = z + beta p in one cooperative launch (krylov.cu).
cudaError_t launch_pcg_glue(int n, int two_level, int K, int ld, const double* inv, const double* r0r,
                            double* y, const int* tptr, const int2* tent, const double* pou,
                            const double* scale, const double* zloc, double* z, const double* r,
                            double* p, double* partials, PcgState* st, cudaStream_t s);
// SELL-32 copy of A (built in set_matrix): slice q = rows 32q..32q+31, entry
// (e, lane) at off[q] + 32 e + lane; padding entries have col = -1, val = 0.
struct SellMatrix {
  int n = 0, slices = 0;
  const int* off = nullptr;    // slices + 1
  const int* col = nullptr;    // padded entries
  const double* val = nullptr;
};
cudaError_t launch_spmv(const SellMatrix& m, const double* x, double* y, cudaStream_t s);
cudaError_t launch_spmv_pq(const SellMatrix& m, const double* p, double* q, double* partials,
                           PcgState* st, cudaStream_t s);
cudaError_t launch_update(int n, double* u, double* r, const double* p, const double* q,
                          double* partials, PcgState* st, double* hist, int identity_precond,
                          cudaStream_t s);
cudaError_t launch_pupdate(int n, double* p, const double* z, PcgState* st, cudaStream_t s);
cudaError_t launch_pcg_init(int n, const double* b, double* r, double* partials, PcgState* st,
                            double* hist, cudaStream_t s);
cudaError_t launch_rz_init(int n, const double* r, const double* z, double* p, double* partials,
                           PcgState* st, cudaStream_t s);
cudaError_t launch_copy(int n, const double* src, double* dst, cudaStream_t s);
// zold (may be null unless st->flexible): previous z for the flexible beta
cudaError_t launch_rz_beta(int n, const double* r, const double* z, const double* zold,
                           double* partials, PcgState* st, cudaStream_t s);
cudaError_t launch_pcg_init_u0(int n, const double* b, const double* au0, double* r,
                               double* partials, PcgState* st, double* hist, cudaStream_t s);

// ic0.cu — IC(0) comparator
struct Ic0Device {
  int n = 0;
  const int *lp = nullptr, *lc = nullptr, *up = nullptr, *uc = nullptr;
  const double *lv = nullptr, *uv = nullptr;
  int *ready_l = nullptr, *ready_u = nullptr, *state = nullptr;
};
int ic0_factor(int n, const int* rp, const int* ci, const double* v, std::vector<int>* lp,
               std::vector<int>* lc, std::vector<double>* lv, std::string* err);
cudaError_t launch_ic0_apply(const Ic0Device& f, const double* r, double* tmp, double* z,
                             const int* skip, cudaStream_t s);

}  // namespace ddmgnn
