// C ABI (include/ddmgnn_b200.h): context management, the preconditioner apply
// pipeline and the device-resident PCG driver.
//
// Apply pipeline (hybrid.py:112-136), all stream-ordered on the device:
//   for each constant-bank chunk c of ceil(k_bar / lmax):
//       D2D copy of the chunk's fp32 weights into the __constant__ bank
//       gnn_kernel<d, global-scratch variant>  (subdomains too large for SMEM)
//       gnn_kernel<d, SMEM variant>            (the rest; LPT order)
//   coarse_gemv_kernel (two-level only)
//   prolong_kernel
// PCG (sparse.py:76-127): one iteration = spmv_pq, update, [apply], pupdate,
// captured once into a CUDA graph and replayed in chunks; every kernel becomes a
// no-op once the device status word leaves "running", and the host polls the
// status once per chunk.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ddmgnn_b200.h"
#include "ddmgnn_internal.h"

using namespace ddmgnn;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

namespace ddmgnn {
int report_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return kOk;
  return fail(kCudaError, std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")");
}
}  // namespace ddmgnn

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail(kCudaError, std::string("CUDA error: ") + cudaGetErrorString(_e) + " (" + \
                                  #expr + ")");                                            \
  } while (0)

template <typename T>
static cudaError_t dalloc(T** p, size_t count) {
  if (*p) {
    cudaFree(*p);
    *p = nullptr;
  }
  if (count == 0) return cudaSuccess;
  return cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * count);
}
template <typename T>
static void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

template <typename T>
static cudaError_t upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = dalloc(dst, std::max<size_t>(v.size(), 1));
  if (e != cudaSuccess) return e;
  if (v.empty()) return cudaSuccess;
  return cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
}

struct ddmgnn_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // big-subdomain GNN kernel (forked from the apply stream)
  // staged input of ddmgnn_apply_host: r copied in kStages chunks on `copy`, each
  // followed by a stream write of its ready flag; the GNN CTAs (subdomains ordered by
  // the last chunk they read) start as soon as their chunk has landed
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_copied = nullptr;
  unsigned int* d_ready = nullptr;  // kStages flags
  int* d_sub_stage = nullptr;       // per subdomain: index of the last chunk it reads
  int* d_order_staged = nullptr;    // big subdomains first (as order), then by stage, LPT
  int staged_ok = 0;                // no flat-path subdomains and stream memory ops work
  int stage_now = 0;                // set while apply_host enqueues a staged apply
  unsigned int stage_epoch = 0;
  long long stage_chunk = 0;        // doubles per chunk (multiple of 16: 128-byte lines)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // matrix
  int n = 0;
  long long nnz = 0;
  int *d_rowptr = nullptr, *d_col = nullptr;
  double* d_val = nullptr;
  int *d_sell_off = nullptr, *d_sell_col = nullptr;  // SELL-32 copy for the SpMV
  double* d_sell_val = nullptr;
  SellMatrix sell;
  // inputs kept on the host until build
  std::vector<double> coords;
  std::vector<int64_t> sub_ptr, sub_idx;
  int K = 0;
  long long batch_cap = 100000;
  // device layout
  bool built = false;
  DeviceLayout lay;
  // model
  bool have_model = false;
  PackedModel model;
  float* d_bank = nullptr;
  int n_big = 0;          // subdomains whose node state does not fit shared memory
  size_t gnn_smem = 0;
  int cap0 = 0;
  // coarse
  int coarse_k = 0;
  double* d_cinv = nullptr;
  int coarse_ld = 0;         // leading dimension of d_cinv (K rounded up to even)
  // apply scratch
  double *d_r0r = nullptr, *d_scale = nullptr, *d_zloc = nullptr, *d_y = nullptr;
  float *d_hbuf = nullptr, *d_cbuf = nullptr, *d_qbuf = nullptr;
  int2* d_bslices = nullptr;  // flat path: (subdomain, slice) of the oversized subdomains
  int n_bslices = 0;
  int* d_csubs = nullptr;     // cluster path: subdomains by cluster size 2, 4, 8
  int cluster_count[3] = {0, 0, 0};
  int cluster_smem[3] = {0, 0, 0}, cluster_threads[3] = {0, 0, 0};
  int two_cta = 1;            // CTA path: two CTAs per SM when they fit (DDMGNN_TWO_CTA)
  int fused_tail = 0;         // PCG: one cooperative launch after the local solves (DDMGNN_FUSED_TAIL=1;
                              // measured slower: 45 us vs 41 us for the three launches it replaces)
  int h0_skip = 1;            // GNN layer 1 without its h rows (h = 0; DDMGNN_H0_SKIP)
  int *d_bad = nullptr, *d_outbad = nullptr, *d_status = nullptr;
  double *d_rin = nullptr, *d_zout = nullptr;  // host-pointer apply staging
  // pcg
  double *d_b = nullptr, *d_u = nullptr, *d_r = nullptr, *d_p = nullptr, *d_q = nullptr,
         *d_z = nullptr, *d_partials = nullptr, *d_hist = nullptr;
  int hist_cap = 0;
  PcgState* d_st = nullptr;
  PcgState* h_st = nullptr;  // pinned
  double *h_pin_a = nullptr, *h_pin_b = nullptr;  // pinned staging (n doubles each)
  cudaGraphExec_t graph_exec[12] = {};  // [level + 6 * flexible]
  int pcg_flex = 0;            // flexible CG in the PCG being enqueued / captured
  double* d_zold = nullptr;    // flexible CG: previous z (IC(0) / host-callback paths)
  // DDM-LU comparator: dense local inverses (row-major, offsets in doubles)
  double* d_ainv = nullptr;
  long long* d_ainv_off = nullptr;
  bool have_asm = false;
  // IC(0) comparator: L (lower, diag last) and U = L^T (upper, diag first) in CSR
  int *d_ic_lp = nullptr, *d_ic_lc = nullptr, *d_ic_up = nullptr, *d_ic_uc = nullptr;
  double *d_ic_lv = nullptr, *d_ic_uv = nullptr, *d_ic_tmp = nullptr;
  int *d_ic_ready = nullptr, *d_ic_state = nullptr;
  Ic0Device ic0;
  bool have_ic0 = false;
};

extern "C" const char* ddmgnn_last_error(void) { return g_err.c_str(); }
extern "C" int ddmgnn_version(void) { return 1; }

extern "C" int ddmgnn_create(int device, ddmgnn_ctx** out) {
  if (!out) return fail(kValueError, "null output pointer");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(kCudaError, std::string("no CUDA device available: ") + cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(kValueError, "device ordinal out of range");
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(kCudaError, "ddmgnn_b200 is built for sm_100a; device " + std::string(prop.name) +
                                " has compute capability " + std::to_string(prop.major) + "." +
                                std::to_string(prop.minor));
  CUDA_TRY(gnn_configure_device());
  auto* c = new ddmgnn_ctx();
  c->device = device;
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(kCudaError, cudaGetErrorString(e));
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_copied, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete c;
    return fail(kCudaError, cudaGetErrorString(e));
  }
  e = cudaMallocHost(reinterpret_cast<void**>(&c->h_st), sizeof(PcgState));
  if (e != cudaSuccess) {
    cudaStreamDestroy(c->stream);
    delete c;
    return fail(kCudaError, cudaGetErrorString(e));
  }
  *out = c;
  return kOk;
}

static void free_graphs(ddmgnn_ctx* c) {
  for (auto& g : c->graph_exec) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
}

static void free_layout(ddmgnn_ctx* c) {
  DeviceLayout& L = c->lay;
  dfree(L.sub_ptr); dfree(L.idx); dfree(L.order); dfree(L.slice_base); dfree(L.slice_off);
  dfree(L.reach); dfree(L.deg); dfree(L.edges); dfree(L.xy); dfree(L.tptr); dfree(L.tent); dfree(L.pou);
  dfree(c->d_r0r); dfree(c->d_scale); dfree(c->d_zloc); dfree(c->d_y);
  dfree(c->d_bad); dfree(c->d_outbad);
  dfree(c->d_hbuf); dfree(c->d_cbuf); dfree(c->d_qbuf); dfree(c->d_bslices); dfree(c->d_csubs);
  dfree(c->d_sub_stage); dfree(c->d_order_staged);
  c->staged_ok = 0;
  dfree(c->d_ainv); dfree(c->d_ainv_off);
  c->have_asm = false;
  c->n_bslices = 0;
  c->built = false;
  free_graphs(c);
}

extern "C" void ddmgnn_destroy(ddmgnn_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  free_layout(c);
  dfree(c->d_rowptr); dfree(c->d_col); dfree(c->d_val);
  dfree(c->d_ic_lp); dfree(c->d_ic_lc); dfree(c->d_ic_up); dfree(c->d_ic_uc);
  dfree(c->d_ic_lv); dfree(c->d_ic_uv); dfree(c->d_ic_tmp); dfree(c->d_ic_ready);
  dfree(c->d_ic_state);
  dfree(c->d_sell_off); dfree(c->d_sell_col); dfree(c->d_sell_val);
  dfree(c->d_bank); dfree(c->d_cinv); dfree(c->d_status);
  dfree(c->d_rin); dfree(c->d_zout); dfree(c->d_ready);
  dfree(c->d_b); dfree(c->d_u); dfree(c->d_r); dfree(c->d_p); dfree(c->d_q); dfree(c->d_z);
  dfree(c->d_partials); dfree(c->d_hist); dfree(c->d_st); dfree(c->d_zold);
  if (c->h_st) cudaFreeHost(c->h_st);
  if (c->h_pin_a) cudaFreeHost(c->h_pin_a);
  if (c->h_pin_b) cudaFreeHost(c->h_pin_b);
  cudaStreamDestroy(c->stream);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->copy) cudaStreamDestroy(c->copy);
  if (c->ev_copied) cudaEventDestroy(c->ev_copied);
  delete c;
}

extern "C" void* ddmgnn_stream(ddmgnn_ctx* c) { return c ? c->stream : nullptr; }

static cudaStream_t pick(ddmgnn_ctx* c, void* s) {
  return s ? reinterpret_cast<cudaStream_t>(s) : c->stream;
}

extern "C" int ddmgnn_set_matrix(ddmgnn_ctx* c, int64_t n, int64_t nnz, const int64_t* indptr,
                                 const int32_t* indices, const double* data) {
  if (!c) return fail(kValueError, "null context");
  if (n <= 0 || n >= (1ll << 31) || nnz < 0 || nnz >= (1ll << 31))
    return fail(kValueError, "matrix dimensions out of range");
  if (indptr[0] != 0 || indptr[n] != nnz) return fail(kValueError, "malformed indptr");
  for (int64_t i = 0; i < n; ++i) {
    if (indptr[i + 1] < indptr[i]) return fail(kValueError, "indptr not nondecreasing");
    for (int64_t t = indptr[i]; t < indptr[i + 1]; ++t) {
      if (indices[t] < 0 || indices[t] >= n || (t > indptr[i] && indices[t] <= indices[t - 1]))
        return fail(kValueError,
                    "row " + std::to_string(i) + ": columns not strictly increasing in range");
    }
  }
  CUDA_TRY(cudaSetDevice(c->device));
  if (c->n != n) free_layout(c);
  c->n = static_cast<int>(n);
  c->nnz = nnz;
  std::vector<int> rp(n + 1);
  for (int64_t i = 0; i <= n; ++i) rp[i] = static_cast<int>(indptr[i]);
  CUDA_TRY(dalloc(&c->d_rowptr, n + 1));
  CUDA_TRY(dalloc(&c->d_col, std::max<int64_t>(nnz, 1)));
  CUDA_TRY(dalloc(&c->d_val, std::max<int64_t>(nnz, 1)));
  CUDA_TRY(cudaMemcpy(c->d_rowptr, rp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
  if (nnz) {
    CUDA_TRY(cudaMemcpy(c->d_col, indices, sizeof(int) * nnz, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c->d_val, data, sizeof(double) * nnz, cudaMemcpyHostToDevice));
  }
  {  // SELL-32 copy (slice = 32 rows, width = longest row of the slice)
    const int slices = static_cast<int>((n + 31) / 32);
    std::vector<int> off(slices + 1, 0);
    for (int q = 0; q < slices; ++q) {
      int64_t w = 0;
      for (int64_t i = 32ll * q; i < std::min<int64_t>(n, 32ll * q + 32); ++i)
        w = std::max<int64_t>(w, indptr[i + 1] - indptr[i]);
      if (off[q] + 32 * w >= (1ll << 31)) return fail(kValueError, "matrix too large for SELL-32");
      off[q + 1] = off[q] + static_cast<int>(32 * w);
    }
    const size_t pad = std::max(off[slices], 1);
    std::vector<int> sc(pad, -1);
    std::vector<double> sv(pad, 0.0);
    for (int64_t i = 0; i < n; ++i) {
      const int base = off[i >> 5] + static_cast<int>(i & 31);
      for (int64_t t = indptr[i]; t < indptr[i + 1]; ++t) {
        sc[base + 32 * (t - indptr[i])] = indices[t];
        sv[base + 32 * (t - indptr[i])] = data[t];
      }
    }
    CUDA_TRY(upload(&c->d_sell_off, off));
    CUDA_TRY(upload(&c->d_sell_col, sc));
    CUDA_TRY(upload(&c->d_sell_val, sv));
    c->sell.n = static_cast<int>(n);
    c->sell.slices = slices;
    c->sell.off = c->d_sell_off;
    c->sell.col = c->d_sell_col;
    c->sell.val = c->d_sell_val;
  }
  // Krylov vectors
  CUDA_TRY(dalloc(&c->d_b, n)); CUDA_TRY(dalloc(&c->d_u, n)); CUDA_TRY(dalloc(&c->d_r, n));
  CUDA_TRY(dalloc(&c->d_p, n)); CUDA_TRY(dalloc(&c->d_q, n)); CUDA_TRY(dalloc(&c->d_z, n));
  CUDA_TRY(dalloc(&c->d_rin, n)); CUDA_TRY(dalloc(&c->d_zout, n));
  dfree(c->d_zold);  // flexible CG scratch, reallocated at the new size on demand
  const int pblocks = std::max((static_cast<int>(n) + 255) / 256, 148 * 8) + 1;
  CUDA_TRY(dalloc(&c->d_partials, 2ull * pblocks));
  if (!c->d_st) {
    CUDA_TRY(cudaMalloc(&c->d_st, sizeof(PcgState)));
    CUDA_TRY(cudaMemset(c->d_st, 0, sizeof(PcgState)));
  }
  if (!c->d_status) {
    CUDA_TRY(cudaMalloc(&c->d_status, sizeof(int)));
    CUDA_TRY(cudaMemset(c->d_status, 0, sizeof(int)));
  }
  if (c->h_pin_a) cudaFreeHost(c->h_pin_a);
  if (c->h_pin_b) cudaFreeHost(c->h_pin_b);
  c->h_pin_a = c->h_pin_b = nullptr;
  CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&c->h_pin_a), sizeof(double) * n));
  CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&c->h_pin_b), sizeof(double) * n));
  free_graphs(c);
  return kOk;
}

extern "C" int ddmgnn_set_geometry(ddmgnn_ctx* c, int64_t n, const double* coords) {
  if (!c) return fail(kValueError, "null context");
  if (c->n && n != c->n) return fail(kValueError, "expected coords of shape (" + std::to_string(c->n) + ", 2)");
  c->coords.assign(coords, coords + 2 * n);
  c->built = false;
  return kOk;
}

extern "C" int ddmgnn_set_decomposition(ddmgnn_ctx* c, int64_t k, const int64_t* sub_ptr,
                                        const int64_t* sub_idx) {
  if (!c) return fail(kValueError, "null context");
  if (k <= 0 || k >= (1ll << 31)) return fail(kValueError, "number of subdomains out of range");
  c->K = static_cast<int>(k);
  c->sub_ptr.assign(sub_ptr, sub_ptr + k + 1);
  c->sub_idx.assign(sub_idx, sub_idx + sub_ptr[k]);
  c->built = false;
  return kOk;
}

extern "C" int ddmgnn_set_batch_cap(ddmgnn_ctx* c, int64_t cap) {
  if (!c) return fail(kValueError, "null context");
  if (cap < 1) return fail(kValueError, "batch node cap must be >= 1");
  c->batch_cap = cap;
  return kOk;
}

static int refresh_classes(ddmgnn_ctx* c);

extern "C" int ddmgnn_set_model(ddmgnn_ctx* c, int k_bar, int d, double alpha,
                                const double* params, int64_t n_params) {
  if (!c) return fail(kValueError, "null context");
  std::string err;
  PackedModel m;
  int st = pack_model(k_bar, d, alpha, params, n_params, &m, &err);
  if (st) return fail(st, err);
  // layer 1 runs on h = 0: its h rows may be skipped when 0 * w = 0 exactly, i.e.
  // when every weight of the slot is finite (else the reference's NaN must appear)
  m.h0_finite = 1;
  for (int i = 0; i < m.stride && i < static_cast<int>(m.bank.size()); ++i)
    if (!std::isfinite(m.bank[i])) m.h0_finite = 0;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(dalloc(&c->d_bank, m.bank.size()));
  CUDA_TRY(cudaMemcpy(c->d_bank, m.bank.data(), sizeof(float) * m.bank.size(),
                      cudaMemcpyHostToDevice));
  const bool dim_changed = !c->have_model || c->model.d != d || c->model.k_bar != k_bar;
  c->model = std::move(m);
  c->have_model = true;
  free_graphs(c);
  if (c->built && dim_changed) return refresh_classes(c);
  return kOk;
}

extern "C" int ddmgnn_set_coarse_inverse(ddmgnn_ctx* c, int64_t k, const double* inv) {
  if (!c) return fail(kValueError, "null context");
  if (c->K && k != c->K) return fail(kValueError, "coarse size must equal the number of subdomains");
  CUDA_TRY(cudaSetDevice(c->device));
  // rows padded to an even length (zero column) so the GEMV streams 16-byte loads
  const int64_t ld = (k + 1) / 2 * 2;
  CUDA_TRY(dalloc(&c->d_cinv, static_cast<size_t>(k) * ld));
  CUDA_TRY(cudaMemset(c->d_cinv, 0, sizeof(double) * k * ld));
  CUDA_TRY(cudaMemcpy2D(c->d_cinv, sizeof(double) * ld, inv, sizeof(double) * k,
                        sizeof(double) * k, k, cudaMemcpyHostToDevice));
  c->coarse_ld = static_cast<int>(ld);
  c->coarse_k = static_cast<int>(k);
  free_graphs(c);
  return kOk;
}


// ---- staged input of ddmgnn_apply_host -------------------------------------------
constexpr int kStages = 4;

// cuStreamWriteValue32 (driver API, resolved at run time so the library has no
// link-time dependency on libcuda): the copy stream writes a chunk's ready flag
// once the chunk's H2D copy has completed, with a memory barrier before the write.
using WriteValue32Fn = int (*)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
static WriteValue32Fn write_value32() {
  static WriteValue32Fn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WriteValue32Fn>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

// Chunk c of r = DOFs [c chunk, (c+1) chunk); subdomain i reads up to its largest
// DOF, so it may start after chunk max_i / chunk.  Order for the staged launch: the
// n_big leading (cluster-path) subdomains as in the LPT order, then the rest by
// stage, LPT within a stage (stable partition of the LPT order).
static cudaError_t plan_staged_input(ddmgnn_ctx* c, int n_big, bool has_flat) {
  dfree(c->d_sub_stage);
  dfree(c->d_order_staged);
  c->staged_ok = 0;
  const char* env = getenv("DDMGNN_STAGED_INPUT");
  if ((env && env[0] == '0') || has_flat || c->n <= 0 || c->K <= 0) return cudaSuccess;
  const long long chunk = ((static_cast<long long>(c->n) + kStages - 1) / kStages + 15) / 16 * 16;
  std::vector<int> stage(c->K);
  for (int i = 0; i < c->K; ++i) {
    int64_t mx = 0;
    for (int64_t t = c->sub_ptr[i]; t < c->sub_ptr[i + 1]; ++t) mx = std::max(mx, c->sub_idx[t]);
    stage[i] = static_cast<int>(std::min<long long>(kStages - 1, mx / chunk));
  }
  const auto& ord = c->lay.h_order;
  std::vector<int> staged(ord.begin(), ord.begin() + n_big);
  for (int st = 0; st < kStages; ++st)
    for (int t = n_big; t < c->K; ++t)
      if (stage[ord[t]] == st) staged.push_back(ord[t]);
  cudaError_t e = upload(&c->d_sub_stage, stage);
  if (e == cudaSuccess) e = upload(&c->d_order_staged, staged);
  if (e == cudaSuccess && !c->d_ready) {
    e = cudaMalloc(&c->d_ready, sizeof(unsigned int) * kStages);
    if (e == cudaSuccess) e = cudaMemset(c->d_ready, 0, sizeof(unsigned int) * kStages);
    c->stage_epoch = 0;
  }
  if (e != cudaSuccess) return e;
  c->stage_chunk = chunk;
  c->staged_ok = write_value32() != nullptr;
  return cudaSuccess;
}

// Plan the shared-memory placement for the current latent dimension and
// (re)allocate the per-node global scratch it needs.
static int refresh_classes(ddmgnn_ctx* c) {
  if (!c->built || !c->have_model) return kOk;
  const int d = c->model.d;
  c->gnn_smem = gnn_plan_smem(d, c->lay.k_max, &c->cap0);
  // DDMGNN_CAP0=<k>: route every subdomain larger than k to the cluster/flat paths
  // (experiments: 0 sends all subdomains through the cluster path)
  if (const char* e = getenv("DDMGNN_CAP0")) c->cap0 = std::min(c->cap0, atoi(e));
  const auto& sp = c->lay.h_sub_ptr;
  // oversized subdomains (k > cap0) lead the LPT order: those an 8-CTA cluster can
  // hold take the cluster path (smallest cluster size whose per-CTA share fits),
  // the rest (the largest, hence the leading ones) the flat path
  // With DDMGNN_CLUSTER_2CTA=1 the cluster size is the smallest whose per-CTA
  // share fits half an SM's shared memory, so two cluster CTAs (448 threads each)
  // share each SM — measured slower than the smallest fitting cluster (twice the
  // DSMEM traffic; profiles/r01_cluster_2cta_configE.jsonl), hence opt-in.
  const char* env = getenv("DDMGNN_CLUSTER");
  const bool use_cluster = !(env && env[0] == '0');
  const char* env5 = getenv("DDMGNN_H0_SKIP");
  c->h0_skip = !(env5 && env5[0] == '0');
  const char* env4 = getenv("DDMGNN_FUSED_TAIL");
  c->fused_tail = env4 && env4[0] == '1';
  const char* env3 = getenv("DDMGNN_TWO_CTA");
  c->two_cta = !(env3 && env3[0] == '0');
  const char* env2 = getenv("DDMGNN_CLUSTER_2CTA");
  const bool two_cta = env2 && env2[0] == '1';
  const int node0 = gnn_smem_node_bytes(d);
  constexpr int kClusterStatic = 1024;  // GnnShared + partial sums, rounded up
  constexpr int kSmPerCtaReserve = 1024;
  const int cap2 = node0 ? (228 * 1024 / 2 - kClusterStatic - kSmPerCtaReserve -
                            static_cast<int>(kTcSmemBytes)) / node0 - 1
                         : 0;
  int nb = 0;
  std::vector<int2> bsl;
  std::vector<int> csub[3];
  for (int t = 0; t < c->K; ++t) {
    const int i = c->lay.h_order[t];
    const int k = sp[i + 1] - sp[i];
    if (k <= c->cap0) break;
    ++nb;
    int j = -1;
    for (int pass = two_cta ? 0 : 1; use_cluster && pass < 2 && j < 0; ++pass)
      for (int jj = 0; jj < 3 && j < 0; ++jj) {
        const int cs = 2 << jj, npc = ((k + cs - 1) / cs + 31) / 32 * 32;
        if (npc <= (pass == 0 ? cap2 : c->cap0)) j = jj;
      }
    if (j >= 0) {
      csub[j].push_back(i);
    } else {
      for (int q = 0; q * 32 < k; ++q) bsl.push_back(make_int2(i, q));
    }
  }
  std::vector<int> cs_all;
  for (int j = 0; j < 3; ++j) {
    c->cluster_count[j] = static_cast<int>(csub[j].size());
    int npc_max = 0;
    for (int i : csub[j]) {
      const int k = sp[i + 1] - sp[i], cs = 2 << j;
      npc_max = std::max(npc_max, ((k + cs - 1) / cs + 31) / 32 * 32);
    }
    const size_t sm = static_cast<size_t>(npc_max + 1) * node0 + kTcSmemBytes;
    c->cluster_smem[j] = static_cast<int>(std::min<size_t>(sm, kGnnSmemMax));
    const bool pair = 2 * (sm + kClusterStatic + kSmPerCtaReserve) <= 228u * 1024u;
    c->cluster_threads[j] = (two_cta && pair) ? kGnnThreads / 2 / 32 * 32 : kGnnThreads;
    cs_all.insert(cs_all.end(), csub[j].begin(), csub[j].end());
  }
  dfree(c->d_csubs);
  c->d_csubs = nullptr;
  if (!cs_all.empty()) CUDA_TRY(upload(&c->d_csubs, cs_all));
  c->n_big = nb;
  const int hs = (d % 2 == 0) ? d : d + 1;
  const int qs = (2 * d + 3) / 4 * 4;
  const size_t V = c->lay.V;
  const bool multi = c->model.n_chunks() > 1;
  // + one dummy row per subdomain (lanes past k / SELL padding targets)
  CUDA_TRY(dalloc(&c->d_hbuf, (multi || nb) ? (V + c->K) * hs : 0));
  CUDA_TRY(dalloc(&c->d_cbuf, (multi || nb) ? V : 0));
  CUDA_TRY(dalloc(&c->d_qbuf, bsl.empty() ? 0 : (V + c->K) * qs));
  CUDA_TRY(plan_staged_input(c, nb, !bsl.empty()));
  dfree(c->d_bslices);
  c->n_bslices = static_cast<int>(bsl.size());
  while (bsl.size() % kFlatWarps) bsl.push_back(make_int2(-1, 0));  // padding slices
  if (!bsl.empty()) CUDA_TRY(upload(&c->d_bslices, bsl));
  return kOk;
}

extern "C" int ddmgnn_build(ddmgnn_ctx* c) {
  if (!c) return fail(kValueError, "null context");
  if (!c->n) return fail(kStateError, "set_matrix must be called before build");
  if (c->coords.size() != 2ull * c->n)
    return fail(kValueError, "expected coords of shape (" + std::to_string(c->n) + ", 2)");
  if (!c->K) return fail(kStateError, "set_decomposition must be called before build");
  CUDA_TRY(cudaSetDevice(c->device));
  // host copy of the CSR structure for the builder
  std::vector<int> rp(c->n + 1);
  CUDA_TRY(cudaMemcpy(rp.data(), c->d_rowptr, sizeof(int) * (c->n + 1), cudaMemcpyDeviceToHost));
  std::vector<int64_t> rp64(rp.begin(), rp.end());
  std::vector<int32_t> col(std::max<long long>(c->nnz, 1));
  if (c->nnz)
    CUDA_TRY(cudaMemcpy(col.data(), c->d_col, sizeof(int) * c->nnz, cudaMemcpyDeviceToHost));
  HostLayout H;
  std::string err;
  int st = build_host_layout(c->n, rp64.data(), col.data(), c->coords.data(), c->K,
                             c->sub_ptr.data(), c->sub_idx.data(), &H, &err);
  if (st) return fail(st, err);
  free_layout(c);
  DeviceLayout& L = c->lay;
  L.n = H.n; L.K = H.K; L.V = H.V; L.S = H.S; L.k_max = H.k_max; L.E = H.E; L.E_pad = H.E_pad;
  CUDA_TRY(upload(&L.sub_ptr, H.sub_ptr));
  CUDA_TRY(upload(&L.idx, H.idx));
  CUDA_TRY(upload(&L.order, H.order));
  CUDA_TRY(upload(&L.slice_base, H.slice_base));
  CUDA_TRY(upload(&L.slice_off, H.slice_off));
  CUDA_TRY(upload(&L.reach, H.reach));
  CUDA_TRY(upload(&L.deg, H.deg));
  CUDA_TRY(dalloc(&L.edges, std::max<long long>(H.E_pad, 1)));
  if (H.E_pad)
    CUDA_TRY(cudaMemcpy(L.edges, H.edges.data(), sizeof(float) * H.edges.size(),
                        cudaMemcpyHostToDevice));
  CUDA_TRY(dalloc(&L.xy, std::max(H.V, 1)));
  CUDA_TRY(cudaMemcpy(L.xy, H.xy.data(), sizeof(float) * H.xy.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(upload(&L.tptr, H.tptr));
  CUDA_TRY(dalloc(&L.tent, std::max(H.V, 1)));
  CUDA_TRY(cudaMemcpy(L.tent, H.tent.data(), sizeof(int) * H.tent.size(), cudaMemcpyHostToDevice));
  CUDA_TRY(upload(&L.pou, H.pou));
  L.h_sub_ptr = H.sub_ptr;
  L.h_order = H.order;
  CUDA_TRY(dalloc(&c->d_r0r, c->K)); CUDA_TRY(dalloc(&c->d_scale, c->K));
  CUDA_TRY(dalloc(&c->d_y, c->K)); CUDA_TRY(dalloc(&c->d_zloc, std::max(H.V, 1)));
  CUDA_TRY(dalloc(&c->d_bad, c->K)); CUDA_TRY(dalloc(&c->d_outbad, c->K));
  CUDA_TRY(cudaMemset(c->d_scale, 0, sizeof(double) * c->K));
  c->built = true;
  return refresh_classes(c);
}

extern "C" int ddmgnn_info(ddmgnn_ctx* c, int64_t* out, int n_out) {
  if (!c) return fail(kValueError, "null context");
  const int ncl = (c->cluster_count[0] > 0) + (c->cluster_count[1] > 0) + (c->cluster_count[2] > 0);
  int64_t v[14] = {c->n, c->K, c->lay.V, c->lay.E, c->lay.E_pad, c->lay.k_max, c->lay.S,
                   c->model.k_bar, c->model.d, c->model.lmax, c->model.n_chunks(), c->n_big,
                   c->cluster_count[0] + c->cluster_count[1] + c->cluster_count[2], ncl};
  for (int i = 0; i < n_out && i < 14; ++i) out[i] = v[i];
  return kOk;
}

extern "C" int ddmgnn_export_local_graph(ddmgnn_ctx* c, int64_t sub, int64_t* n_edges,
                                         int32_t* src, int32_t* dst, float* vec3) {
  if (!c || !c->built) return fail(kStateError, "build must be called first");
  if (sub < 0 || sub >= c->K) return fail(kValueError, "subdomain out of range");
  const DeviceLayout& L = c->lay;
  const int b = L.h_sub_ptr[sub], k = L.h_sub_ptr[sub + 1] - b;
  std::vector<uint16_t> deg(std::max(k, 1));
  if (k) CUDA_TRY(cudaMemcpy(deg.data(), L.deg + b, sizeof(uint16_t) * k, cudaMemcpyDeviceToHost));
  int64_t ne = 0;
  for (int a = 0; a < k; ++a) ne += deg[a];
  *n_edges = ne;
  if (!src) return kOk;
  int sb = 0;
  CUDA_TRY(cudaMemcpy(&sb, L.slice_base + sub, sizeof(int), cudaMemcpyDeviceToHost));
  const int ns = (k + 31) / 32;
  std::vector<int> so(ns + 1);
  CUDA_TRY(cudaMemcpy(so.data(), L.slice_off + sb, sizeof(int) * (ns + 1), cudaMemcpyDeviceToHost));
  std::vector<float2> rec(std::max(so[ns] - so[0], 1));
  if (so[ns] > so[0])
    CUDA_TRY(cudaMemcpy(rec.data(), L.edges + so[0], sizeof(float2) * (so[ns] - so[0]),
                        cudaMemcpyDeviceToHost));
  std::vector<int> gidx(std::max(k, 1));
  if (k) CUDA_TRY(cudaMemcpy(gidx.data(), L.idx + b, sizeof(int) * k, cudaMemcpyDeviceToHost));
  int64_t o = 0;
  for (int a = 0; a < k; ++a) {
    for (int e = 0; e < deg[a]; ++e) {
      const float2 r = rec[so[a >> 5] - so[0] + 32 * e + (a & 31)];
      src[o] = a;
      int t;
      std::memcpy(&t, &r.y, 4);
      dst[o] = t;
      // the device folds edge_vec into per-node projections; report the fp32
      // rounding of the fp64 difference it stands for (dss.py:184)
      const int gs = gidx[a], gt = gidx[t];
      vec3[3 * o] = static_cast<float>(c->coords[2 * gt] - c->coords[2 * gs]);
      vec3[3 * o + 1] = static_cast<float>(c->coords[2 * gt + 1] - c->coords[2 * gs + 1]);
      vec3[3 * o + 2] = r.x;
      ++o;
    }
  }
  return kOk;
}

static int ready(ddmgnn_ctx* c, int level) {
  if (!c) return fail(kValueError, "null context");
  if (level == DDMGNN_PRECOND_NONE) return c->n ? kOk : fail(kStateError, "no matrix set");
  if (level == DDMGNN_IC0) return c->have_ic0 ? kOk : fail(kStateError, "IC(0) apply needs set_ic0");
  if (level == DDMGNN_ASM_ONE || level == DDMGNN_ASM_TWO) {
    if (!c->have_asm) return fail(kStateError, "DDM-LU apply needs alloc_local_inverses");
    if (level == DDMGNN_ASM_TWO && c->coarse_k != c->K)
      return fail(kStateError, "two-level apply needs set_coarse_inverse");
    return kOk;
  }
  if (level != DDMGNN_LEVEL_ONE && level != DDMGNN_LEVEL_TWO)
    return fail(kValueError, "level must be 1 (one-level) or 2 (two-level)");
  if (!c->built) return fail(kStateError, "build must be called before apply");
  if (!c->have_model) return fail(kStateError, "set_model must be called before apply");
  if (level == DDMGNN_LEVEL_TWO && c->coarse_k != c->K)
    return fail(kStateError, "two-level apply needs set_coarse_inverse");
  return kOk;
}

// ---- the GNN weight bank is process-global device state ----
// The fused GNN kernels read their weights from a __constant__ bank per compiled
// latent width (gnn_dim.cu), which every apply re-fills on its stream before the
// launch.  Two applies on different streams (two contexts, or one context used from
// two streams) must therefore not overlap: every bank use is chained behind the
// previous one on the device by an event whenever the stream changes.  The host
// mutex keeps upload + launch + record of one use together.
namespace {
struct BankChain {
  std::mutex m;
  cudaEvent_t ev = nullptr;
  cudaStream_t last = nullptr;
  bool valid = false;
};
BankChain g_bank[64];

class BankUse {
 public:
  BankUse(int device, cudaStream_t s) : s_(s) {
    g_ = (device >= 0 && device < 64) ? &g_bank[device] : nullptr;
    if (!g_) return;
    lk_ = std::unique_lock<std::mutex>(g_->m);
    if (!g_->ev) err_ = cudaEventCreateWithFlags(&g_->ev, cudaEventDisableTiming);
    if (err_ == cudaSuccess && g_->valid && g_->last != s) err_ = cudaStreamWaitEvent(s, g_->ev, 0);
  }
  cudaError_t error() const { return err_; }
  // call after the last bank-reading launch has been enqueued on s
  cudaError_t done() {
    if (!g_ || err_ != cudaSuccess) return err_;
    err_ = cudaEventRecord(g_->ev, s_);
    g_->last = s_;
    g_->valid = err_ == cudaSuccess;
    return err_;
  }

 private:
  BankChain* g_ = nullptr;
  cudaStream_t s_;
  std::unique_lock<std::mutex> lk_;
  cudaError_t err_ = cudaSuccess;
};

bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}
}  // namespace

static cudaError_t enqueue_gnn_impl(ddmgnn_ctx* c, const double* r, int* status, const int* skip,
                                    cudaStream_t s);

// Enqueue restriction + GNN chunks.  status/skip: apply error word and PCG skip word.
// Under stream capture (PCG graph) the chain is kept around the graph launches instead.
static cudaError_t enqueue_gnn(ddmgnn_ctx* c, const double* r, int* status, const int* skip,
                               cudaStream_t s) {
  if (capturing(s)) return enqueue_gnn_impl(c, r, status, skip, s);
  BankUse use(c->device, s);
  if (use.error() != cudaSuccess) return use.error();
  cudaError_t e = enqueue_gnn_impl(c, r, status, skip, s);
  if (e != cudaSuccess) return e;
  return use.done();
}

static cudaError_t enqueue_gnn_impl(ddmgnn_ctx* c, const double* r, int* status, const int* skip,
                               cudaStream_t s) {
  const DeviceLayout& L = c->lay;
  const PackedModel& M = c->model;
  GnnArgs a{};
  a.sub_ptr = L.sub_ptr; a.idx = L.idx; a.order = L.order; a.slice_base = L.slice_base;
  a.slice_off = L.slice_off; a.deg = L.deg;
  {  // DDMGNN_DATAFLOW=0: two CTA barriers per layer (the schedule before round 2's end)
    const char* df = getenv("DDMGNN_DATAFLOW");
    a.reach = (df && df[0] == '0') ? nullptr : L.reach;
  } a.edges = L.edges; a.xy = L.xy; a.pou = L.pou;
  a.r = r; a.r0r = c->d_r0r; a.scale = c->d_scale; a.zloc = c->d_zloc;
  a.hbuf = c->d_hbuf; a.cbuf = c->d_cbuf; a.qbuf = c->d_qbuf;
  a.bslices = c->d_bslices; a.n_bslices = c->n_bslices;
  a.csubs = c->d_csubs;
  a.two_cta = c->two_cta;
  a.h0_skip = M.h0_finite && c->h0_skip;
  for (int j = 0; j < 3; ++j) {
    a.cluster_count[j] = c->cluster_count[j];
    a.cluster_smem[j] = c->cluster_smem[j];
    a.cluster_threads[j] = c->cluster_threads[j];
  }
  a.bad_layer = c->d_bad; a.out_bad = c->d_outbad; a.status = status; a.skip = skip;
  a.alpha = M.alpha;
  const int nch = M.n_chunks();
  for (int ch = 0; ch < nch; ++ch) {
    cudaError_t e = upload_bank(M.d, c->d_bank + static_cast<size_t>(ch) * kConstFloats, s);
    if (e != cudaSuccess) return e;
    a.first = ch == 0;
    a.last = ch == nch - 1;
    if (c->stage_now && ch == 0) {  // ddmgnn_apply_host: r still arriving in chunks
      a.order = c->d_order_staged;
      a.ready = c->d_ready;
      a.sub_stage = c->d_sub_stage;
      a.epoch = c->stage_epoch;
    } else {
      a.order = L.order;
      a.ready = nullptr;
      a.sub_stage = nullptr;
      a.epoch = 0;
    }
    a.layer0 = ch * M.lmax + 1;
    a.nl = std::min(M.lmax, M.k_bar - ch * M.lmax);
    a.order_begin = 0;
    a.cap0 = c->cap0;
    const int k_small = c->n_big < c->K ? c->lay.h_sub_ptr[c->lay.h_order[c->n_big] + 1] -
                                              c->lay.h_sub_ptr[c->lay.h_order[c->n_big]]
                                        : 0;
    e = launch_gnn(M.d, c->K, c->n_big, k_small, c->gnn_smem, a, s, c->side, c->ev_fork,
                   c->ev_join);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Full apply: z = M r.  mode 1 = PCG (fused <r,z>, beta).
static cudaError_t enqueue_apply(ddmgnn_ctx* c, const double* r, double* z, int level,
                                 int* status, const int* skip, int mode, cudaStream_t s) {
  const bool asm_ = level == DDMGNN_ASM_ONE || level == DDMGNN_ASM_TWO;
  const bool two = level == DDMGNN_LEVEL_TWO || level == DDMGNN_ASM_TWO;
  cudaError_t e;
  if (level == DDMGNN_IC0) {  // z = L^-T (L^-1 r)  (sparse.py:177-179)
    const bool flex = mode == 1 && c->pcg_flex;
    if (flex) {
      e = cudaMemcpyAsync(c->d_zold, z, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return e;
    }
    e = launch_ic0_apply(c->ic0, r, c->d_ic_tmp, z, skip, s);
    if (e != cudaSuccess || mode != 1) return e;
    return launch_rz_beta(c->n, r, z, flex ? c->d_zold : nullptr, c->d_partials, c->d_st, s);
  }
  if (asm_) {
    e = launch_asm_local(c->K, c->lay.k_max, c->lay.sub_ptr, c->lay.idx, c->d_ainv_off,
                         c->d_ainv, c->lay.pou, r, c->d_zloc, c->d_r0r, c->d_scale, skip, s);
  } else {
    e = enqueue_gnn(c, r, status, skip, s);
  }
  if (e != cudaSuccess) return e;
  if (two) {
    e = launch_coarse_gemv(c->K, c->coarse_ld, c->d_cinv, c->d_r0r, c->d_y, skip, s);
    if (e != cudaSuccess) return e;
  }
  return launch_prolong(c->n, (two ? 1 : 0) | (asm_ ? 2 : 0), c->lay.tptr, c->lay.tent,
                        c->lay.pou, c->d_y, c->d_scale, c->d_zloc, z, r, c->d_partials, c->d_st,
                        mode, skip, s);
}

// Reproduce the reference's error precedence (hybrid.py:121-131, dss.py:324-325):
// batches of loaded subdomains in order; within a batch a latent error (smallest
// layer) wins over an output error (smallest subdomain).
static int report_apply_error(ddmgnn_ctx* c) {
  const int K = c->K;
  std::vector<int> bad(K), outbad(K);
  std::vector<double> scale(K);
  CUDA_TRY(cudaMemcpy(bad.data(), c->d_bad, sizeof(int) * K, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(outbad.data(), c->d_outbad, sizeof(int) * K, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(scale.data(), c->d_scale, sizeof(double) * K, cudaMemcpyDeviceToHost));
  const auto& sp = c->lay.h_sub_ptr;
  std::vector<int> loaded;
  for (int i = 0; i < K; ++i)
    if (scale[i] != 0.0) loaded.push_back(i);
  size_t pos = 0;
  while (pos < loaded.size()) {
    size_t end = pos;
    long long load = 0;
    while (end < loaded.size()) {  // plan_batches, hybrid.py:49-68
      const long long cnt = sp[loaded[end] + 1] - sp[loaded[end]];
      if (end > pos && load + cnt > c->batch_cap) break;
      load += cnt;
      ++end;
    }
    int min_layer = 0;
    for (size_t t = pos; t < end; ++t) {
      const int b = bad[loaded[t]];
      if (b && (!min_layer || b < min_layer)) min_layer = b;
    }
    if (min_layer)
      return fail(kRuntimeError, "non-finite latent state at message-passing iteration " +
                                     std::to_string(min_layer));
    for (size_t t = pos; t < end; ++t)
      if (outbad[loaded[t]])
        return fail(kRuntimeError,
                    "non-finite model output in subdomain " + std::to_string(loaded[t]));
    pos = end;
  }
  return fail(kRuntimeError, "non-finite model state (unlocated)");
}

static int check_status_word(ddmgnn_ctx* c, cudaStream_t s) {
  int st = 0;
  CUDA_TRY(cudaMemcpyAsync(&c->h_st->pad, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  st = c->h_st->pad;
  if (st == kStagingTimeout) {
    CUDA_TRY(cudaMemsetAsync(c->d_status, 0, sizeof(int), s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return fail(kCudaError, "input staging timed out (a chunk of r never reached the device)");
  }
  if (st != 0) {
    CUDA_TRY(cudaMemsetAsync(c->d_status, 0, sizeof(int), s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return report_apply_error(c);
  }
  return kOk;
}

extern "C" int ddmgnn_apply(ddmgnn_ctx* c, const double* r, double* z, int level, void* stream,
                            int check) {
  int st = ready(c, level);
  if (st) return st;
  if (level == DDMGNN_PRECOND_NONE) return fail(kValueError, "level must be 1 or 2");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = pick(c, stream);
  if (check) CUDA_TRY(cudaMemsetAsync(c->d_status, 0, sizeof(int), s));
  CUDA_TRY(enqueue_apply(c, r, z, level, c->d_status, nullptr, 0, s));
  if (check) return check_status_word(c, s);
  return kOk;
}

extern "C" int ddmgnn_apply_host(ddmgnn_ctx* c, const double* r, double* z, int level) {
  int st = ready(c, level);
  if (st) return st;
  if (level == DDMGNN_PRECOND_NONE) return fail(kValueError, "level must be 1 or 2");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  const size_t bytes = sizeof(double) * c->n;
  // page-locked caller buffers are DMA'd directly; pageable ones go through the
  // context's pinned staging buffers
  auto pinned = [](const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool r_pin = pinned(r), z_pin = pinned(z);
  const double* src = r;
  if (!r_pin) {
    std::memcpy(c->h_pin_a, r, bytes);
    src = c->h_pin_a;
  }
  const bool gnn = level == DDMGNN_LEVEL_ONE || level == DDMGNN_LEVEL_TWO;
  if (gnn && c->staged_ok) {
    // r in kStages chunks on the copy stream, each followed by its ready flag; the
    // GNN's CTAs (ordered by the chunk they need) start on the first chunk while the
    // rest is still crossing PCIe
    // the copies and flag writes are enqueued BEFORE the kernels that wait for them:
    // streams can share hardware queues, so a copy queued behind a spinning kernel
    // could never start
    const unsigned int ep = ++c->stage_epoch;
    WriteValue32Fn wv = write_value32();
    for (int ci = 0; ci < kStages; ++ci) {
      const long long off = ci * c->stage_chunk;
      const long long cnt = std::min<long long>(c->stage_chunk, c->n - off);
      if (cnt > 0)
        CUDA_TRY(cudaMemcpyAsync(c->d_rin + off, src + off, sizeof(double) * cnt,
                                 cudaMemcpyHostToDevice, c->copy));
      if (wv(c->copy, reinterpret_cast<unsigned long long>(c->d_ready + ci), ep, 0) != 0)
        return fail(kCudaError, "cuStreamWriteValue32 failed");
    }
    CUDA_TRY(cudaEventRecord(c->ev_copied, c->copy));
    CUDA_TRY(cudaMemsetAsync(c->d_status, 0, sizeof(int), s));
    c->stage_now = 1;
    cudaError_t e = enqueue_apply(c, c->d_rin, c->d_zout, level, c->d_status, nullptr, 0, s);
    c->stage_now = 0;
    CUDA_TRY(e);
    CUDA_TRY(cudaStreamWaitEvent(s, c->ev_copied, 0));  // formal join of the copy stream
  } else {
    CUDA_TRY(cudaMemcpyAsync(c->d_rin, src, bytes, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(c->d_status, 0, sizeof(int), s));
    CUDA_TRY(enqueue_apply(c, c->d_rin, c->d_zout, level, c->d_status, nullptr, 0, s));
  }
  CUDA_TRY(cudaMemcpyAsync(z_pin ? z : c->h_pin_b, c->d_zout, bytes, cudaMemcpyDeviceToHost, s));
  st = check_status_word(c, s);
  if (st) return st;
  if (!z_pin) std::memcpy(z, c->h_pin_b, bytes);
  return kOk;
}

extern "C" int ddmgnn_launch_gnn_only(ddmgnn_ctx* c, const double* r, void* stream) {
  int st = ready(c, DDMGNN_LEVEL_ONE);
  if (st) return st;
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(enqueue_gnn(c, r, c->d_status, nullptr, pick(c, stream)));
  return kOk;
}

extern "C" int ddmgnn_apply_status(ddmgnn_ctx* c, void* stream) {
  if (!c || !c->built) return fail(kStateError, "build must be called first");
  CUDA_TRY(cudaSetDevice(c->device));
  return check_status_word(c, pick(c, stream));
}

extern "C" int ddmgnn_set_ic0(ddmgnn_ctx* c) {
  if (!c || !c->n) return fail(kStateError, "no matrix set");
  CUDA_TRY(cudaSetDevice(c->device));
  const int n = c->n;
  std::vector<int> rp(n + 1), ci(std::max<long long>(c->nnz, 1));
  std::vector<double> v(std::max<long long>(c->nnz, 1));
  CUDA_TRY(cudaMemcpy(rp.data(), c->d_rowptr, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost));
  if (c->nnz) {
    CUDA_TRY(cudaMemcpy(ci.data(), c->d_col, sizeof(int) * c->nnz, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(v.data(), c->d_val, sizeof(double) * c->nnz, cudaMemcpyDeviceToHost));
  }
  std::vector<int> lp, lc;
  std::vector<double> lv;
  std::string err;
  const int st = ic0_factor(n, rp.data(), ci.data(), v.data(), &lp, &lc, &lv, &err);
  if (st) return fail(st, err);
  // U = L^T: row j of U = column j of L, diagonal first (rows of L ascending)
  const int nnz = lp[n];
  std::vector<int> up(n + 1, 0), uc(nnz);
  std::vector<double> uv(nnz);
  for (int t = 0; t < nnz; ++t) up[lc[t] + 1]++;
  for (int j = 0; j < n; ++j) up[j + 1] += up[j];
  {
    std::vector<int> cur(up.begin(), up.end() - 1);
    for (int i = 0; i < n; ++i)
      for (int t = lp[i]; t < lp[i + 1]; ++t) {
        const int slot = cur[lc[t]]++;
        uc[slot] = i;
        uv[slot] = lv[t];
      }
  }
  CUDA_TRY(upload(&c->d_ic_lp, lp)); CUDA_TRY(upload(&c->d_ic_lc, lc));
  CUDA_TRY(upload(&c->d_ic_lv, lv)); CUDA_TRY(upload(&c->d_ic_up, up));
  CUDA_TRY(upload(&c->d_ic_uc, uc)); CUDA_TRY(upload(&c->d_ic_uv, uv));
  CUDA_TRY(dalloc(&c->d_ic_tmp, n));
  CUDA_TRY(dalloc(&c->d_ic_ready, 2 * n));
  CUDA_TRY(cudaMemset(c->d_ic_ready, 0, sizeof(int) * 2 * n));
  CUDA_TRY(dalloc(&c->d_ic_state, 4));
  CUDA_TRY(cudaMemset(c->d_ic_state, 0, sizeof(int) * 4));
  Ic0Device& f = c->ic0;
  f.n = n;
  f.lp = c->d_ic_lp; f.lc = c->d_ic_lc; f.lv = c->d_ic_lv;
  f.up = c->d_ic_up; f.uc = c->d_ic_uc; f.uv = c->d_ic_uv;
  f.ready_l = c->d_ic_ready; f.ready_u = c->d_ic_ready + n; f.state = c->d_ic_state;
  c->have_ic0 = true;
  free_graphs(c);
  return kOk;
}

extern "C" int ddmgnn_export_ic0(ddmgnn_ctx* c, int64_t* nnz, int32_t* indptr, int32_t* indices,
                                 double* data) {
  if (!c || !c->have_ic0) return fail(kStateError, "set_ic0 must be called first");
  int total = 0;
  CUDA_TRY(cudaMemcpy(&total, c->d_ic_lp + c->n, sizeof(int), cudaMemcpyDeviceToHost));
  *nnz = total;
  if (!indptr) return kOk;
  CUDA_TRY(cudaMemcpy(indptr, c->d_ic_lp, sizeof(int) * (c->n + 1), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(indices, c->d_ic_lc, sizeof(int) * total, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(data, c->d_ic_lv, sizeof(double) * total, cudaMemcpyDeviceToHost));
  return kOk;
}

extern "C" int ddmgnn_alloc_local_inverses(ddmgnn_ctx* c, const int64_t* off, double** dev_out) {
  if (!c || !c->built) return fail(kStateError, "build must be called first");
  if (!off || !dev_out) return fail(kValueError, "null argument");
  const auto& sp = c->lay.h_sub_ptr;
  for (int i = 0; i < c->K; ++i) {
    const int64_t k = sp[i + 1] - sp[i];
    if (off[i + 1] - off[i] != k * k) return fail(kValueError, "offsets must hold k_i^2 entries");
  }
  CUDA_TRY(cudaSetDevice(c->device));
  const long long total = off[c->K];
  CUDA_TRY(dalloc(&c->d_ainv, std::max<long long>(total, 1)));
  std::vector<long long> o(off, off + c->K + 1);
  CUDA_TRY(upload(&c->d_ainv_off, o));
  c->have_asm = true;
  free_graphs(c);
  *dev_out = c->d_ainv;
  return kOk;
}

extern "C" int ddmgnn_set_pou(ddmgnn_ctx* c, int64_t n, const double* pou) {
  if (!c || !c->built) return fail(kStateError, "build must be called first");
  if (n != c->n) return fail(kValueError, "expected pou of length " + std::to_string(c->n));
  for (int64_t j = 0; j < n; ++j)
    if (!(pou[j] > 0.0)) return fail(kValueError, "pou weights must be positive");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaMemcpy(c->lay.pou, pou, sizeof(double) * n, cudaMemcpyHostToDevice));
  return kOk;
}

extern "C" int ddmgnn_local_outputs(ddmgnn_ctx* c, double** zloc, double** scale,
                                    double** r0r) {
  if (!c || !c->built) return fail(kStateError, "build must be called first");
  if (zloc) *zloc = c->d_zloc;
  if (scale) *scale = c->d_scale;
  if (r0r) *r0r = c->d_r0r;
  return kOk;
}

extern "C" int ddmgnn_spmv(ddmgnn_ctx* c, const double* x, double* y, void* stream) {
  if (!c || !c->n) return fail(kStateError, "no matrix set");
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(launch_spmv(c->sell, x, y, pick(c, stream)));
  return kOk;
}

// ------------------------------------------------------------------ PCG

// One PCG iteration (sparse.py:106-126) as stream work; level 0 = CG.
static cudaError_t enqueue_iteration(ddmgnn_ctx* c, int level, cudaStream_t s) {
  const int n = c->n;
  int* sw = &c->d_st->status;
  cudaError_t e = launch_spmv_pq(c->sell, c->d_p, c->d_q,
                                 c->d_partials, c->d_st, s);
  if (e != cudaSuccess) return e;
  e = launch_update(n, c->d_u, c->d_r, c->d_p, c->d_q, c->d_partials, c->d_st, c->d_hist,
                    level == DDMGNN_PRECOND_NONE, s);
  if (e != cudaSuccess) return e;
  const bool gnn = level == DDMGNN_LEVEL_ONE || level == DDMGNN_LEVEL_TWO;
  const bool asm_ = level == DDMGNN_ASM_ONE || level == DDMGNN_ASM_TWO;
  if ((gnn || asm_) && c->fused_tail) {
    // local solves, then the fused tail: coarse GEMV + gluing + <r, z> + beta + p update
    if (asm_) {
      e = launch_asm_local(c->K, c->lay.k_max, c->lay.sub_ptr, c->lay.idx, c->d_ainv_off,
                           c->d_ainv, c->lay.pou, c->d_r, c->d_zloc, c->d_r0r, c->d_scale, sw, s);
    } else {
      e = enqueue_gnn(c, c->d_r, sw, sw, s);
    }
    if (e != cudaSuccess) return e;
    const bool two = level == DDMGNN_LEVEL_TWO || level == DDMGNN_ASM_TWO;
    return launch_pcg_glue(n, (two ? 1 : 0) | (asm_ ? 2 : 0), c->K, c->coarse_ld, c->d_cinv,
                           c->d_r0r, c->d_y,
                           c->lay.tptr, c->lay.tent, c->lay.pou, c->d_scale, c->d_zloc, c->d_z,
                           c->d_r, c->d_p, c->d_partials, c->d_st, s);
  }
  if (level != DDMGNN_PRECOND_NONE) {
    e = enqueue_apply(c, c->d_r, c->d_z, level, sw, sw, 1, s);
    if (e != cudaSuccess) return e;
  }
  return launch_pupdate(n, c->d_p, level == DDMGNN_PRECOND_NONE ? c->d_r : c->d_z, c->d_st, s);
}

static int get_graph(ddmgnn_ctx* c, int level, cudaGraphExec_t* out) {
  const int slot = level + 6 * (c->pcg_flex ? 1 : 0);
  if (!c->graph_exec[slot]) {
    cudaGraph_t g;
    CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = enqueue_iteration(c, level, c->stream);
    cudaError_t e2 = cudaStreamEndCapture(c->stream, &g);
    if (e != cudaSuccess) return fail(kCudaError, std::string("graph capture: ") + cudaGetErrorString(e));
    if (e2 != cudaSuccess) return fail(kCudaError, std::string("graph capture: ") + cudaGetErrorString(e2));
    e = cudaGraphInstantiate(&c->graph_exec[slot], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(kCudaError, std::string("graph instantiate: ") + cudaGetErrorString(e));
  }
  *out = c->graph_exec[slot];
  return kOk;
}

static int ensure_hist(ddmgnn_ctx* c, int max_iter) {
  if (c->hist_cap < max_iter + 1) {
    const int cap = std::max(max_iter + 1, 1024);
    CUDA_TRY(dalloc(&c->d_hist, cap));
    c->hist_cap = cap;
    free_graphs(c);  // captured iterations reference the old history buffer
  }
  return kOk;
}

// Common PCG prologue: u, r, ||b||, hist[0].  Returns 1 in *early if the solve ends
// before the first iteration (sparse.py:92-99).
static int pcg_prologue(ddmgnn_ctx* c, const double* b, const double* u0, int device_ptrs,
                        double tol, int max_iter, cudaStream_t s, int* early, int* iterations,
                        double* history, int* converged, double* u_out) {
  const int n = c->n;
  const size_t bytes = sizeof(double) * n;
  const cudaMemcpyKind kin = device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  int st = ensure_hist(c, max_iter);
  if (st) return st;
  PcgState init{};
  init.tol = tol;
  init.max_iter = max_iter;
  init.flexible = c->pcg_flex;
  if (c->pcg_flex && !c->d_zold) CUDA_TRY(dalloc(&c->d_zold, n));
  *c->h_st = init;
  CUDA_TRY(cudaMemcpyAsync(c->d_st, c->h_st, sizeof(PcgState), cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(c->d_b, b, bytes, kin, s));
  if (u0) {
    CUDA_TRY(cudaMemcpyAsync(c->d_u, u0, bytes, kin, s));
    CUDA_TRY(launch_spmv(c->sell, c->d_u, c->d_q, s));
    CUDA_TRY(launch_pcg_init_u0(n, c->d_b, c->d_q, c->d_r, c->d_partials, c->d_st, c->d_hist, s));
  } else {
    CUDA_TRY(cudaMemsetAsync(c->d_u, 0, bytes, s));
    CUDA_TRY(launch_pcg_init(n, c->d_b, c->d_r, c->d_partials, c->d_st, c->d_hist, s));
  }
  CUDA_TRY(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  double h0 = 0.0;
  CUDA_TRY(cudaMemcpyAsync(&c->h_pin_a[0], c->d_hist, sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  h0 = c->h_pin_a[0];
  *early = 0;
  const cudaMemcpyKind kout = device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  if (c->h_st->nb == 0.0) {  // sparse.py:93-94
    CUDA_TRY(cudaMemsetAsync(c->d_u, 0, bytes, s));
    CUDA_TRY(cudaMemcpyAsync(u_out, c->d_u, bytes, kout, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *iterations = 0;
    history[0] = 0.0;
    *converged = 1;
    *early = 1;
    return kOk;
  }
  if (h0 < tol) {  // sparse.py:98-99
    CUDA_TRY(cudaMemcpyAsync(u_out, c->d_u, bytes, kout, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *iterations = 0;
    history[0] = h0;
    *converged = 1;
    *early = 1;
  }
  return kOk;
}

static int pcg_epilogue(ddmgnn_ctx* c, int device_ptrs, cudaStream_t s, double* u_out,
                        int* iterations, double* history, int* converged) {
  const size_t bytes = sizeof(double) * c->n;
  CUDA_TRY(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  const PcgState st = *c->h_st;
  if (st.status == kNotSpd) return fail(kRuntimeError, "matrix not SPD: <p, Ap> <= 0");
  if (st.status == kNonFiniteResidual)
    return fail(kRuntimeError, "non-finite residual at iteration " + std::to_string(st.iter + 1));
  CUDA_TRY(cudaMemcpyAsync(u_out, c->d_u, bytes,
                           device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaMemcpyAsync(history, c->d_hist, sizeof(double) * (st.iter + 1),
                           cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  *iterations = st.iter;
  *converged = st.status == kConverged;
  return kOk;
}

extern "C" int ddmgnn_pcg(ddmgnn_ctx* c, const double* b, const double* u0, double* u, double tol,
                          int max_iter, int level, int device_ptrs, void* stream, int* iterations,
                          double* history, int* converged) {
  if (!c) return fail(kValueError, "null context");
  const int flex = (level & DDMGNN_FLEXIBLE) ? 1 : 0;
  level &= ~DDMGNN_FLEXIBLE;
  int st = ready(c, level);
  if (st) return st;
  if (!(tol > 0)) return fail(kValueError, "tol must be positive");
  // the reference's loop simply does not run for max_iter < 0 (sparse.py:105)
  if (max_iter < 0) max_iter = 0;
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = pick(c, stream);
  c->pcg_flex = flex;
  int early = 0;
  st = pcg_prologue(c, b, u0, device_ptrs, tol, max_iter, s, &early, iterations, history,
                    converged, u);
  if (st || early) return st;
  const int n = c->n;
  // z0 = M r0, p0 = z0, rho0 = <r0, z0>  (sparse.py:101-103)
  if (level == DDMGNN_PRECOND_NONE) {
    CUDA_TRY(launch_rz_init(n, c->d_r, c->d_r, c->d_p, c->d_partials, c->d_st, s));
  } else {
    CUDA_TRY(cudaMemsetAsync(c->d_status, 0, sizeof(int), s));
    CUDA_TRY(enqueue_apply(c, c->d_r, c->d_z, level, c->d_status, nullptr, 0, s));
    st = check_status_word(c, s);
    if (st) return st;
    CUDA_TRY(launch_rz_init(n, c->d_r, c->d_z, c->d_p, c->d_partials, c->d_st, s));
  }
  if (max_iter > 0) {
    cudaGraphExec_t gx;
    st = get_graph(c, level, &gx);
    if (st) return st;
    const bool gnn = level == DDMGNN_LEVEL_ONE || level == DDMGNN_LEVEL_TWO;
    int done = 0, chunk = 2;
    while (!done) {
      for (int t = 0; t < chunk; ++t) {
        if (gnn) {  // the captured iteration re-fills the weight bank (see BankUse)
          BankUse use(c->device, s);
          CUDA_TRY(use.error());
          CUDA_TRY(cudaGraphLaunch(gx, s));
          CUDA_TRY(use.done());
        } else {
          CUDA_TRY(cudaGraphLaunch(gx, s));
        }
      }
      CUDA_TRY(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      done = c->h_st->status != kRunning;
      chunk = std::min(chunk * 2, 16);
    }
    if (c->h_st->status == kPrecondError) {
      // the device stopped at the failing apply; rerun it unskipped for the exact message
      CUDA_TRY(cudaMemsetAsync(c->d_status, 0, sizeof(int), s));
      CUDA_TRY(enqueue_apply(c, c->d_r, c->d_z, level, c->d_status, nullptr, 0, s));
      st = check_status_word(c, s);
      return st ? st : fail(kRuntimeError, "non-finite model state");
    }
  } else {
    c->h_st->status = kMaxIter;
    CUDA_TRY(cudaMemcpyAsync(&c->d_st->status, &c->h_st->status, sizeof(int),
                             cudaMemcpyHostToDevice, s));
  }
  return pcg_epilogue(c, device_ptrs, s, u, iterations, history, converged);
}

extern "C" int ddmgnn_pcg_host_precond(ddmgnn_ctx* c, const double* b, const double* u0,
                                       double* u, double tol, int max_iter, int flexible,
                                       ddmgnn_host_precond_fn fn, void* user, int* iterations,
                                       double* history, int* converged) {
  int st = ready(c, DDMGNN_PRECOND_NONE);
  if (st) return st;
  if (!(tol > 0)) return fail(kValueError, "tol must be positive");
  if (!fn) return fail(kValueError, "null preconditioner callback");
  if (max_iter < 0) max_iter = 0;  // sparse.py:105: the loop does not run
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  c->pcg_flex = flexible ? 1 : 0;
  int early = 0;
  st = pcg_prologue(c, b, u0, 0, tol, max_iter, s, &early, iterations, history, converged, u);
  if (st || early) return st;
  const int n = c->n;
  const size_t bytes = sizeof(double) * n;
  std::vector<double> rh(n), zh(n);
  auto host_apply = [&]() -> int {
    CUDA_TRY(cudaMemcpyAsync(rh.data(), c->d_r, bytes, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (fn(user, rh.data(), zh.data(), n) != 0)
      return fail(kRuntimeError, "preconditioner callback failed");
    CUDA_TRY(cudaMemcpyAsync(c->d_z, zh.data(), bytes, cudaMemcpyHostToDevice, s));
    return kOk;
  };
  st = host_apply();
  if (st) return st;
  CUDA_TRY(launch_rz_init(n, c->d_r, c->d_z, c->d_p, c->d_partials, c->d_st, s));
  if (max_iter == 0) {
    c->h_st->status = kMaxIter;
    CUDA_TRY(cudaMemcpyAsync(&c->d_st->status, &c->h_st->status, sizeof(int),
                             cudaMemcpyHostToDevice, s));
  }
  for (int it = 0; it < max_iter; ++it) {
    CUDA_TRY(launch_spmv_pq(c->sell, c->d_p, c->d_q, c->d_partials,
                            c->d_st, s));
    CUDA_TRY(launch_update(n, c->d_u, c->d_r, c->d_p, c->d_q, c->d_partials, c->d_st, c->d_hist,
                           0, s));
    CUDA_TRY(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (c->h_st->status != kRunning) break;
    if (c->pcg_flex)
      CUDA_TRY(cudaMemcpyAsync(c->d_zold, c->d_z, bytes, cudaMemcpyDeviceToDevice, s));
    st = host_apply();
    if (st) return st;
    // rho' = <r, z>, beta, p = z + beta p via the prolong-free path
    CUDA_TRY(launch_rz_beta(n, c->d_r, c->d_z, c->pcg_flex ? c->d_zold : nullptr, c->d_partials,
                            c->d_st, s));
    CUDA_TRY(launch_pupdate(n, c->d_p, c->d_z, c->d_st, s));
  }
  return pcg_epilogue(c, 0, s, u, iterations, history, converged);
}
