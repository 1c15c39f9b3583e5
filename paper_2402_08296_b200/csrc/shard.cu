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
#include <algorithm>
#include <cmath>
#include <cstring>

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
  return cuda_status(launch_coarse_gemv(static_cast<int>(k), static_cast<int>(k), a, x, y, nullptr,
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

// ---------------------------------------------------------------- peer collectives
// Device-resident exchanges between the ranks' GPUs over peer memory (CUDA IPC
// mappings; NVLink/NVSwitch between the GPUs of one box), ordered by device flags
// only, so every call is stream-ordered and graph-capturable (no host barrier).
// Every rank owns a flag block int64[DDMGNN_PEER_FLAG_WORDS] (zeroed, mapped by all);
// channel c occupies words [32 c, 32 c + 32):
//   sig[h]  (+0..7)   epoch of the last message rank h delivered to this rank
//   ack[h]  (+8..15)  epoch of the last message of this rank that rank h consumed
//   ctr     (+16)     this rank's epoch counter of the channel (bumped by the sender side)
//   done[h] (+17..24) block-completion counters of the multi-block kernels
//   fin     (+25)     completion counter over all destination slices
// Every rank makes the same sequence of calls per channel, so the counters agree.
// Before overwriting a peer's receive buffer with epoch e the sender waits for the
// peer's acknowledgement of e - 1; the receiver acknowledges after consuming.
namespace ddmgnn {
namespace {

constexpr int kPeerMax = DDMGNN_PEER_MAX;
constexpr int kChanWords = 32;
enum { kSig = 0, kAck = 8, kCtr = 16, kDone = 17, kFin = 25 };
constexpr int kErrWord = DDMGNN_PEER_FLAG_WORDS - 1;  // in channel 7's spare words

struct PeerArgs {
  long long* flags[kPeerMax];  // rank h's flag block (this rank's own at [me])
  double* buf[kPeerMax];       // per-rank destination base (put: receive buffer of h)
  long long off[kPeerMax + 1]; // segment offsets (send side: into idx; recv side: into recv)
  long long doff[kPeerMax];    // put: offset of this rank's segment in h's receive buffer
  int g, me, chan;
};

__device__ __forceinline__ long long ld_acq(const long long* p) {
  long long v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(long long* p, long long v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Spin until *p >= v.  A peer that never arrives (a rank that died or diverged)
// does not hang the GPU: after kPeerTimeoutNs the wait gives up and raises the
// rank's error word (flags[kErrWord]), which the host checks at its status polls.
constexpr unsigned long long kPeerTimeoutNs = 30ull * 1000 * 1000 * 1000;
__device__ __forceinline__ void wait_geq(const long long* p, long long v, long long* err) {
  if (ld_acq(p) >= v) return;
  const unsigned long long t0 = globaltimer();
  while (ld_acq(p) < v) {
    __nanosleep(200);
    if (globaltimer() - t0 > kPeerTimeoutNs) {
      atomicExch(reinterpret_cast<unsigned long long*>(err), 1ull);
      return;
    }
  }
}
__device__ __forceinline__ long long* chan_of(const PeerArgs& a, int h) {
  return a.flags[h] + a.chan * kChanWords;
}

// grid (x blocks, g slices): slice h copies src[idx[off[h] .. off[h+1])] into
// buf[h] + doff[h]; the last block of a slice signals h; the last slice bumps ctr.
__global__ void __launch_bounds__(kT) peer_put_kernel(const double* __restrict__ src,
                                                       const int* __restrict__ idx, PeerArgs a) {
  long long* my = chan_of(a, a.me);
  const int h = blockIdx.y;
  const long long b0 = a.off[h], cnt = a.off[h + 1] - b0;
  const long long e = ld_acq(my + kCtr) + 1;
  const bool send = cnt > 0 && h != a.me;
  if (send) {
    if (threadIdx.x == 0) wait_geq(my + kAck + h, e - 1, a.flags[a.me] + kErrWord);  // h consumed e - 1
    __syncthreads();
    double* dst = a.buf[h] + a.doff[h];
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < cnt;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
      dst[i] = src[idx[b0 + i]];
    __threadfence_system();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long d =
        atomicAdd(reinterpret_cast<unsigned long long*>(my + kDone + h), 1ull);
    if (d == gridDim.x - 1) {  // last block of slice h
      my[kDone + h] = 0;
      if (send) {
        __threadfence_system();
        st_rel(chan_of(a, h) + kSig + a.me, e);
      }
      __threadfence();
      const unsigned long long f =
          atomicAdd(reinterpret_cast<unsigned long long*>(my + kFin), 1ull);
      if (f == gridDim.y - 1) {  // every slice done: every block has read ctr
        my[kFin] = 0;
        __threadfence();
        st_rel(my + kCtr, e);
      }
    }
  }
}

// Wait for epoch ctr from every rank with a non-empty segment, then (pos != null)
// ext[pos[i]] = recv[i]; with `ack`, the last block acknowledges to the senders.
__global__ void __launch_bounds__(kT) peer_wait_kernel(const double* __restrict__ recv,
                                                        const int* __restrict__ pos, long long n,
                                                        double* __restrict__ ext, int ack,
                                                        PeerArgs a) {
  long long* my = chan_of(a, a.me);
  const long long e = ld_acq(my + kCtr);  // the sender side of this call site bumped it
  const int h = threadIdx.x;
  if (h < a.g && h != a.me && a.off[h + 1] > a.off[h])
    wait_geq(my + kSig + h, e, a.flags[a.me] + kErrWord);
  __syncthreads();
  if (pos != nullptr)
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
      ext[pos[i]] = __ldcg(recv + i);  // written by peers: bypass L1
  if (!ack) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long d =
        atomicAdd(reinterpret_cast<unsigned long long*>(my + kDone), 1ull);
    if (d == gridDim.x - 1) {
      my[kDone] = 0;
      for (int s = 0; s < a.g; ++s)
        if (s != a.me && a.off[s + 1] > a.off[s]) st_rel(chan_of(a, s) + kAck + a.me, e);
    }
  }
}

// acknowledgement alone (receive buffer consumed by a later kernel)
__global__ void peer_ack_kernel(PeerArgs a) {
  long long* my = chan_of(a, a.me);
  const long long e = ld_acq(my + kCtr);
  const int s = threadIdx.x;
  if (s < a.g && s != a.me && a.off[s + 1] > a.off[s]) st_rel(chan_of(a, s) + kAck + a.me, e);
}

// All-gather of k doubles per rank into every rank's out (= buf[h], layout [g][k]);
// with `reduce`, out[0..k) of this rank = sum over ranks in rank order (buf[h] are
// then g x k slot areas) — identical bits on every rank.  One block.
__global__ void __launch_bounds__(kT) peer_gather_kernel(const double* __restrict__ in,
                                                          long long k, double* out, int reduce,
                                                          PeerArgs a) {
  long long* my = chan_of(a, a.me);
  const long long e = ld_acq(my + kCtr) + 1;
  __shared__ double vin[16];
  if (reduce && threadIdx.x < k) vin[threadIdx.x] = in[threadIdx.x];
  __syncthreads();
  for (int h = 0; h < a.g; ++h) {
    if (h != a.me) {
      if (threadIdx.x == 0) wait_geq(my + kAck + h, e - 1, a.flags[a.me] + kErrWord);
      __syncthreads();
    }
    double* dst = a.buf[h] + static_cast<long long>(a.me) * k;
    for (long long j = threadIdx.x; j < k; j += blockDim.x) dst[j] = reduce ? vin[j] : in[j];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < a.g && threadIdx.x != a.me) st_rel(chan_of(a, threadIdx.x) + kSig + a.me, e);
  if (threadIdx.x < a.g && threadIdx.x != a.me)
    wait_geq(my + kSig + threadIdx.x, e, a.flags[a.me] + kErrWord);
  __syncthreads();
  if (reduce) {
    const double* slots = a.buf[a.me];
    if (threadIdx.x < k) {
      double acc = 0.0;
      for (int h = 0; h < a.g; ++h) acc += __ldcg(slots + h * k + threadIdx.x);
      out[threadIdx.x] = acc;
    }
  }
  __syncthreads();  // this rank's slots / out read before the acknowledgement
  if (threadIdx.x < a.g && threadIdx.x != a.me) st_rel(chan_of(a, threadIdx.x) + kAck + a.me, e);
  if (threadIdx.x == 0) st_rel(my + kCtr, e);
}

int fill_peer(PeerArgs* a, int g, int me, int chan, int64_t* const* flags) {
  if (g < 1 || g > kPeerMax || me < 0 || me >= g || chan < 0 || chan >= DDMGNN_PEER_CHANNELS)
    return kValueError;
  *a = PeerArgs{};
  a->g = g;
  a->me = me;
  a->chan = chan;
  for (int h = 0; h < g; ++h) a->flags[h] = reinterpret_cast<long long*>(flags[h]);
  return 0;
}

}  // namespace
}  // namespace ddmgnn

extern "C" int ddmgnn_peer_put(int g, int me, int chan, int64_t* const* flags, const double* src,
                               const int32_t* idx, const int64_t* send_off, double* const* dst,
                               const int64_t* dst_off, void* stream) {
  PeerArgs a;
  if (fill_peer(&a, g, me, chan, flags)) return kValueError;
  long long mx = 0;
  for (int h = 0; h <= g; ++h) a.off[h] = send_off[h];
  for (int h = 0; h < g; ++h) {
    a.buf[h] = dst[h];
    a.doff[h] = dst_off[h];
    mx = std::max<long long>(mx, send_off[h + 1] - send_off[h]);
  }
  const int bx = std::max(1, std::min(64, static_cast<int>((mx + kT - 1) / kT)));
  peer_put_kernel<<<dim3(bx, g), kT, 0, static_cast<cudaStream_t>(stream)>>>(src, idx, a);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_peer_wait(int g, int me, int chan, int64_t* const* flags,
                                const int64_t* recv_off, const double* recv, const int32_t* pos,
                                double* ext, int ack, void* stream) {
  PeerArgs a;
  if (fill_peer(&a, g, me, chan, flags)) return kValueError;
  for (int h = 0; h <= g; ++h) a.off[h] = recv_off[h];
  const long long n = recv_off[g];
  const int nb = pos ? std::max(1, std::min(64, static_cast<int>((n + kT - 1) / kT))) : 1;
  peer_wait_kernel<<<nb, kT, 0, static_cast<cudaStream_t>(stream)>>>(recv, pos, n, ext, ack, a);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_peer_ack(int g, int me, int chan, int64_t* const* flags,
                               const int64_t* recv_off, void* stream) {
  PeerArgs a;
  if (fill_peer(&a, g, me, chan, flags)) return kValueError;
  for (int h = 0; h <= g; ++h) a.off[h] = recv_off[h];
  peer_ack_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_peer_allgather(int g, int me, int chan, int64_t* const* flags,
                                     double* const* out, const double* in, int64_t k,
                                     void* stream) {
  PeerArgs a;
  if (fill_peer(&a, g, me, chan, flags) || k < 0) return kValueError;
  for (int h = 0; h < g; ++h) a.buf[h] = out[h];
  peer_gather_kernel<<<1, kT, 0, static_cast<cudaStream_t>(stream)>>>(in, k, nullptr, 0, a);
  return cuda_status(cudaGetLastError());
}

extern "C" int ddmgnn_peer_allreduce(int g, int me, int chan, int64_t* const* flags,
                                     double* const* slots, double* inout, int k, void* stream) {
  PeerArgs a;
  if (fill_peer(&a, g, me, chan, flags) || k < 1 || k > 16) return kValueError;
  for (int h = 0; h < g; ++h) a.buf[h] = slots[h];
  peer_gather_kernel<<<1, kT, 0, static_cast<cudaStream_t>(stream)>>>(inout, k, inout, 1, a);
  return cuda_status(cudaGetLastError());
}

// Peer-visible device buffers and their CUDA IPC handles (the exchange arenas of
// paper_2402_08296_b200/sharded.py): cudaMalloc'd directly so that a handle names
// exactly the buffer; opened with lazy peer access from the calling rank's device.
extern "C" int ddmgnn_peer_alloc(int device, int64_t bytes, void** ptr) {
  if (!ptr || bytes < 0) return kValueError;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(ptr, std::max<int64_t>(bytes, 8));
  if (e == cudaSuccess) e = cudaMemset(*ptr, 0, std::max<int64_t>(bytes, 8));
  return cuda_status(e);
}

extern "C" int ddmgnn_peer_free(void* ptr) { return cuda_status(cudaFree(ptr)); }

extern "C" int ddmgnn_ipc_get(void* ptr, unsigned char* handle) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e == cudaSuccess) memcpy(handle, &h, sizeof(h));
  return cuda_status(e);
}

extern "C" int ddmgnn_ipc_open(int device, const unsigned char* handle, void** ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return cuda_status(e);
}

extern "C" int ddmgnn_ipc_close(void* ptr) { return cuda_status(cudaIpcCloseMemHandle(ptr)); }
