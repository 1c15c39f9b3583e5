// Fused per-subdomain DSS message-passing inference for sm_100a.
//
// Replaces the reference's batched numpy forward (pkg/src/ddmgnn/dss.py:302-329)
// together with the restriction/normalisation in front of it
// (hybrid.py:100-109) and the rescaling behind it (hybrid.py:135, s_i * sol_i).
//
// One CTA owns one subdomain for the whole chunk of message-passing layers:
//   prologue  r_i = r[idx_i] (fp64), s_i = ||r_i||_2, c_i = fp32(r_i / s_i),
//             (R0 r)_i = sum_j pou_j r_j, h = 0            (first chunk only)
//   layer l   phase A: Q_t = h_t . W1cat[d:2d]               -> SMEM (2d fp32/node)
//             phase B (thread per node s, out-edges in ascending dst order):
//                P_s  = h_s . W1cat[0:d] + b1cat
//                S_s  = sum_e relu(P_s + Q_dst(e) + [dx,dy,|d|]_e . W1cat[2d:2d+3])
//                phi  = S_s . blockdiag(W2_out, W2_in) + deg_s * [b2_out, b2_in]
//                h_s += alpha * psi([h_s, c_s, phi_out, phi_in])
//   epilogue  zloc = s_i * fp64(decoder(h))                  (last chunk only)
// This is the reference's math with the edge MLP factorised: relu(x_e W1 + b1)
// with x_e = [h_src, h_dst, dx, dy, |d|] splits into per-node products P, Q plus a
// 3-term edge part, and the second (linear) MLP layer commutes with the scatter-
// sum (dss.py:319-322), so the per-edge work is 2d*(1 add + 3 FMA + relu + add).
//
// All MLP weights of a chunk live in a 64 KB __constant__ bank at compile-time
// offsets (the layer loop is unrolled over bank slots), so weights reach the FFMAs
// as uniform-register operands loaded by LDCU.128 — no per-thread loads and no
// vector register-file pressure.  Arithmetic is FP32 CUDA-core FMA: TF32 tensor
// cores miss the 1e-5 parity bar (SURVEY.md finding 6).  ReLU propagates NaN like
// numpy.maximum (max.NaN).
#pragma once
#include <climits>

#include "ddmgnn_internal.h"
#include "gnn_cfg.h"

// Each translation unit that includes this header defines its own
//   static __constant__ float c_w[kConstFloats];
// (one 64 KB constant bank per compiled latent dimension) before the include.

namespace ddmgnn {

__device__ __forceinline__ float relu_nan(float x) {
  float y;
  asm("max.NaN.f32 %0, %1, 0f00000000;" : "=f"(y) : "f"(x));
  return y;
}

template <int N>
__device__ __forceinline__ void load_vec(const float* __restrict__ p, float (&v)[N]) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      float4 t = *reinterpret_cast<const float4*>(p + i);
      v[i] = t.x; v[i + 1] = t.y; v[i + 2] = t.z; v[i + 3] = t.w;
    }
  } else if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      float2 t = *reinterpret_cast<const float2*>(p + i);
      v[i] = t.x; v[i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = p[i];
  }
}

template <int N>
__device__ __forceinline__ void store_vec(float* __restrict__ p, const float (&v)[N]) {
  if constexpr (N % 4 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 4)
      *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  } else if constexpr (N % 2 == 0) {
#pragma unroll
    for (int i = 0; i < N; i += 2) *reinterpret_cast<float2*>(p + i) = make_float2(v[i], v[i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) p[i] = v[i];
  }
}

template <int D>
__device__ __forceinline__ void load_h(const float* p, float (&h)[D]) {
  constexpr int HS = Cfg<D>::HS;
  float t[HS];
  load_vec<HS>(p, t);
#pragma unroll
  for (int i = 0; i < D; ++i) h[i] = t[i];
}
template <int D>
__device__ __forceinline__ void store_h(float* p, const float (&h)[D]) {
  constexpr int HS = Cfg<D>::HS;
  float t[HS];
#pragma unroll
  for (int i = 0; i < HS; ++i) t[i] = i < D ? h[i] : 0.f;
  store_vec<HS>(p, t);
}

// acc[j] += sum_m x[m] * W[m][j], W at bank offset OFF with row stride RS (outer
// loop over inputs so every inner step reads consecutive constants).
template <int NIN, int NOUT, int OFF, int RS>
__device__ __forceinline__ void matvec_acc(const float (&x)[NIN], float (&acc)[NOUT]) {
#pragma unroll
  for (int m = 0; m < NIN; ++m) {
#pragma unroll
    for (int j = 0; j < NOUT; ++j) acc[j] = fmaf(x[m], c_w[OFF + m * RS + j], acc[j]);
  }
}

// Per-CTA views of the node state.  MODE 0: h, Q, c in shared memory; MODE 1: Q in
// shared memory, h and c in per-node global scratch; MODE 2: everything in global
// scratch (L1/L2 resident).  The mode is chosen per CTA from the subdomain size, so
// one launch covers every subdomain.
template <int D, int MODE>
struct NodeState {
  float* h;  // k rows of HS floats
  float* q;  // k rows of QS floats
  float* c;  // k floats
  __device__ __forceinline__ NodeState(int k, float* gq, float* gh, float* gc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if constexpr (MODE == 0) {
      q = reinterpret_cast<float*>(smem_raw);
      h = q + static_cast<size_t>(k) * Cfg<D>::QS;
      c = h + static_cast<size_t>(k) * Cfg<D>::HS;
    } else if constexpr (MODE == 1) {
      q = reinterpret_cast<float*>(smem_raw);
      h = gh;
      c = gc;
    } else {
      q = gq;
      h = gh;
      c = gc;
    }
  }
};

// One message-passing layer for the CTA's subdomain.  L is the layer's slot in
// the constant bank (compile-time, so every weight address is an immediate).
template <int D, int L, int MODE>
__device__ __noinline__ void gnn_layer(int k, float* gq, float* gh, float* gc,
                                       const float4* __restrict__ edges,
                                       const int* __restrict__ slice_off,
                                       const uint16_t* __restrict__ deg, float alpha, int* bad,
                                       int layer_no) {
  using C = Cfg<D>;
  constexpr int W = L * C::STRIDE;
  constexpr int D2 = C::D2;
  const int tid = threadIdx.x, nthr = blockDim.x;
  NodeState<D, MODE> ns(k, gq, gh, gc);
  // ---- phase A: destination projections Q_t = h_t . W1cat[d:2d] ----
  for (int n = tid; n < k; n += nthr) {
    float h[D];
    load_h<D>(ns.h + n * C::HS, h);
    float q[C::QS];
#pragma unroll
    for (int j = 0; j < C::QS; ++j) q[j] = 0.f;
    float qq[D2];
#pragma unroll
    for (int j = 0; j < D2; ++j) qq[j] = 0.f;
    matvec_acc<D, D2, W + C::OFF_WDST, C::D2P>(h, qq);
#pragma unroll
    for (int j = 0; j < D2; ++j) q[j] = qq[j];
    store_vec<C::QS>(ns.q + n * C::QS, q);
  }
  __syncthreads();
  // ---- phase B: edge aggregation + node update, thread per node ----
  int first_bad = 0;
  for (int n = tid; n < k; n += nthr) {
    float h[D];
    load_h<D>(ns.h + n * C::HS, h);
    const float cn = ns.c[n];
    float p[D2], s[D2];
#pragma unroll
    for (int j = 0; j < D2; ++j) {
      p[j] = c_w[W + C::OFF_B1 + j];
      s[j] = 0.f;
    }
    matvec_acc<D, D2, W + C::OFF_WSRC, C::D2P>(h, p);
    const int dg = deg[n];
    const float4* ep = edges + slice_off[n >> 5] + (n & 31);
    float4 rec = dg > 0 ? __ldg(ep) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int e = 0; e < dg; ++e) {
      const float4 cur = rec;
      if (e + 1 < dg) rec = __ldg(ep + 32 * (e + 1));
      const int t = __float_as_int(cur.w);
      float qt[C::QS];
      load_vec<C::QS>(ns.q + t * C::QS, qt);
#pragma unroll
      for (int j = 0; j < D2; ++j) {
        float x = p[j] + qt[j];
        x = fmaf(cur.x, c_w[W + C::OFF_WE + j], x);
        x = fmaf(cur.y, c_w[W + C::OFF_WE + C::D2P + j], x);
        x = fmaf(cur.z, c_w[W + C::OFF_WE + 2 * C::D2P + j], x);
        s[j] += relu_nan(x);
      }
    }
    // phi_out / phi_in = S . W2 + deg * b2 (linear second layer commuted with the sum)
    const float fdeg = static_cast<float>(dg);
    float x[3 * D + 1];
    float so[D], si[D], ao[D], ai[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      so[i] = s[i];
      si[i] = s[D + i];
      ao[i] = fdeg * c_w[W + C::OFF_B2O + i];
      ai[i] = fdeg * c_w[W + C::OFF_B2I + i];
    }
    matvec_acc<D, D, W + C::OFF_W2O, C::DP>(so, ao);
    matvec_acc<D, D, W + C::OFF_W2I, C::DP>(si, ai);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      x[i] = h[i];
      x[D + 1 + i] = ao[i];
      x[2 * D + 1 + i] = ai[i];
    }
    x[D] = cn;
    // psi: u = relu(x . Wp1 + bp1); o = u . Wp2 + bp2; h += alpha * o
    float u[D], o[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      u[i] = c_w[W + C::OFF_BP1 + i];
      o[i] = c_w[W + C::OFF_BP2 + i];
    }
    matvec_acc<3 * D + 1, D, W + C::OFF_WP1, C::DP>(x, u);
#pragma unroll
    for (int i = 0; i < D; ++i) u[i] = relu_nan(u[i]);
    matvec_acc<D, D, W + C::OFF_WP2, C::DP>(u, o);
    float fin = 0.f;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      h[i] = fmaf(alpha, o[i], h[i]);
      fin = fmaf(h[i], 0.f, fin);  // NaN iff some h[i] is non-finite (dss.py:324)
    }
    if (fin != 0.f && first_bad == 0) first_bad = layer_no;
    store_h<D>(ns.h + n * C::HS, h);
  }
  if (first_bad != 0 && *bad == 0) *bad = first_bad;
  __syncthreads();
}

template <int D, int L, int MODE>
struct LayerLoop {
  __device__ __forceinline__ static void run(int nl, int k, float* gq, float* gh, float* gc,
                                             const float4* edges, const int* slice_off,
                                             const uint16_t* deg, float alpha, int* bad,
                                             int layer0) {
    if constexpr (L < Cfg<D>::LMAX) {
      if (L < nl) {
        gnn_layer<D, L, MODE>(k, gq, gh, gc, edges, slice_off, deg, alpha, bad, layer0 + L);
        LayerLoop<D, L + 1, MODE>::run(nl, k, gq, gh, gc, edges, slice_off, deg, alpha, bad,
                                     layer0);
      }
    }
  }
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct GnnShared {
  double red[2][kGnnThreads / 32];
  int bad;
  double scale;
};

template <int D, int MODE>
__device__ __forceinline__ void gnn_body(const GnnArgs& a, GnnShared& sh, int sub, int pos0,
                                         int k) {
  using C = Cfg<D>;
  constexpr bool SV = MODE == 0;  // node state fully in shared memory
  const int tid = threadIdx.x, nthr = blockDim.x;
  float* gq = MODE == 2 ? a.qbuf + static_cast<size_t>(pos0) * C::QS : nullptr;
  float* gh = MODE >= 1 ? a.hbuf + static_cast<size_t>(pos0) * C::HS : nullptr;
  float* gc = MODE >= 1 ? a.cbuf + pos0 : nullptr;
  NodeState<D, MODE> ns(k, gq, gh, gc);
  double (&red)[2][kGnnThreads / 32] = sh.red;
  int& sh_bad = sh.bad;
  double& sh_scale = sh.scale;
  if (tid == 0) sh_bad = 0;

  double s;
  if (a.first) {
    // ---- restriction (hybrid.py:103-108) and coarse RHS row (R0 r)_i ----
    double* scratch = reinterpret_cast<double*>(ns.q);  // k doubles fit in k*QS floats
    double ss = 0.0, rr0 = 0.0;
    for (int n = tid; n < k; n += nthr) {
      const int g = a.idx[pos0 + n];
      const double v = a.r[g];
      ss = fma(v, v, ss);
      rr0 = fma(a.pou[g], v, rr0);
      scratch[n] = v;
    }
    ss = warp_sum(ss);
    rr0 = warp_sum(rr0);
    if ((tid & 31) == 0) {
      red[0][tid >> 5] = ss;
      red[1][tid >> 5] = rr0;
    }
    __syncthreads();
    if (tid == 0) {
      double t0 = 0.0, t1 = 0.0;
      for (int w = 0; w < (nthr >> 5); ++w) {
        t0 += red[0][w];
        t1 += red[1][w];
      }
      const double sc = sqrt(t0);
      sh_scale = sc;
      a.scale[sub] = sc;
      a.r0r[sub] = t1;
    }
    __syncthreads();
    s = sh_scale;
    if (s == 0.0) {  // zero local residual: the subdomain contributes nothing
      if (tid == 0) {
        a.bad_layer[sub] = 0;
        a.out_bad[sub] = 0;
      }
      return;
    }
    for (int n = tid; n < k; n += nthr) {
      const float c = static_cast<float>(scratch[n] / s);
      ns.c[n] = c;
      if (SV && !a.last) a.cbuf[pos0 + n] = c;
    }
    __syncthreads();  // scratch (aliasing Q) fully consumed
    for (int n = tid; n < k; n += nthr) {
      float z[D];
#pragma unroll
      for (int i = 0; i < D; ++i) z[i] = 0.f;
      store_h<D>(ns.h + n * C::HS, z);
    }
  } else {
    s = a.scale[sub];
    if (s == 0.0) return;
    if constexpr (SV) {
      for (int n = tid; n < k; n += nthr) {
        ns.c[n] = a.cbuf[pos0 + n];
        float hv[D];
        load_h<D>(a.hbuf + static_cast<size_t>(pos0 + n) * C::HS, hv);
        store_h<D>(ns.h + n * C::HS, hv);
      }
    }
  }
  __syncthreads();

  LayerLoop<D, 0, MODE>::run(a.nl, k, gq, gh, gc, a.edges, a.slice_off + a.slice_base[sub],
                           a.deg + pos0, a.alpha, &sh_bad, a.layer0);

  int outbad = 0;
  if (a.last) {
    // ---- decoder of the final layer (dss.py:327) and rescaling (hybrid.py:135) ----
    for (int n = tid; n < k; n += nthr) {
      float h[D];
      load_h<D>(ns.h + n * C::HS, h);
      float u[D];
#pragma unroll
      for (int i = 0; i < D; ++i) u[i] = c_w[C::DEC_B1 + i];
      matvec_acc<D, D, C::DEC_W1, C::DP>(h, u);
      float o = c_w[C::DEC_B2];
#pragma unroll
      for (int i = 0; i < D; ++i) o = fmaf(relu_nan(u[i]), c_w[C::DEC_W2 + i], o);
      if (!isfinite(o)) outbad = 1;
      a.zloc[pos0 + n] = s * static_cast<double>(o);
    }
  } else if constexpr (SV) {
    for (int n = tid; n < k; n += nthr) {
      float hv[D];
      load_h<D>(ns.h + n * C::HS, hv);
      store_h<D>(a.hbuf + static_cast<size_t>(pos0 + n) * C::HS, hv);
    }
  }
  outbad = __syncthreads_or(outbad);
  if (tid == 0) {
    const int b = sh_bad;
    if (a.first) {
      a.bad_layer[sub] = b;
      a.out_bad[sub] = outbad;
    } else {
      if (b != 0 && a.bad_layer[sub] == 0) a.bad_layer[sub] = b;
      if (outbad) a.out_bad[sub] = 1;
    }
    if (b != 0 || outbad) atomicMax(a.status, static_cast<int>(kPrecondError));
  }
}

// One CTA per subdomain (LPT order); the node-state placement is chosen per CTA:
// a.cap0 = largest k with h, Q, c in the launch's shared memory, a.cap1 = largest
// k with Q alone in shared memory.
template <int D>
__global__ void __launch_bounds__(kGnnThreads, 1) gnn_kernel(GnnArgs a) {
  if (a.skip != nullptr && *a.skip != 0) return;
  __shared__ GnnShared sh;
  const int sub = a.order[a.order_begin + blockIdx.x];
  const int pos0 = a.sub_ptr[sub];
  const int k = a.sub_ptr[sub + 1] - pos0;
  if (k <= a.cap0) {
    gnn_body<D, 0>(a, sh, sub, pos0, k);
  } else if (k <= a.cap1) {
    gnn_body<D, 1>(a, sh, sub, pos0, k);
  } else {
    gnn_body<D, 2>(a, sh, sub, pos0, k);
  }
}

}  // namespace ddmgnn
