// Fused per-subdomain DSS message-passing inference for sm_100a.
//
// Replaces the reference's batched numpy forward (pkg/src/ddmgnn/dss.py:302-329)
// together with the restriction/normalisation in front of it
// (hybrid.py:100-109) and the rescaling behind it (hybrid.py:135, s_i * sol_i).
//
// One CTA owns one subdomain for the whole chunk of message-passing layers:
//   prologue  r_i = r[idx_i] (fp64), s_i = ||r_i||_2, c_i = fp32(r_i / s_i),
//             (R0 r)_i = sum_j pou_j r_j, h = 0            (first chunk only)
//   layer l   phase A (thread per node t):  Q_t = [h_t, x_t, y_t] . WQ   -> SMEM
//             phase B (thread per node s, out-edges in ascending dst order):
//                P_s  = b1 + [h_s, x_s, y_s] . WP
//                S2_s = sum_e 2 relu(P_s + Q_dst(e) + |d|_e WL)
//                u    = 2 relu(bp1 + deg_s bdeg + [h_s, c_s] . Wp1[h,c] + S2_s . M)
//                h_s += alpha (bp2 + u . (Wp2 / 2))
//   epilogue  zloc = s_i * fp64(decoder(h))                  (last chunk only)
//
// This is the reference's arithmetic rewritten without changing its value in
// exact arithmetic (fp32 rounding differs by O(1e-7); SURVEY.md §8a / DESIGN.md §4):
//  * edge MLP factorised: relu(x_e W1 + b1) with x_e = [h_src, h_dst, dx, dy, |d|]
//    and (dx, dy) = xy_dst - xy_src (dss.py:184, subdomain-centred coordinates),
//    so per edge only P_s + Q_t + |d| WL remains (dss.py:316-318);
//  * the messages' second (linear) layer commutes with the scatter-sum
//    (dss.py:319-322) and is folded into psi's first layer (M = W2 . Wp1[phi rows],
//    bdeg = b2 . Wp1[phi rows] per unit degree);
//  * relu(x) = (x + |x|) / 2 — one packed FADD2 with an |.| operand instead of two
//    FMNMX; the 1/2 is folded into M and Wp2.  NaN propagates like numpy.maximum.
// All per-pair arithmetic is packed f32x2 (FFMA2/FADD2: two FP32 lanes per issue
// slot), with the weight pair as a uniform-register operand loaded by LDCU.128
// from a 64 KB __constant__ bank (layer slot = uniform base register + immediate).
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

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 bcast(float x) { return make_float2(x, x); }
// 2 relu(x) elementwise: x + |x| (exact; NaN stays NaN)
__device__ __forceinline__ float2 relu2x(float2 x) {
  return fadd2(x, make_float2(fabsf(x.x), fabsf(x.y)));
}
__device__ __forceinline__ float2 cpair(int off) {
  return *reinterpret_cast<const float2*>(&c_w[off]);
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

// acc[j] += sum_m x[m] * W[m][2j:2j+2], W at bank offset base + OFF with row stride
// RS.  `base` is warp-uniform (the layer's slot), so every weight pair is one
// uniform-register-addressed constant load feeding a packed FFMA2.
template <int NIN, int NPO, int OFF, int RS>
__device__ __forceinline__ void mv2(int base, const float (&x)[NIN], float2 (&acc)[NPO]) {
#pragma unroll
  for (int m = 0; m < NIN; ++m) {
#pragma unroll
    for (int j = 0; j < NPO; ++j)
      acc[j] = ffma2(bcast(x[m]), cpair(base + OFF + m * RS + 2 * j), acc[j]);
  }
}

// The same for NPT nodes at once: every weight pair (one LDCU) feeds NPT FFMA2.
template <int NPT, int NIN, int NPO, int OFF, int RS>
__device__ __forceinline__ void mv2n(int base, const float (&x)[NPT][NIN],
                                     float2 (&acc)[NPT][NPO]) {
#pragma unroll
  for (int m = 0; m < NIN; ++m) {
#pragma unroll
    for (int j = 0; j < NPO; ++j) {
      const float2 w = cpair(base + OFF + m * RS + 2 * j);
#pragma unroll
      for (int t = 0; t < NPT; ++t) acc[t][j] = ffma2(bcast(x[t][m]), w, acc[t][j]);
    }
  }
}

// [h (D), x, y] of a node: h from the node state, (x, y) subdomain-centred coordinates.
template <int D>
__device__ __forceinline__ void load_hxy(const float* hrow, float2 xy, float (&v)[D + 2]) {
  constexpr int DH = Cfg<D>::DH;
  float t[DH];
  load_vec<DH>(hrow, t);
#pragma unroll
  for (int i = 0; i < D; ++i) v[i] = t[i];
  v[D] = xy.x;
  v[D + 1] = xy.y;
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
      h = q + static_cast<size_t>(k + 1) * Cfg<D>::QS;  // Q rows 0..k (k = dummy)
      c = h + static_cast<size_t>(k + 1) * Cfg<D>::HS;  // h rows 0..k (k = dummy)
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

// Warp-uniform value (lane 0's): lets ptxas keep loop bounds and the layer's bank
// offset in uniform registers, so weight pairs are LDCU.128 c[bank][UR + imm]
// operands of FFMA2 even inside the node loops.
__device__ __forceinline__ int uni(int v) { return __shfl_sync(0xffffffffu, v, 0); }

// One message-passing layer for the CTA's subdomain.  WT >= 0: the layer's slot
// offset in the constant bank as a compile-time constant (every weight pair is an
// immediate-addressed LDCU.128 feeding FFMA2 — the fast path); WT < 0: runtime
// offset w_rt (used only by the rare big-subdomain kernel).
//
// Node loops run a uniform trip count: each warp handles NPT consecutive SELL
// slices (32 local nodes each) per iteration, node t of lane = n0 + 32 t + lane,
// so one weight load feeds NPT nodes.  Slice widths (max degree in the slice)
// bound the edge loop; padding records point at the dummy Q row k (all -1e30),
// whose 2 relu term is exactly 0.  Lanes past k recompute node k-1 (phase A,
// identical store) or write the dummy h row k (phase B): no divergent branches,
// so the weight loads stay uniform.
template <int D, int MODE, int WT, int NPT>
__device__ __forceinline__ void gnn_layer(int w_rt, int k, int warp, float* gq, float* gh,
                                          float* gc, const float2* __restrict__ xy,
                                          const float2* __restrict__ edges,
                                          const int* __restrict__ slice_off,
                                          const uint16_t* __restrict__ deg, float alpha,
                                          int* bad, int layer_no) {
  using C = Cfg<D>;
  const int W = WT >= 0 ? WT : w_rt;
  constexpr int NP2 = C::NP2, NPH = C::NPH;
  const int lane = threadIdx.x & 31, nthr = blockDim.x;
  const int step = NPT * nthr;
  NodeState<D, MODE> ns(k, gq, gh, gc);
  // ---- phase A: destination projections Q_t = [h_t, x_t, y_t] . WQ ----
  for (int n0 = 32 * NPT * warp; n0 < k; n0 += step) {
    float hin[NPT][D + 2];
    int nn[NPT];
#pragma unroll
    for (int t = 0; t < NPT; ++t) {
      nn[t] = min(n0 + 32 * t + lane, k - 1);
      load_hxy<D>(ns.h + nn[t] * C::HS, __ldg(xy + nn[t]), hin[t]);
    }
    float2 q[NPT][NP2];
#pragma unroll
    for (int t = 0; t < NPT; ++t)
#pragma unroll
      for (int j = 0; j < NP2; ++j) q[t][j] = make_float2(0.f, 0.f);
    mv2n<NPT, D + 2, NP2, C::OFF_WQ, C::D2P>(W, hin, q);
#pragma unroll
    for (int t = 0; t < NPT; ++t) {
      float qs[C::QS];
#pragma unroll
      for (int j = 0; j < C::QS; ++j) qs[j] = 0.f;
#pragma unroll
      for (int j = 0; j < NP2; ++j) {
        qs[2 * j] = q[t][j].x;
        qs[2 * j + 1] = q[t][j].y;
      }
      store_vec<C::QS>(ns.q + nn[t] * C::QS, qs);
    }
  }
  __syncthreads();
  // ---- phase B: edge aggregation + node update ----
  int first_bad = 0;
  const float2 dummy = make_float2(0.f, __int_as_float(k));
  for (int n0 = 32 * NPT * warp; n0 < k; n0 += step) {
    int nn[NPT], width[NPT];
    float2 p[NPT][NP2], s[NPT][NP2];
    const float2* ep[NPT];
    {
      float hin[NPT][D + 2];
#pragma unroll
      for (int t = 0; t < NPT; ++t) {
        nn[t] = min(n0 + 32 * t + lane, k - 1);
        load_hxy<D>(ns.h + nn[t] * C::HS, __ldg(xy + nn[t]), hin[t]);
#pragma unroll
        for (int j = 0; j < NP2; ++j) {
          p[t][j] = cpair(W + C::OFF_B1 + 2 * j);
          s[t][j] = make_float2(0.f, 0.f);
        }
      }
      mv2n<NPT, D + 2, NP2, C::OFF_WP, C::D2P>(W, hin, p);
    }
    int wmax = 0;
#pragma unroll
    for (int t = 0; t < NPT; ++t) {
      const int q = (n0 >> 5) + t;
      const bool live = n0 + 32 * t < k;  // warp-uniform
      const int so = uni(slice_off[live ? q : 0]);
      width[t] = live ? (uni(slice_off[q + 1]) - so) >> 5 : 0;
      ep[t] = edges + so + lane;
      wmax = max(wmax, width[t]);
    }
    float2 rec[NPT];
#pragma unroll
    for (int t = 0; t < NPT; ++t) rec[t] = width[t] > 0 ? __ldg(ep[t]) : dummy;
    for (int e = 0; e < wmax; ++e) {
      float2 cur[NPT];
#pragma unroll
      for (int t = 0; t < NPT; ++t) {
        cur[t] = rec[t];
        rec[t] = e + 1 < width[t] ? __ldg(ep[t] + 32 * (e + 1)) : dummy;
      }
#pragma unroll
      for (int t = 0; t < NPT; ++t) {
        float qt[C::QS];
        load_vec<C::QS>(ns.q + __float_as_int(cur[t].y) * C::QS, qt);
        const float2 len = bcast(cur[t].x);
#pragma unroll
        for (int j = 0; j < NP2; ++j) {
          float2 x = fadd2(p[t][j], make_float2(qt[2 * j], qt[2 * j + 1]));
          x = ffma2(len, cpair(W + C::OFF_WL + 2 * j), x);
          s[t][j] = fadd2(s[t][j], relu2x(x));
        }
      }
    }
    // psi first layer with the messages' second layer folded in
    float2 u[NPT][NPH];
    float hc[NPT][D + 2];
#pragma unroll
    for (int t = 0; t < NPT; ++t) {
#pragma unroll
      for (int j = 0; j < NPH; ++j) u[t][j] = cpair(W + C::OFF_BP1 + 2 * j);
      float hv[C::DH];
      load_vec<C::DH>(ns.h + nn[t] * C::HS, hv);
#pragma unroll
      for (int i = 0; i < D; ++i) hc[t][i] = hv[i];
      hc[t][D] = ns.c[nn[t]];
      hc[t][D + 1] = static_cast<float>(deg[nn[t]]);
    }
    mv2n<NPT, D + 2, NPH, C::OFF_WU, C::DP>(W, hc, u);
    {
      float sv[NPT][2 * D];
#pragma unroll
      for (int t = 0; t < NPT; ++t)
#pragma unroll
        for (int j = 0; j < NP2; ++j) {
          sv[t][2 * j] = s[t][j].x;
          sv[t][2 * j + 1] = s[t][j].y;
        }
      // second, independent accumulator chain for the message part (ILP)
      float2 u2[NPT][NPH];
#pragma unroll
      for (int t = 0; t < NPT; ++t)
#pragma unroll
        for (int j = 0; j < NPH; ++j) u2[t][j] = make_float2(0.f, 0.f);
      mv2n<NPT, 2 * D, NPH, C::OFF_WU + (D + 2) * C::DP, C::DP>(W, sv, u2);
#pragma unroll
      for (int t = 0; t < NPT; ++t)
#pragma unroll
        for (int j = 0; j < NPH; ++j) u[t][j] = fadd2(u[t][j], u2[t][j]);
    }
    float uv[NPT][D];
    float2 o[NPT][NPH];
#pragma unroll
    for (int t = 0; t < NPT; ++t)
#pragma unroll
      for (int j = 0; j < NPH; ++j) {
        const float2 r2 = relu2x(u[t][j]);
        if (2 * j < D) uv[t][2 * j] = r2.x;
        if (2 * j + 1 < D) uv[t][2 * j + 1] = r2.y;
        o[t][j] = cpair(W + C::OFF_BP2 + 2 * j);
      }
    mv2n<NPT, D, NPH, C::OFF_WP2, C::DP>(W, uv, o);
    const float2 al = bcast(alpha);
#pragma unroll
    for (int t = 0; t < NPT; ++t) {
      const int n = n0 + 32 * t + lane;
      float hn[C::DH];
      float2 fin = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < NPH; ++j) {
        float2 hp = make_float2(hc[t][2 * j], 2 * j + 1 < D ? hc[t][2 * j + 1] : 0.f);
        hp = ffma2(al, o[t][j], hp);
        fin = ffma2(hp, make_float2(0.f, 0.f), fin);  // NaN iff some h is non-finite (dss.py:324)
        hn[2 * j] = hp.x;
        hn[2 * j + 1] = (2 * j + 1 < D) ? hp.y : 0.f;
      }
      if ((fin.x != 0.f || fin.y != 0.f) && first_bad == 0 && n < k) first_bad = layer_no;
      // every thread of the warp has read its nodes' h above (same iteration), so the
      // in-place update cannot race; lanes past k write the dummy row k
      store_vec<C::DH>(ns.h + min(n, k) * C::HS, hn);
    }
  }
  if (first_bad != 0 && *bad == 0) *bad = first_bad;
  __syncthreads();
}

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

template <int D, int MODE, bool SLOTS, int NPT>
__device__ __forceinline__ void gnn_body(const GnnArgs& a, GnnShared& sh, int sub, int pos0,
                                         int k) {
  using C = Cfg<D>;
  constexpr bool SV = MODE == 0;  // node state fully in shared memory
  const int tid = threadIdx.x, nthr = blockDim.x;
  // global Q scratch keeps one extra (dummy) row per subdomain
  float* gq = MODE == 2 ? a.qbuf + static_cast<size_t>(pos0 + sub) * C::QS : nullptr;
  float* gh = MODE >= 1 ? a.hbuf + static_cast<size_t>(pos0 + sub) * C::HS : nullptr;
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
    s = __shfl_sync(0xffffffffu, sh_scale, 0);
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
      float z[C::DH];
#pragma unroll
      for (int i = 0; i < C::DH; ++i) z[i] = 0.f;
      store_vec<C::DH>(ns.h + n * C::HS, z);
    }
  } else {
    s = __shfl_sync(0xffffffffu, a.scale[sub], 0);
    if (s == 0.0) return;
    if constexpr (SV) {
      for (int n = tid; n < k; n += nthr) {
        ns.c[n] = a.cbuf[pos0 + n];
        float hv[C::DH];
        load_vec<C::DH>(a.hbuf + static_cast<size_t>(pos0 + sub + n) * C::HS, hv);
        store_vec<C::DH>(ns.h + n * C::HS, hv);
      }
    }
  }
  // dummy Q row k: target of the SELL padding records (2 relu(P - 1e30) == 0)
  for (int j = tid; j < C::QS; j += nthr) ns.q[static_cast<size_t>(k) * C::QS + j] = -1e30f;
  __syncthreads();

  {
    const int warp = uni(tid >> 5);
    const float2* xy = a.xy + pos0;
    const int* so = a.slice_off + a.slice_base[sub];
    const uint16_t* dg = a.deg + pos0;
    if constexpr (SLOTS) {
      // compile-time bank slots (LMAX <= 10)
#define DDM_LAYER(LL)                                                                        \
  if constexpr (LL < C::LMAX) {                                                              \
    if (LL < a.nl)                                                                           \
      gnn_layer<D, MODE, LL * C::STRIDE, NPT>(0, k, warp, gq, gh, gc, xy, a.edges, so, dg, a.alpha, \
                                         &sh_bad, a.layer0 + LL);                            \
  }
      DDM_LAYER(0) DDM_LAYER(1) DDM_LAYER(2) DDM_LAYER(3) DDM_LAYER(4)
      DDM_LAYER(5) DDM_LAYER(6) DDM_LAYER(7) DDM_LAYER(8) DDM_LAYER(9)
#undef DDM_LAYER
    } else {
#pragma unroll 1
      for (int l = 0; l < a.nl; ++l)
        gnn_layer<D, MODE, -1, NPT>(l * C::STRIDE, k, warp, gq, gh, gc, xy, a.edges, so, dg, a.alpha,
                               &sh_bad, a.layer0 + l);
    }
  }

  int outbad = 0;
  if (a.last) {
    // ---- decoder of the final layer (dss.py:327) and rescaling (hybrid.py:135) ----
    for (int n = tid; n < k; n += nthr) {
      float hv[C::DH];
      load_vec<C::DH>(ns.h + n * C::HS, hv);
      float h[D];
#pragma unroll
      for (int i = 0; i < D; ++i) h[i] = hv[i];
      float2 u[C::NPH];
#pragma unroll
      for (int j = 0; j < C::NPH; ++j) u[j] = cpair(C::DEC_B1 + 2 * j);
      mv2<D, C::NPH, C::DEC_W1, C::DP>(0, h, u);
      float o = c_w[C::DEC_B2];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const float ui = (i & 1) ? u[i >> 1].y : u[i >> 1].x;
        o = fmaf(relu_nan(ui), c_w[C::DEC_W2 + i], o);
      }
      if (!isfinite(o)) outbad = 1;
      a.zloc[pos0 + n] = s * static_cast<double>(o);
    }
  } else if constexpr (SV) {
    for (int n = tid; n < k; n += nthr) {
      float hv[C::DH];
      load_vec<C::DH>(ns.h + n * C::HS, hv);
      store_vec<C::DH>(a.hbuf + static_cast<size_t>(pos0 + sub + n) * C::HS, hv);
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

// Subdomains whose node state (h, Q, c) fits the launch's shared memory (k <=
// a.cap0): one CTA per subdomain in LPT order, compile-time bank slots.
template <int D>
__global__ void __launch_bounds__(kGnnThreads / kGnnNpt, 1) gnn_kernel(GnnArgs a) {
  if (a.skip != nullptr && uni(*a.skip) != 0) return;
  __shared__ GnnShared sh;
  const int sub = uni(a.order[a.order_begin + blockIdx.x]);
  const int pos0 = uni(a.sub_ptr[sub]);
  const int k = uni(a.sub_ptr[sub + 1] - pos0);
  gnn_body<D, 0, true, kGnnNpt>(a, sh, sub, pos0, k);
}

// The few oversized subdomains (k > a.cap0): Q alone in shared memory (k <= a.cap1,
// compile-time bank slots) or everything in global scratch (runtime bank slots).  Launched concurrently with
// gnn_kernel on a side stream (gnn.cu).
template <int D>
__global__ void __launch_bounds__(kGnnThreads, 1) gnn_big_kernel(GnnArgs a) {
  if (a.skip != nullptr && uni(*a.skip) != 0) return;
  __shared__ GnnShared sh;
  const int sub = uni(a.order[a.order_begin + blockIdx.x]);
  const int pos0 = uni(a.sub_ptr[sub]);
  const int k = uni(a.sub_ptr[sub + 1] - pos0);
  if (k <= a.cap1) {
    gnn_body<D, 1, true, 1>(a, sh, sub, pos0, k);
  } else {
    gnn_body<D, 2, false, 1>(a, sh, sub, pos0, k);
  }
}

}  // namespace ddmgnn
