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
#include <cooperative_groups.h>

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

__device__ __forceinline__ float max_nan(float x, float y) {
  float z;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(z) : "f"(x), "f"(y));
  return z;
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
// Rows m < M0 are skipped (their inputs are known to be exactly zero: the latent
// state of the first layer, see H0 below).
template <int NIN, int NPO, int OFF, int RS, int M0 = 0>
__device__ __forceinline__ void mv2(int base, const float (&x)[NIN], float2 (&acc)[NPO]) {
#pragma unroll
  for (int m = M0; m < NIN; ++m) {
#pragma unroll
    for (int j = 0; j < NPO; ++j)
      acc[j] = ffma2(bcast(x[m]), cpair(base + OFF + m * RS + 2 * j), acc[j]);
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

// Warp-uniform value (lane 0's): keeps loop bounds and branch conditions that ptxas
// cannot prove uniform out of divergent control flow (which would demote the
// weight loads from uniform LDCU to per-thread LDC).
__device__ __forceinline__ int uni(int v) { return __shfl_sync(0xffffffffu, v, 0); }

// ---------------------------------------------------------------------------- one slice
// The per-node work of one layer on one SELL slice (32 consecutive local nodes =
// one warp; node n0 + lane).  `W` is the layer's slot offset in the constant bank:
// a compile-time constant in every caller, so each weight pair is an
// immediate-addressed LDCU.128 operand of FFMA2.  No divergent branch: lanes past
// k recompute node k-1 (phase A, identical store) or write the dummy h row k
// (phase B), and the edge loop's trip count is the slice width (warp-uniform)
// with padding records pointing at the dummy Q row k (all -1e30, whose 2 relu term
// is exactly 0) — that is what keeps the weight loads in uniform registers.

// phase A: destination projection Q_t = [h_t, x_t, y_t] . WQ
template <int D, int W>
__device__ __forceinline__ void slice_q(int n0, int k, const float* h, float* q,
                                        const float2* __restrict__ xy) {
  using C = Cfg<D>;
  constexpr int NP2 = C::NP2;
  const int nn = min(n0 + static_cast<int>(threadIdx.x & 31), k - 1);
  float hin[D + 2];
  load_hxy<D>(h + nn * C::HS, __ldg(xy + nn), hin);
  float2 qa[NP2];
#pragma unroll
  for (int j = 0; j < NP2; ++j) qa[j] = make_float2(0.f, 0.f);
  mv2<D + 2, NP2, W + C::OFF_WQ, C::D2P>(0, hin, qa);
  float qs[C::QS];
#pragma unroll
  for (int j = 0; j < C::QS; ++j) qs[j] = 0.f;
#pragma unroll
  for (int j = 0; j < NP2; ++j) {
    qs[2 * j] = qa[j].x;
    qs[2 * j + 1] = qa[j].y;
  }
  store_vec<C::QS>(q + nn * C::QS, qs);
}

// phase A for two slices at once (n0a, n0b): every weight pair loaded once feeds
// both slices' FFMA2; the outputs are produced in two halves to bound registers.
// H0: the latent state is exactly zero (first layer of a model, h = 0 after the
// restriction, dss.py:309), so the h rows of every node mat-vec are skipped — the
// host enables it only when those weights are finite, where 0 * w = 0 exactly.
template <int D, int W, bool H0 = false>
__device__ __forceinline__ void slice_q2(int n0a, int n0b, int k, const float* h, float* q,
                                         const float2* __restrict__ xy) {
  using C = Cfg<D>;
  constexpr int NP2 = C::NP2, H1 = NP2 / 2;
  constexpr int M0 = H0 ? D : 0;
  const int lane = threadIdx.x & 31;
  const int na = min(n0a + lane, k - 1), nb = min(n0b + lane, k - 1);
  float xa[D + 2], xb[D + 2];
  if constexpr (H0) {
    const float2 pa = __ldg(xy + na), pb = __ldg(xy + nb);
#pragma unroll
    for (int i = 0; i < D; ++i) xa[i] = xb[i] = 0.f;
    xa[D] = pa.x; xa[D + 1] = pa.y;
    xb[D] = pb.x; xb[D + 1] = pb.y;
  } else {
    load_hxy<D>(h + na * C::HS, __ldg(xy + na), xa);
    load_hxy<D>(h + nb * C::HS, __ldg(xy + nb), xb);
  }
  float qsa[C::QS], qsb[C::QS];
#pragma unroll
  for (int j = 0; j < C::QS; ++j) qsa[j] = qsb[j] = 0.f;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int j0 = half ? H1 : 0, j1 = half ? NP2 : H1;
    float2 aa[NP2 - H1 > H1 ? NP2 - H1 : H1], ab[NP2 - H1 > H1 ? NP2 - H1 : H1];
#pragma unroll
    for (int j = 0; j < j1 - j0; ++j) aa[j] = ab[j] = make_float2(0.f, 0.f);
#pragma unroll
    for (int m = M0; m < D + 2; ++m) {
#pragma unroll
      for (int j = j0; j < j1; ++j) {
        const float2 w = cpair(W + C::OFF_WQ + m * C::D2P + 2 * j);
        aa[j - j0] = ffma2(bcast(xa[m]), w, aa[j - j0]);
        ab[j - j0] = ffma2(bcast(xb[m]), w, ab[j - j0]);
      }
    }
#pragma unroll
    for (int j = j0; j < j1; ++j) {
      qsa[2 * j] = aa[j - j0].x;
      qsa[2 * j + 1] = aa[j - j0].y;
      qsb[2 * j] = ab[j - j0].x;
      qsb[2 * j + 1] = ab[j - j0].y;
    }
  }
  store_vec<C::QS>(q + na * C::QS, qsa);
  store_vec<C::QS>(q + nb * C::QS, qsb);
}

// Q-row addressing of phase B: rows of the CTA's own shared memory ...
struct LocalRows {
  const float* q;
  template <int QS>
  __device__ __forceinline__ void load(int t, float (&v)[QS]) const { load_vec<QS>(q + t * QS, v); }
};

// phase B: edge aggregation + node update; returns whether the lane's node became
// non-finite and leaves the updated latent in hn (for a fused decoder)
template <int D, int W, class Rows = LocalRows, bool H0 = false>
__device__ __forceinline__ bool slice_u(int n0, int k, float* h, Rows q,
                                        const float* c, const float2* __restrict__ xy,
                                        const float2* __restrict__ edges, int so, int width,
                                        const uint16_t* __restrict__ deg, float alpha,
                                        float (&hn)[Cfg<D>::DH], int kdummy = -1) {
  using C = Cfg<D>;
  constexpr int NP2 = C::NP2, NPH = C::NPH;
  constexpr int M0 = H0 ? D : 0;  // first input row that can be non-zero
  const int lane = threadIdx.x & 31;
  const int n = n0 + lane;
  const int nn = min(n, k - 1);
#if GNN_EDGE_PREFETCH
  // the slice's edge records (width rows of 32 x 8 B) are re-read from L2 in every
  // layer (they do not fit L1 next to the node state): ask for them now, one
  // 128-byte line per lane, so the edge loop below finds them in L1 after the P
  // mat-vec instead of waiting on L2 one record ahead
  {
    const char* line = reinterpret_cast<const char*>(edges + so) + 128 * lane;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %1, %2;\n\t@p prefetch.global.L1 [%0];\n\t}"
                 ::"l"(line), "r"(lane), "r"(2 * width));
  }
#endif
  float2 p[NP2], s[NP2];
  {
    float hin[D + 2];
    if constexpr (H0) {
      const float2 pxy = __ldg(xy + nn);
#pragma unroll
      for (int i = 0; i < D; ++i) hin[i] = 0.f;
      hin[D] = pxy.x;
      hin[D + 1] = pxy.y;
    } else {
      load_hxy<D>(h + nn * C::HS, __ldg(xy + nn), hin);
    }
#pragma unroll
    for (int j = 0; j < NP2; ++j) {
      p[j] = cpair(W + C::OFF_B1 + 2 * j);
      s[j] = make_float2(0.f, 0.f);
    }
    mv2<D + 2, NP2, W + C::OFF_WP, C::D2P, M0>(0, hin, p);
  }
  const float2 dummy = make_float2(0.f, __int_as_float(kdummy < 0 ? k : kdummy));
  const float2* ep = edges + so + lane;
  float2 rec = width > 0 ? __ldg(ep) : dummy;
  for (int e = 0; e < width; ++e) {
    const float2 cur = rec;
    rec = e + 1 < width ? __ldg(ep + 32 * (e + 1)) : dummy;
    float qt[C::QS];
    q.template load<C::QS>(__float_as_int(cur.y), qt);
    const float2 len = bcast(cur.x);
#pragma unroll
    for (int j = 0; j < NP2; ++j) {
#if GNN_EDGE_SHIFT
      // relu(P + y) = max(y, -P) + P with y = Q_t + |d| WL: the P of every edge is
      // added once after the loop (width P; a padding record's y = -1e30 gives
      // max = -P, so it contributes exactly nothing), which leaves 2 of the 3 packed
      // FMA-pipe ops per pair and edge; max.NaN propagates NaN like numpy.maximum
      const float2 y = ffma2(len, cpair(W + C::OFF_WL + 2 * j),
                             make_float2(qt[2 * j], qt[2 * j + 1]));
      s[j] = fadd2(s[j], make_float2(max_nan(y.x, -p[j].x), max_nan(y.y, -p[j].y)));
#else
      float2 x = fadd2(p[j], make_float2(qt[2 * j], qt[2 * j + 1]));
      x = ffma2(len, cpair(W + C::OFF_WL + 2 * j), x);
#if GNN_EDGE_RELU_MAX
      // relu on the ALU pipe (FMNMX.NAN, NaN-propagating like numpy.maximum): the
      // FMA pipe, which bounds the kernel, keeps 3 of the 4 packed ops per pair
      s[j] = fadd2(s[j], make_float2(relu_nan(x.x), relu_nan(x.y)));
#else
      s[j] = fadd2(s[j], relu2x(x));
#endif
#endif
    }
  }
#if GNN_EDGE_SHIFT
  {
    const float2 wdt = bcast(static_cast<float>(width));
#pragma unroll
    for (int j = 0; j < NP2; ++j) s[j] = ffma2(wdt, p[j], s[j]);
  }
#endif
  // psi first layer with the messages' second layer folded in; the message part
  // accumulates in a second, independent chain (ILP)
  float2 u[NPH], u2[NPH];
  float hc[D + 2];
  {
    if constexpr (H0) {
#pragma unroll
      for (int i = 0; i < D; ++i) hc[i] = 0.f;
    } else {
      float hv[C::DH];
      load_vec<C::DH>(h + nn * C::HS, hv);
#pragma unroll
      for (int i = 0; i < D; ++i) hc[i] = hv[i];
    }
    hc[D] = c[nn];
    hc[D + 1] = static_cast<float>(deg[nn]);
  }
#pragma unroll
  for (int j = 0; j < NPH; ++j) {
    u[j] = cpair(W + C::OFF_BP1 + 2 * j);
    u2[j] = make_float2(0.f, 0.f);
  }
  mv2<D + 2, NPH, W + C::OFF_WU, C::DP, M0>(0, hc, u);
  {
    float sv[2 * D];
#pragma unroll
    for (int j = 0; j < NP2; ++j) {
      sv[2 * j] = s[j].x;
      sv[2 * j + 1] = s[j].y;
    }
    mv2<2 * D, NPH, W + C::OFF_WU + (D + 2) * C::DP, C::DP>(0, sv, u2);
  }
  float uv[D];
  float2 o[NPH];
#pragma unroll
  for (int j = 0; j < NPH; ++j) {
    const float2 r2 = relu2x(fadd2(u[j], u2[j]));
    if (2 * j < D) uv[2 * j] = r2.x;
    if (2 * j + 1 < D) uv[2 * j + 1] = r2.y;
    o[j] = cpair(W + C::OFF_BP2 + 2 * j);
  }
  mv2<D, NPH, W + C::OFF_WP2, C::DP>(0, uv, o);
  const float2 al = bcast(alpha);
  float2 fin = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < NPH; ++j) {
    float2 hp = make_float2(hc[2 * j], 2 * j + 1 < D ? hc[2 * j + 1] : 0.f);
    hp = ffma2(al, o[j], hp);
    fin = ffma2(hp, make_float2(0.f, 0.f), fin);  // NaN iff some h is non-finite (dss.py:324)
    hn[2 * j] = hp.x;
    hn[2 * j + 1] = (2 * j + 1 < D) ? hp.y : 0.f;
  }
  // the lane's own row only: in-place update; lanes past k write the dummy row k.
  // Lanes past k read row k-1 above, so order those reads before the valid lane's
  // write of row k-1 explicitly (no divergence here, but keep the warp contract)
  __syncwarp();
  store_vec<C::DH>(h + min(n, k) * C::HS, hn);
  return (fin.x != 0.f || fin.y != 0.f) && n < k;
}

// decoder of the final layer (dss.py:327) on one latent (immediate offsets)
template <int D>
__device__ __forceinline__ float decode(const float (&hv)[Cfg<D>::DH]) {
  using C = Cfg<D>;
  float hd[D];
#pragma unroll
  for (int i = 0; i < D; ++i) hd[i] = hv[i];
  float2 u[C::NPH];
#pragma unroll
  for (int j = 0; j < C::NPH; ++j) u[j] = cpair(C::DEC_B1 + 2 * j);
  mv2<D, C::NPH, C::DEC_W1, C::DP>(0, hd, u);
  float o = c_w[C::DEC_B2];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const float ui = (i & 1) ? u[i >> 1].y : u[i >> 1].x;
    o = fmaf(relu_nan(ui), c_w[C::DEC_W2 + i], o);
  }
  return o;
}

// ---------------------------------------------------------------------------- CTA path
// Node state (h, Q, c) of the CTA's subdomain in shared memory: Q rows 0..k
// (k = dummy), h rows 0..k (k = dummy), c.
template <int D>
struct SmemState {
  float *q, *h, *c;
  unsigned char* tc;  // tensor-core staging (kTcSmemBytes) when GNN_TC_Q
  __device__ __forceinline__ explicit SmemState(int k) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    tc = smem_raw;
    q = reinterpret_cast<float*>(smem_raw + kTcSmemBytes);
    h = q + static_cast<size_t>(k + 1) * Cfg<D>::QS;
    c = h + static_cast<size_t>(k + 1) * Cfg<D>::HS;
  }
};

// ---------------------------------------------------------------------------- tcgen05
// Phase A on the 5th-generation tensor cores (GNN_TC_Q): Q = [h, x, y] . WQ for a
// 128-node tile as one tcgen05.mma kind::tf32 GEMM (M=128, N=32 >= 2d, K=16 >=
// d+2), in 3xTF32 (a_hi b_hi + a_hi b_lo + a_lo b_hi: fp32-level accuracy,
// tools/ubench/tc_tf32_test.cu).  A (the tile's [h,x,y] split into tf32 hi/lo)
// is written to TMEM by the four warps that own the tile's 32-row lane quarters
// (tcgen05.st), B (WQ^T hi/lo, K-major, SWIZZLE_NONE) sits in shared memory, the
// fp32 accumulator in TMEM is read back with tcgen05.ld and stored as Q rows.
// Groups of four warps (7 at 28 warps) work on their tiles independently
// (named barrier + one mbarrier per group).
#if GNN_TC_Q
constexpr int kTcK = 16, kTcN = 32;
constexpr int kTcGroupCols = 64;  // per group: A_hi 16 | A_lo 16 | D 32 TMEM columns

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// K-major SWIZZLE_NONE canonical layout: core matrix = 8 rows x 16 B
__device__ __forceinline__ int tc_kmaj(int r, int k) {
  return (r >> 3) * ((kTcK / 4) * 128) + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
}
__device__ __forceinline__ uint64_t tc_sdesc(uint32_t addr, uint32_t sbo = (kTcK / 4) * 128) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>(128 >> 4) << 16) |                     // LBO: next K core
         (static_cast<uint64_t>(sbo >> 4) << 32) |                     // SBO: next 8 rows
         (static_cast<uint64_t>(1) << 46);                             // sm_100 version
}
// K-major SWIZZLE_NONE index for a K-wide operand
__device__ __forceinline__ int tc_kmaj_k(int r, int k, int kk) {
  return (r >> 3) * ((kk / 4) * 128) + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4;
}
constexpr uint32_t tc_idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (8u << 24);
}
constexpr uint32_t kTcIdesc = (1u << 4) | (2u << 7) | (2u << 10) |
                              (static_cast<uint32_t>(kTcN >> 3) << 17) | (8u << 24);
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void tc_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
      "%13,%14,%15,%16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
      "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]),
      "f"(v[15]));
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, float (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
        "=f"(v[7]), "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]),
        "=f"(v[14]), "=f"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tc_ld4(uint32_t taddr, float (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tc_mma(uint32_t d, uint32_t a, uint64_t b, int acc,
                                       uint32_t idesc = kTcIdesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n\t}\n"
      ::"r"(d), "r"(a), "l"(b), "r"(acc), "r"(idesc));
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tTC_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra TC_DONE;\n\tbra TC_WAIT;\n\tTC_DONE:\n\t}" ::"r"(mbar), "r"(parity));
}

// B operand of layer slot W: WQ^T split into tf32 hi/lo, K-major, into tc (whole CTA)
template <int D, int W>
__device__ __forceinline__ void tc_stage_wq(unsigned char* tc) {
  using C = Cfg<D>;
  float* bh = reinterpret_cast<float*>(tc);
  float* bl = bh + kTcN * kTcK;
  for (int i = threadIdx.x; i < kTcN * kTcK; i += blockDim.x) {
    const int n = i / kTcK, k = i % kTcK;
    const float w = (n < 2 * D && k < D + 2) ? c_w[W + C::OFF_WQ + k * C::D2P + n] : 0.f;
    const float hi = tf32_rna(w);
    bh[tc_kmaj(n, k) >> 2] = hi;
    bl[tc_kmaj(n, k) >> 2] = tf32_rna(w - hi);
  }
  asm volatile("fence.proxy.async.shared::cta;");
}

// phase A of one layer on the tensor cores, all tiles of the subdomain
template <int D>
__device__ __forceinline__ void tc_phase_q(int k, int warp, uint32_t tmem, unsigned char* tc,
                                           uint64_t* mbar, uint32_t& uses, const float* h,
                                           float* q, const float2* __restrict__ xy) {
  using C = Cfg<D>;
  static_assert(2 * D <= kTcN && D + 2 <= kTcK, "tile shape");
  const int lane = threadIdx.x & 31, quarter = warp & 3, group = warp >> 2;
  const int ngroups = blockDim.x >> 7;
  const uint32_t cols = tmem + group * kTcGroupCols;
  const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
  const uint32_t b_hi = smem_u32(tc), b_lo = b_hi + kTcN * kTcK * 4;
  const uint32_t mb = smem_u32(&mbar[group]);
  const int ntiles = (k + 127) >> 7;
  for (int t = group; t < ntiles; t += ngroups) {
    const int nn = min(t * 128 + quarter * 32 + lane, k - 1);
    float hin[D + 2];
    load_hxy<D>(h + nn * C::HS, __ldg(xy + nn), hin);
    float ahi[16], alo[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float x = i < D + 2 ? hin[i] : 0.f;
      ahi[i] = tf32_rna(x);
      alo[i] = tf32_rna(x - ahi[i]);
    }
    tc_st16(cols + lane_base, ahi);
    tc_st16(cols + lane_base + 16, alo);
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("bar.sync %0, 128;" ::"r"(1 + group));
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (quarter == 0 && lane == 0) {
      const uint32_t d = cols + 32;
#pragma unroll
      for (int ks = 0; ks < kTcK / 8; ++ks) {
        tc_mma(d, cols + 8 * ks, tc_sdesc(b_hi + ks * 256), ks > 0);      // a_hi b_hi
        tc_mma(d, cols + 8 * ks, tc_sdesc(b_lo + ks * 256), 1);           // a_hi b_lo
        tc_mma(d, cols + 16 + 8 * ks, tc_sdesc(b_hi + ks * 256), 1);      // a_lo b_hi
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   ::"r"(mb));
    }
    mbar_wait(mb, uses & 1);
    ++uses;
    asm volatile("tcgen05.fence::after_thread_sync;");
    float v0[16], v1[4];
    tc_ld16(cols + lane_base + 32, v0);
    tc_ld4(cols + lane_base + 48, v1);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    float qs[C::QS];
#pragma unroll
    for (int j = 0; j < C::QS; ++j) qs[j] = j < 16 ? v0[j] : (j < 20 ? v1[j - 16] : 0.f);
#pragma unroll
    for (int j = 2 * D; j < C::QS; ++j) qs[j] = 0.f;
    store_vec<C::QS>(q + nn * C::QS, qs);
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
}
#endif


#if GNN_TC_Q == 2
// ---- the whole layer's node mat-vecs on the tensor cores (GNN_TC_Q == 2) ----------
// Per layer the CTA stages four B operands (tf32 hi/lo, K-major) in shared memory:
// WQ^T and WP^T (N=32, K=16), WU^T (N=16, K=32: psi's first layer with the folded
// message layer), WP2^T (N=16, K=16).  Each 4-warp group owns 96 TMEM columns
// (A staging 0..63, accumulator 64..95) and walks its 128-node tiles: Q (phase A),
// then per tile P -> edge loop on the CUDA cores -> psi1 -> psi2 (phase B), each
// mat-vec a 3xTF32 GEMM issued by one thread after a group barrier and completed
// through the group's mbarrier.
constexpr int kTcCols = 96;
constexpr int kTcB_Q = 0, kTcB_P = 2 * 512, kTcB_U = 4 * 512, kTcB_2 = 6 * 512;  // floats

template <int D, int W>
__device__ __forceinline__ void tc_stage_all(unsigned char* tc) {
  using C = Cfg<D>;
  float* b = reinterpret_cast<float*>(tc);
  for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) {  // WQ / WP: N=32, K=16
    const int n = i / 16, kk = i % 16;
    const bool in = n < 2 * D && kk < D + 2;
    const float wq = in ? c_w[W + C::OFF_WQ + kk * C::D2P + n] : 0.f;
    const float wp = in ? c_w[W + C::OFF_WP + kk * C::D2P + n] : 0.f;
    const int o = tc_kmaj_k(n, kk, 16) >> 2;
    float hi = tf32_rna(wq);
    b[kTcB_Q + o] = hi;
    b[kTcB_Q + 512 + o] = tf32_rna(wq - hi);
    hi = tf32_rna(wp);
    b[kTcB_P + o] = hi;
    b[kTcB_P + 512 + o] = tf32_rna(wp - hi);
  }
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) {  // WU: N=16, K=32
    const int n = i / 32, kk = i % 32;
    const float w = (n < D && kk < 3 * D + 2) ? c_w[W + C::OFF_WU + kk * C::DP + n] : 0.f;
    const int o = tc_kmaj_k(n, kk, 32) >> 2;
    const float hi = tf32_rna(w);
    b[kTcB_U + o] = hi;
    b[kTcB_U + 512 + o] = tf32_rna(w - hi);
  }
  for (int i = threadIdx.x; i < 16 * 16; i += blockDim.x) {  // WP2: N=16, K=16
    const int n = i / 16, kk = i % 16;
    const float w = (n < D && kk < D) ? c_w[W + C::OFF_WP2 + kk * C::DP + n] : 0.f;
    const int o = tc_kmaj_k(n, kk, 16) >> 2;
    const float hi = tf32_rna(w);
    b[kTcB_2 + o] = hi;
    b[kTcB_2 + 256 + o] = tf32_rna(w - hi);
  }
  asm volatile("fence.proxy.async.shared::cta;");
}

// stage NV values (hi at col a0, lo at col a0 + NV) of this thread's TMEM row
// The split is hi = x with the 13 low mantissa bits cleared (one LOP3; cvt.rna.tf32
// is a ~10-instruction sequence here) and lo = x - hi (exact); the tensor core
// reads lo as tf32 by truncation, an error below 2^-21 |x|.
template <int NV>
__device__ __forceinline__ void tc_stage_row(uint32_t row_addr, const float (&v)[NV]) {
  static_assert(NV % 16 == 0, "16-column groups");
#pragma unroll
  for (int g = 0; g < NV / 16; ++g) {
    float hi[16], lo[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      hi[i] = __uint_as_float(__float_as_uint(v[16 * g + i]) & 0xFFFFE000u);
      lo[i] = v[16 * g + i] - hi[i];
    }
    tc_st16(row_addr + 16 * g, hi);
    tc_st16(row_addr + NV + 16 * g, lo);
  }
}

// group GEMM: D(cols + 64) = A(cols, K = 8 KSTEPS, hi | lo) . B(smem hi | lo)
template <int KSTEPS, int N>
__device__ __forceinline__ void tc_group_gemm(int group, int quarter, int lane, uint32_t cols,
                                              uint32_t b_hi, uint32_t b_lo, uint32_t mb,
                                              uint32_t& uses) {
  constexpr uint32_t sbo = KSTEPS * 2 * 128;
  constexpr uint32_t idesc = tc_idesc(N);
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("bar.sync %0, 128;" ::"r"(1 + group));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (quarter == 0 && lane == 0) {
    const uint32_t d = cols + 64;
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
      tc_mma(d, cols + 8 * ks, tc_sdesc(b_hi + ks * 256, sbo), ks > 0, idesc);
      tc_mma(d, cols + 8 * ks, tc_sdesc(b_lo + ks * 256, sbo), 1, idesc);
      tc_mma(d, cols + 8 * KSTEPS + 8 * ks, tc_sdesc(b_hi + ks * 256, sbo), 1, idesc);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(mb));
  }
  mbar_wait(mb, uses & 1);
  ++uses;
  asm volatile("tcgen05.fence::after_thread_sync;");
}

template <int D, int W>
__device__ __forceinline__ void tc_layer(const SmemState<D>& ns, int k, int warp,
                                         const float2* xy, const float2* edges,
                                         const int* slice_off, const uint16_t* deg, float alpha,
                                         int* bad, int layer_no, uint32_t tmem, uint64_t* mbar,
                                         uint32_t& uses) {
  using C = Cfg<D>;
  constexpr int NP2 = C::NP2, NPH = C::NPH;
  static_assert(2 * D <= 32 && D + 2 <= 16 && 3 * D + 2 <= 32, "tile shapes");
  const int lane = threadIdx.x & 31, quarter = warp & 3, group = warp >> 2;
  const int ngroups = blockDim.x >> 7;
  const uint32_t cols = tmem + group * kTcCols;
  const uint32_t row = cols + (static_cast<uint32_t>(quarter * 32) << 16);
  const uint32_t bq = smem_u32(ns.tc);
  const uint32_t mb = smem_u32(&mbar[group]);
  const int ntiles = (k + 127) >> 7;
  tc_stage_all<D, W>(ns.tc);
  __syncthreads();
  // ---- phase A: Q rows ----
  for (int t = group; t < ntiles; t += ngroups) {
    const int nn = min(t * 128 + quarter * 32 + lane, k - 1);
    float a[16];
    {
      float hin[D + 2];
      load_hxy<D>(ns.h + nn * C::HS, __ldg(xy + nn), hin);
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = i < D + 2 ? hin[i] : 0.f;
    }
    tc_stage_row<16>(row, a);
    tc_group_gemm<2, 32>(group, quarter, lane, cols, bq + 4 * kTcB_Q, bq + 4 * (kTcB_Q + 512), mb,
                         uses);
    float v0[16], v1[4];
    tc_ld16(row + 64, v0);
    tc_ld4(row + 80, v1);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    float qs[C::QS];
#pragma unroll
    for (int j = 0; j < C::QS; ++j) qs[j] = j < 2 * D ? (j < 16 ? v0[j] : v1[j - 16]) : 0.f;
    store_vec<C::QS>(ns.q + nn * C::QS, qs);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // ---- phase B ----
  int first_bad = 0;
  for (int t = group; t < ntiles; t += ngroups) {
    const int n0 = t * 128 + quarter * 32;
    const int n = n0 + lane, nn = min(n, k - 1);
    float hv[C::DH];
    load_vec<C::DH>(ns.h + nn * C::HS, hv);
    float2 xyn = __ldg(xy + nn);
    // P = b1 + [h, x, y] . WP
    float2 p[NP2];
    {
      float a[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = i < D ? hv[i] : (i == D ? xyn.x : (i == D + 1 ? xyn.y : 0.f));
      tc_stage_row<16>(row, a);
      tc_group_gemm<2, 32>(group, quarter, lane, cols, bq + 4 * kTcB_P, bq + 4 * (kTcB_P + 512),
                           mb, uses);
      float v0[16], v1[4];
      tc_ld16(row + 64, v0);
      tc_ld4(row + 80, v1);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int j = 0; j < NP2; ++j) {
        const float x0 = 2 * j < 16 ? v0[2 * j] : v1[2 * j - 16];
        const float x1 = 2 * j + 1 < 16 ? v0[2 * j + 1] : v1[2 * j + 1 - 16];
        p[j] = fadd2(make_float2(x0, x1), cpair(W + C::OFF_B1 + 2 * j));
      }
    }
    // edge aggregation on the CUDA cores (as slice_u)
    float2 s[NP2];
#pragma unroll
    for (int j = 0; j < NP2; ++j) s[j] = make_float2(0.f, 0.f);
    {
      const bool live = n0 < k;  // warp-uniform
      const int so = live ? uni(slice_off[n0 >> 5]) : 0;
      const int width = live ? (uni(slice_off[(n0 >> 5) + 1]) - so) >> 5 : 0;
      const float2 dummy = make_float2(0.f, __int_as_float(k));
      const float2* ep = edges + so + lane;
      float2 rec = width > 0 ? __ldg(ep) : dummy;
      for (int e = 0; e < width; ++e) {
        const float2 cur = rec;
        rec = e + 1 < width ? __ldg(ep + 32 * (e + 1)) : dummy;
        float qt[C::QS];
        load_vec<C::QS>(ns.q + __float_as_int(cur.y) * C::QS, qt);
        const float2 len = bcast(cur.x);
#pragma unroll
        for (int j = 0; j < NP2; ++j) {
          float2 x = fadd2(p[j], make_float2(qt[2 * j], qt[2 * j + 1]));
          x = ffma2(len, cpair(W + C::OFF_WL + 2 * j), x);
#if GNN_EDGE_RELU_MAX
          s[j] = fadd2(s[j], make_float2(relu_nan(x.x), relu_nan(x.y)));
#else
          s[j] = fadd2(s[j], relu2x(x));
#endif
        }
      }
    }
    // psi first layer: [h, c, deg, S] . WU
    float u[16];
    {
      float a[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) a[i] = 0.f;
#pragma unroll
      for (int i = 0; i < D; ++i) a[i] = hv[i];
      a[D] = ns.c[nn];
      a[D + 1] = static_cast<float>(deg[nn]);
#pragma unroll
      for (int j = 0; j < NP2; ++j) {
        a[D + 2 + 2 * j] = s[j].x;
        a[D + 3 + 2 * j] = s[j].y;
      }
      tc_stage_row<32>(row, a);
      tc_group_gemm<4, 16>(group, quarter, lane, cols, bq + 4 * kTcB_U, bq + 4 * (kTcB_U + 512),
                           mb, uses);
      tc_ld16(row + 64, u);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
    }
    // relu (u + bp1) -> psi second layer
    float o16[16];
    {
      float a[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float ui = i < D ? u[i] + c_w[W + C::OFF_BP1 + i] : 0.f;
        a[i] = ui + fabsf(ui);  // 2 relu, the 1/2 is folded into WP2
      }
      tc_stage_row<16>(row, a);
      tc_group_gemm<2, 16>(group, quarter, lane, cols, bq + 4 * kTcB_2, bq + 4 * (kTcB_2 + 256),
                           mb, uses);
      tc_ld16(row + 64, o16);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
    }
    float hn[C::DH];
    float fin = 0.f;
#pragma unroll
    for (int i = 0; i < C::DH; ++i) {
      if (i < D) {
        const float o = o16[i] + c_w[W + C::OFF_BP2 + i];
        hn[i] = fmaf(alpha, o, hv[i]);
        fin = fmaf(hn[i], 0.f, fin);
      } else {
        hn[i] = 0.f;
      }
    }
    if (fin != 0.f && first_bad == 0 && n < k) first_bad = layer_no;
    store_vec<C::DH>(ns.h + min(n, k) * C::HS, hn);
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  if (first_bad != 0) atomicCAS(bad, 0, first_bad);  // first bad layer wins
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
}
#endif

// one layer, all slices of the CTA's subdomain (warp w: slices w, w + nwarps, ...)
template <int D, int W, bool H0 = false>
__device__ __forceinline__ void cta_layer(const SmemState<D>& ns, int k, int warp,
                                          const float2* xy, const float2* edges,
                                          const int* slice_off, const uint16_t* deg,
                                          float alpha, int* bad, int layer_no,
                                          uint32_t tmem, uint64_t* mbar, uint32_t& uses) {
  const int step = blockDim.x;
#if GNN_TC_Q == 2
  tc_layer<D, W>(ns, k, warp, xy, edges, slice_off, deg, alpha, bad, layer_no, tmem, mbar, uses);
  return;
#elif GNN_TC_Q
  tc_stage_wq<D, W>(ns.tc);
  __syncthreads();
  tc_phase_q<D>(k, warp, tmem, ns.tc, mbar, uses, ns.h, ns.q, xy);
#else
#if GNN_Q2
  {  // slice pairs (s, s + nslices/2 rounded): one weight load feeds both
    const int nsl = (k + 31) >> 5, half = (nsl + 1) >> 1;
    for (int sa = warp; sa < half; sa += step >> 5) {
      const int sb = sa + half < nsl ? sa + half : sa;  // odd count: last pair repeats sa
      slice_q2<D, W, H0>(sa * 32, sb * 32, k, ns.h, ns.q, xy);
    }
  }
#else
  for (int n0 = 32 * warp; n0 < k; n0 += step) slice_q<D, W>(n0, k, ns.h, ns.q, xy);
#endif
#endif
  __syncthreads();
  int first_bad = 0;
  for (int n0 = 32 * warp; n0 < k; n0 += step) {
    const int so = uni(slice_off[n0 >> 5]);
    const int width = (uni(slice_off[(n0 >> 5) + 1]) - so) >> 5;
    float hn[Cfg<D>::DH];
    const bool b = slice_u<D, W, LocalRows, H0>(n0, k, ns.h, LocalRows{ns.q}, ns.c, xy, edges,
                                                so, width, deg, alpha, hn);
    if (b && first_bad == 0) first_bad = layer_no;
  }
  if (first_bad != 0) atomicCAS(bad, 0, first_bad);  // first bad layer wins
  __syncthreads();
}

// ---- dataflow schedule of the CTA path (GNN_DATAFLOW) -----------------------------
// The two CTA barriers per layer leave warps idle whenever a phase has fewer slices
// left than warps (config C: 34-61 slices over 28 warps).  A slice's edges reach at
// most R slices away (the subdomain's DOF order is banded; layout.cpp measures R), so
// the dependencies are local:
//   A(l, s)  overwrites Q rows of s: every B(l-1, s') with |s' - s| <= R has read them
//   B(l, s)  reads the Q rows of slices s-R..s+R: A(l, s') done for |s' - s| <= R
// Work items (A pairs of adjacent slices, then B slices, layer after layer) are dealt
// round robin over the warps as ONE sequence, so the assignment rotates from layer to
// layer and the load balances over the whole chunk instead of within each phase.  An
// item only waits for items earlier in the sequence, each warp takes its items in
// sequence order, so the earliest unfinished item is always ready: no deadlock.
// flags: fa[s] = layers whose phase A wrote s, fb[s] = layers whose phase B updated s.
__device__ __forceinline__ void df_wait(const int* f, int lo, int hi, int nsl, int need) {
  lo = max(lo, 0);
  hi = min(hi, nsl - 1);
  const int s = lo + static_cast<int>(threadIdx.x & 31);
  const volatile int* vf = f;
  while (true) {
    const int v = s <= hi ? vf[s] : need;
    if (__all_sync(0xffffffffu, v >= need)) break;
    __nanosleep(GNN_DF_SLEEP);
  }
  asm volatile("fence.acq_rel.cta;" ::: "memory");  // acquire: rows written before the flags
}

__device__ __forceinline__ void df_post(int* f, int s1, int s2, int val) {
  asm volatile("fence.acq_rel.cta;" ::: "memory");  // release: this warp's rows before the flag
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    volatile int* vf = f;
    vf[s1] = val;
    vf[s2] = val;
  }
}

template <int D, int W, bool H0 = false>
__device__ __forceinline__ void cta_layer_df(const SmemState<D>& ns, int k, int warp, int nw,
                                             const float2* xy, const float2* edges,
                                             const int* slice_off, const uint16_t* deg,
                                             float alpha, int* bad, int layer_no, int ll,
                                             int reach, int (&df)[2][kDfMaxSlices], int& t0) {
  const int nsl = (k + 31) >> 5;
#if GNN_DF_PAIRS
  // phase A: pairs (2j, 2j + 1) (odd count: the last pair repeats its slice)
  const int npairs = (nsl + 1) >> 1;
  for (int j = (warp - t0 % nw + nw) % nw; j < npairs; j += nw) {
    const int s1 = 2 * j, s2 = min(2 * j + 1, nsl - 1);
    df_wait(df[1], s1 - reach, s2 + reach, nsl, ll);
    slice_q2<D, W, H0>(s1 * 32, s2 * 32, k, ns.h, ns.q, xy);
    df_post(df[0], s1, s2, ll + 1);
  }
  t0 += npairs;
#else
  // phase A one slice per item: A(l, s) sits nsl positions after B(l-1, s) in the
  // item sequence, as B(l, s) after A(l, s), so every dependency is >= nsl - R items back
  for (int sl = (warp - t0 % nw + nw) % nw; sl < nsl; sl += nw) {
    df_wait(df[1], sl - reach, sl + reach, nsl, ll);
    slice_q<D, W>(sl * 32, k, ns.h, ns.q, xy);
    df_post(df[0], sl, sl, ll + 1);
  }
  t0 += nsl;
#endif
  int first_bad = 0;
  for (int sl = (warp - t0 % nw + nw) % nw; sl < nsl; sl += nw) {
    df_wait(df[0], sl - reach, sl + reach, nsl, ll + 1);
    const int so = uni(slice_off[sl]);
    const int width = (uni(slice_off[sl + 1]) - so) >> 5;
    float hn[Cfg<D>::DH];
    const bool b = slice_u<D, W, LocalRows, H0>(sl * 32, k, ns.h, LocalRows{ns.q}, ns.c, xy, edges,
                                                so, width, deg, alpha, hn);
    if (b && first_bad == 0) first_bad = layer_no;
    df_post(df[1], sl, sl, ll + 1);
  }
  t0 += nsl;
  if (first_bad != 0) atomicCAS(bad, 0, first_bad);  // first bad layer wins
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct GnnShared {
  double red[2][kGnnThreads / 32];
  int df[2][kDfMaxSlices];  // dataflow schedule: layers done per slice, phase A / phase B
  int bad;
  double scale;
  uint64_t mbar[kGnnThreads / 128];  // tensor-core groups (GNN_TC_Q)
  uint32_t tmem;
};

// Staged input: wait until the chunk of r this subdomain reads has arrived (flag
// written by the copy stream after the chunk's H2D copy; ddmgnn_apply_host).
__device__ __forceinline__ void wait_input(const GnnArgs& a, int sub) {
  if (a.ready == nullptr) return;
  if (threadIdx.x == 0) {
    const unsigned int* f = a.ready + a.sub_stage[sub];
    unsigned int v;
    unsigned long long t0 = 0;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (static_cast<int>(v - a.epoch) >= 0) break;
      __nanosleep(256);
      // never hang the GPU on a chunk that does not come: give up after ~5 s and
      // raise the apply's error word (the host reports it; the result is discarded)
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      if (t - t0 > 5000000000ull) {
        atomicMax(a.status, static_cast<int>(kStagingTimeout));
        break;
      }
    }
  }
  __syncthreads();
}

// Restriction of r to subdomain `sub` (hybrid.py:103-108) and its coarse RHS row
// (R0 r)_i, by the whole CTA: writes scale/r0r, c (fp32 r_i / s_i) into c_out and
// zeroes h rows 0..k-1.  Returns s_i (uniform).
template <int D>
__device__ __forceinline__ double restrict_sub(const GnnArgs& a, GnnShared& sh, int sub,
                                               int pos0, int k, double* scratch, float* c_out,
                                               float* h) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  double ss = 0.0, rr0 = 0.0;
  for (int n = tid; n < k; n += nthr) {
    const int g = a.idx[pos0 + n];
    const double v = __ldcg(a.r + g);  // L2: r may still be arriving in chunks
    ss = fma(v, v, ss);
    rr0 = fma(a.pou[g], v, rr0);
    scratch[n] = v;
  }
  ss = warp_sum(ss);
  rr0 = warp_sum(rr0);
  if ((tid & 31) == 0) {
    sh.red[0][tid >> 5] = ss;
    sh.red[1][tid >> 5] = rr0;
  }
  __syncthreads();
  if (tid == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int w = 0; w < (nthr >> 5); ++w) {
      t0 += sh.red[0][w];
      t1 += sh.red[1][w];
    }
    const double sc = sqrt(t0);
    sh.scale = sc;
    a.scale[sub] = sc;
    a.r0r[sub] = t1;
  }
  __syncthreads();
  const double s = __shfl_sync(0xffffffffu, sh.scale, 0);
  if (s == 0.0) return s;  // zero local residual: the subdomain contributes nothing
  for (int n = tid; n < k; n += nthr) c_out[n] = static_cast<float>(scratch[n] / s);
  __syncthreads();  // scratch may alias Q
  for (int n = tid; n < k; n += nthr) {
    float z[Cfg<D>::DH];
#pragma unroll
    for (int i = 0; i < Cfg<D>::DH; ++i) z[i] = 0.f;
    store_vec<Cfg<D>::DH>(h + n * Cfg<D>::HS, z);
  }
  return s;
}

// Subdomains whose node state fits the launch's shared memory (k <= a.cap0): one
// CTA per subdomain (LPT order), the whole chunk of layers on chip.
// Threads per CTA of the CTA and cluster paths: wide latents (d > 10) carry twice
// the per-lane state, so they trade warps for registers (512 x 128 instead of
// 896 x 72) rather than spill.
template <int D>
constexpr int gnn_cta_threads() { return D > 10 ? 512 : kGnnThreads; }

template <int D>
__global__ void __launch_bounds__(gnn_cta_threads<D>(), 1) gnn_kernel(GnnArgs a) {
  using C = Cfg<D>;
  if (a.skip != nullptr && uni(*a.skip) != 0) return;
  __shared__ GnnShared sh;
  const int sub = uni(a.order[a.order_begin + blockIdx.x]);
  const int pos0 = uni(a.sub_ptr[sub]);
  const int k = uni(a.sub_ptr[sub + 1] - pos0);
  const int tid = threadIdx.x, nthr = blockDim.x;
  SmemState<D> ns(k);
  if (tid == 0) sh.bad = 0;
  double s;
  if (a.first) {
    wait_input(a, sub);
    s = restrict_sub<D>(a, sh, sub, pos0, k, reinterpret_cast<double*>(ns.q), ns.c, ns.h);
    if (s == 0.0) {
      if (tid == 0) {
        a.bad_layer[sub] = 0;
        a.out_bad[sub] = 0;
      }
      return;
    }
    if (!a.last)
      for (int n = tid; n < k; n += nthr) a.cbuf[pos0 + n] = ns.c[n];
  } else {  // later chunk of a deep model: reload the node state
    s = __shfl_sync(0xffffffffu, a.scale[sub], 0);
    if (s == 0.0) return;
    for (int n = tid; n < k; n += nthr) {
      ns.c[n] = a.cbuf[pos0 + n];
      float hv[C::DH];
      load_vec<C::DH>(a.hbuf + static_cast<size_t>(pos0 + sub + n) * C::HS, hv);
      store_vec<C::DH>(ns.h + n * C::HS, hv);
    }
  }
  for (int j = tid; j < C::QS; j += nthr) ns.q[static_cast<size_t>(k) * C::QS + j] = -1e30f;
#if GNN_DATAFLOW && !GNN_TC_Q
  const int reach = a.reach != nullptr ? uni(a.reach[sub]) : -1;
  // only for a full-size CTA with more slices than warps: with fewer slices every
  // phase is one round anyway, and next to a second CTA on the SM (two-CTA mode) the
  // dataflow CTAs measured 1.9x slower than barrier CTAs (cause open; a poll back-off
  // did not change it: profiles/r02_exp_dataflow_{cluster_twocta,backoff_twocta})
  const bool dflow = reach >= 0 && reach <= kDfMaxReach && ((k + 31) >> 5) <= kDfMaxSlices &&
                     nthr == gnn_cta_threads<D>() && ((k + 31) >> 5) > (nthr >> 5);
  for (int i = tid; i < 2 * kDfMaxSlices; i += nthr) (&sh.df[0][0])[i] = 0;
#endif
  __syncthreads();
  uint32_t tmem = 0, uses = 0;
#if GNN_TC_Q
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 ::"r"(smem_u32(&sh.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < (nthr >> 7))
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sh.mbar[tid])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  tmem = sh.tmem;
#endif
  {
    const int warp = uni(tid >> 5);
    const float2* xy = a.xy + pos0;
    const int* so = a.slice_off + a.slice_base[sub];
    const uint16_t* dg = a.deg + pos0;
#define DDM_LAYER(LL)                                                                        \
  if constexpr (LL < C::LMAX) {                                                              \
    if (LL < a.nl)                                                                           \
      cta_layer<D, LL * C::STRIDE>(ns, k, warp, xy, a.edges, so, dg, a.alpha, &sh.bad,       \
                                   a.layer0 + LL, tmem, sh.mbar, uses);                      \
  }
#if GNN_DATAFLOW && !GNN_TC_Q
    if (dflow) {
      const int nw = uni(nthr >> 5);
      int t0 = 0;
#define DDM_LAYER_DF(LL)                                                                     \
  if constexpr (LL < C::LMAX) {                                                              \
    if (LL < a.nl)                                                                           \
      cta_layer_df<D, LL * C::STRIDE>(ns, k, warp, nw, xy, a.edges, so, dg, a.alpha, &sh.bad, \
                                      a.layer0 + LL, LL, reach, sh.df, t0);                  \
  }
      if (a.first && a.h0_skip) {
        if (a.nl > 0)
          cta_layer_df<D, 0, true>(ns, k, warp, nw, xy, a.edges, so, dg, a.alpha, &sh.bad,
                                   a.layer0, 0, reach, sh.df, t0);
      } else {
        DDM_LAYER_DF(0)
      }
      DDM_LAYER_DF(1) DDM_LAYER_DF(2) DDM_LAYER_DF(3) DDM_LAYER_DF(4)
      DDM_LAYER_DF(5) DDM_LAYER_DF(6) DDM_LAYER_DF(7) DDM_LAYER_DF(8) DDM_LAYER_DF(9)
#undef DDM_LAYER_DF
      __syncthreads();
    } else
#endif
    {
#if !GNN_TC_Q
    // the first layer of the model starts from h = 0 (dss.py:309)
    if (a.first && a.h0_skip) {
      if (a.nl > 0)
        cta_layer<D, 0, true>(ns, k, warp, xy, a.edges, so, dg, a.alpha, &sh.bad, a.layer0, tmem,
                              sh.mbar, uses);
    } else {
      DDM_LAYER(0)
    }
#else
    DDM_LAYER(0)
#endif
    DDM_LAYER(1) DDM_LAYER(2) DDM_LAYER(3) DDM_LAYER(4)
    DDM_LAYER(5) DDM_LAYER(6) DDM_LAYER(7) DDM_LAYER(8) DDM_LAYER(9)
    }
#undef DDM_LAYER
  }
#if GNN_TC_Q
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
#endif
  int outbad = 0;
  if (a.last) {
    // decoder of the final layer (dss.py:327) and rescaling (hybrid.py:135)
    for (int n = tid; n < k; n += nthr) {
      float hv[C::DH];
      load_vec<C::DH>(ns.h + n * C::HS, hv);
      const float o = decode<D>(hv);
      if (!isfinite(o)) outbad = 1;
      a.zloc[pos0 + n] = s * static_cast<double>(o);
    }
  } else {
    for (int n = tid; n < k; n += nthr) {
      float hv[C::DH];
      load_vec<C::DH>(ns.h + n * C::HS, hv);
      store_vec<C::DH>(a.hbuf + static_cast<size_t>(pos0 + sub + n) * C::HS, hv);
    }
  }
  outbad = __syncthreads_or(outbad);
  if (tid == 0) {
    const int b = sh.bad;
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

// ---------------------------------------------------------------------------- flat path
// Subdomains too large for one CTA's shared memory (k > a.cap0): node-parallel,
// one launch per phase per layer over all their slices (warp = slice, listed in
// a.bslices as (subdomain, slice)), node state in global scratch (L2-resident):
// h rows at hbuf[(pos0 + sub) ...], Q rows at qbuf[(pos0 + sub) ...] (each with a
// dummy row k), c at cbuf[pos0 ...].  Same per-node arithmetic as the CTA path.

// restriction of every big subdomain (CTA per subdomain, order[order_begin ...])
template <int D>
__global__ void __launch_bounds__(kGnnThreads, 1) gnn_flat_prologue(GnnArgs a) {
  using C = Cfg<D>;
  if (a.skip != nullptr && uni(*a.skip) != 0) return;
  __shared__ GnnShared sh;
  const int sub = uni(a.order[a.order_begin + blockIdx.x]);
  const int pos0 = uni(a.sub_ptr[sub]);
  const int k = uni(a.sub_ptr[sub + 1] - pos0);
  float* h = a.hbuf + static_cast<size_t>(pos0 + sub) * C::HS;
  float* q = a.qbuf + static_cast<size_t>(pos0 + sub) * C::QS;
  // restriction scratch: k doubles in the subdomain's Q rows (k*QS floats >= 2k)
  const double s = restrict_sub<D>(a, sh, sub, pos0, k, reinterpret_cast<double*>(q),
                                   a.cbuf + pos0, h);
  if (threadIdx.x == 0) {
    a.bad_layer[sub] = 0;
    a.out_bad[sub] = 0;
  }
  if (s == 0.0) return;
  for (int j = threadIdx.x; j < C::QS; j += blockDim.x) q[static_cast<size_t>(k) * C::QS + j] = -1e30f;
}

template <int D>
struct FlatSlice {
  int sub, pos0, k, n0;
  double s;
  // warp w of CTA b takes slice b * kFlatWarps + w: consecutive slices of one
  // subdomain share a CTA (and its L1) since neighbours' Q rows are mostly within
  // a few slices; padding entries (sub = -1) make s = 0 (the warp exits)
  __device__ __forceinline__ explicit FlatSlice(const GnnArgs& a) {
    const int2 bs = a.bslices[blockIdx.x * kFlatWarps + uni(static_cast<int>(threadIdx.x) >> 5)];
    sub = uni(bs.x);
    const bool pad = sub < 0;
    if (pad) sub = 0;
    n0 = uni(bs.y) * 32;
    pos0 = uni(a.sub_ptr[sub]);
    k = uni(a.sub_ptr[sub + 1] - pos0);
    s = pad ? 0.0 : __shfl_sync(0xffffffffu, a.scale[sub], 0);
  }
};

template <int D, int W>
__global__ void __launch_bounds__(32 * kFlatWarps) gnn_flat_q(GnnArgs a) {
  using C = Cfg<D>;
  if (a.skip != nullptr && uni(*a.skip) != 0) return;
  const FlatSlice<D> f(a);
  if (f.s == 0.0) return;
  slice_q<D, W>(f.n0, f.k, a.hbuf + static_cast<size_t>(f.pos0 + f.sub) * C::HS,
                a.qbuf + static_cast<size_t>(f.pos0 + f.sub) * C::QS, a.xy + f.pos0);
}

template <int D, int W>
__global__ void __launch_bounds__(32 * kFlatWarps) gnn_flat_u(GnnArgs a, int layer_no, int decode_last) {
  using C = Cfg<D>;
  if (a.skip != nullptr && uni(*a.skip) != 0) return;
  const FlatSlice<D> f(a);
  if (f.s == 0.0) return;
  const int* so_p = a.slice_off + a.slice_base[f.sub] + (f.n0 >> 5);
  const int so = uni(so_p[0]);
  const int width = (uni(so_p[1]) - so) >> 5;
  float hn[C::DH];
  const bool bad = slice_u<D, W>(f.n0, f.k, a.hbuf + static_cast<size_t>(f.pos0 + f.sub) * C::HS,
                                 LocalRows{a.qbuf + static_cast<size_t>(f.pos0 + f.sub) * C::QS},
                                 a.cbuf + f.pos0, a.xy + f.pos0, a.edges, so, width,
                                 a.deg + f.pos0, a.alpha, hn);
  // layers run in order (one launch each), so the first non-zero wins
  if (bad) {
    atomicCAS(&a.bad_layer[f.sub], 0, layer_no);
    atomicMax(a.status, static_cast<int>(kPrecondError));
  }
  if (decode_last) {
    const int n = f.n0 + static_cast<int>(threadIdx.x & 31);
    const float o = decode<D>(hn);
    if (n < f.k) {
      if (!isfinite(o)) {
        a.out_bad[f.sub] = 1;
        atomicMax(a.status, static_cast<int>(kPrecondError));
      }
      a.zloc[f.pos0 + n] = f.s * static_cast<double>(o);
    }
  }
}


// ---------------------------------------------------------------------------- cluster path
// Subdomains up to 8x the shared-memory capacity of one CTA: a thread-block cluster
// of CS CTAs per subdomain, CTA r holding the node state of local nodes
// [r npc, (r+1) npc) in its shared memory; phase B reads neighbours' Q rows through
// distributed shared memory (cluster.map_shared_rank), phases are separated by
// cluster barriers, and the restriction sums meet in CTA 0.  Same per-node
// arithmetic as the CTA path.
struct ClusterRows {
  uint32_t q;  // shared-window address of this CTA's Q rows (same offset in every CTA)
  int npc, last;
  float inv_npc;
  template <int QS>
  __device__ __forceinline__ void load(int t, float (&v)[QS]) const {
    static_assert(QS % 4 == 0, "Q rows are float4-aligned");
    int r = __float2int_rz(__int2float_rn(t) * inv_npc);
    r -= (r * npc > t);
    r += ((r + 1) * npc <= t);
    r = min(r, last);
    uint32_t a;
    asm("mapa.shared::cluster.u32 %0, %1, %2;"
        : "=r"(a) : "r"(q + static_cast<uint32_t>((t - r * npc) * QS * 4)), "r"(r));
#pragma unroll
    for (int i = 0; i < QS; i += 4)
      asm("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=f"(v[i]), "=f"(v[i + 1]), "=f"(v[i + 2]), "=f"(v[i + 3])
                   : "r"(a + 4 * i));
  }
};

template <int D>
__global__ void __launch_bounds__(gnn_cta_threads<D>(), 1) gnn_cluster_kernel(GnnArgs a) {
  using C = Cfg<D>;
  namespace cg = cooperative_groups;
  if (a.skip != nullptr && uni(*a.skip) != 0) return;  // same flag for the whole cluster
  __shared__ GnnShared sh;
  __shared__ double cpart[2][8];
  __shared__ int cbad;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = static_cast<int>(cl.num_blocks()), rank = static_cast<int>(cl.block_rank());
  const int sub = uni(a.csubs[blockIdx.x / CS]);
  const int pos0 = uni(a.sub_ptr[sub]);
  const int k = uni(a.sub_ptr[sub + 1] - pos0);
  const int npc = ((k + CS - 1) / CS + 31) / 32 * 32;
  const int lo = rank * npc;
  const int cnt = max(0, min(k - lo, npc));
  const int tid = threadIdx.x, nthr = blockDim.x;
  SmemState<D> ns(npc);
  if (tid == 0) {
    sh.bad = 0;
    cbad = INT_MAX;
  }
  double s;
  if (a.first) {
    wait_input(a, sub);
    double* scratch = reinterpret_cast<double*>(ns.q);
    double ss = 0.0, rr0 = 0.0;
    for (int n = tid; n < cnt; n += nthr) {
      const int g = a.idx[pos0 + lo + n];
      const double v = __ldcg(a.r + g);
      ss = fma(v, v, ss);
      rr0 = fma(a.pou[g], v, rr0);
      scratch[n] = v;
    }
    ss = warp_sum(ss);
    rr0 = warp_sum(rr0);
    if ((tid & 31) == 0) {
      sh.red[0][tid >> 5] = ss;
      sh.red[1][tid >> 5] = rr0;
    }
    cl.sync();  // also: every CTA of the cluster has started before DSMEM is written
    if (tid == 0) {
      double t0 = 0.0, t1 = 0.0;
      for (int w = 0; w < (nthr >> 5); ++w) {
        t0 += sh.red[0][w];
        t1 += sh.red[1][w];
      }
      double* dst = cl.map_shared_rank(&cpart[0][0], 0);
      dst[rank] = t0;
      dst[8 + rank] = t1;
    }
    cl.sync();
    if (tid == 0) {
      const double* src = cl.map_shared_rank(&cpart[0][0], 0);
      double t0 = 0.0, t1 = 0.0;
      for (int j = 0; j < CS; ++j) {
        t0 += src[j];
        t1 += src[8 + j];
      }
      sh.scale = sqrt(t0);
      if (rank == 0) {
        a.scale[sub] = sh.scale;
        a.r0r[sub] = t1;
        a.bad_layer[sub] = 0;
        a.out_bad[sub] = 0;
      }
    }
    cl.sync();  // CTA 0's partials read by everyone before anyone may leave
    s = __shfl_sync(0xffffffffu, sh.scale, 0);
    if (s == 0.0) return;
    for (int n = tid; n < cnt; n += nthr) {
      const float c = static_cast<float>(scratch[n] / s);
      ns.c[n] = c;
      if (!a.last) a.cbuf[pos0 + lo + n] = c;
    }
    __syncthreads();
    for (int n = tid; n < cnt; n += nthr) {
      float z[C::DH];
#pragma unroll
      for (int i = 0; i < C::DH; ++i) z[i] = 0.f;
      store_vec<C::DH>(ns.h + n * C::HS, z);
    }
  } else {
    s = __shfl_sync(0xffffffffu, a.scale[sub], 0);
    if (s == 0.0) return;
    for (int n = tid; n < cnt; n += nthr) {
      ns.c[n] = a.cbuf[pos0 + lo + n];
      float hv[C::DH];
      load_vec<C::DH>(a.hbuf + static_cast<size_t>(pos0 + sub + lo + n) * C::HS, hv);
      store_vec<C::DH>(ns.h + n * C::HS, hv);
    }
  }
  // dummy Q row: the SELL padding target t = k lands in the last CTA at row cnt
  for (int j = tid; j < C::QS; j += nthr) ns.q[static_cast<size_t>(cnt) * C::QS + j] = -1e30f;
  cl.sync();
  {
    const int warp = uni(tid >> 5);
    const float2* xy = a.xy + pos0 + lo;
    const int* so_p = a.slice_off + a.slice_base[sub] + (lo >> 5);
    const uint16_t* dg = a.deg + pos0 + lo;
    const ClusterRows rows{static_cast<uint32_t>(__cvta_generic_to_shared(ns.q)), npc, CS - 1,
                           1.0f / static_cast<float>(npc)};
    const int nsl = (cnt + 31) >> 5, half = (nsl + 1) >> 1;
#define DDM_CLAYER(LL)                                                                        \
  if constexpr (LL < C::LMAX) {                                                               \
    if (LL < a.nl) {                                                                          \
      for (int sa = warp; sa < half; sa += nthr >> 5) {                                       \
        const int sb = sa + half < nsl ? sa + half : sa;                                      \
        slice_q2<D, LL * C::STRIDE>(sa * 32, sb * 32, cnt, ns.h, ns.q, xy);                   \
      }                                                                                       \
      cl.sync();                                                                              \
      int fb = 0;                                                                             \
      for (int n0 = 32 * warp; n0 < cnt; n0 += nthr) {                                        \
        const int so = uni(so_p[n0 >> 5]);                                                    \
        const int width = (uni(so_p[(n0 >> 5) + 1]) - so) >> 5;                               \
        float hn[C::DH];                                                                      \
        const bool b = slice_u<D, LL * C::STRIDE, ClusterRows>(                               \
            n0, cnt, ns.h, rows, ns.c, xy, a.edges, so, width, dg, a.alpha, hn, k);           \
        if (b && fb == 0) fb = a.layer0 + LL;                                                 \
      }                                                                                       \
      if (fb != 0) atomicCAS(&sh.bad, 0, fb); /* first bad layer wins */                    \
      cl.sync();                                                                              \
    }                                                                                         \
  }
    DDM_CLAYER(0) DDM_CLAYER(1) DDM_CLAYER(2) DDM_CLAYER(3) DDM_CLAYER(4)
    DDM_CLAYER(5) DDM_CLAYER(6) DDM_CLAYER(7) DDM_CLAYER(8) DDM_CLAYER(9)
#undef DDM_CLAYER
  }
  int outbad = 0;
  if (a.last) {
    for (int n = tid; n < cnt; n += nthr) {
      float hv[C::DH];
      load_vec<C::DH>(ns.h + n * C::HS, hv);
      const float o = decode<D>(hv);
      if (!isfinite(o)) outbad = 1;
      a.zloc[pos0 + lo + n] = s * static_cast<double>(o);
    }
  } else {
    for (int n = tid; n < cnt; n += nthr) {
      float hv[C::DH];
      load_vec<C::DH>(ns.h + n * C::HS, hv);
      store_vec<C::DH>(a.hbuf + static_cast<size_t>(pos0 + sub + lo + n) * C::HS, hv);
    }
  }
  outbad = __syncthreads_or(outbad);
  // combine the CTAs' flags in CTA 0: first (smallest) bad layer, any bad output
  if (tid == 0 && sh.bad != 0) atomicMin(cl.map_shared_rank(&cbad, 0), sh.bad);
  cl.sync();
  if (tid == 0) {
    if (outbad) {
      a.out_bad[sub] = 1;
      atomicMax(a.status, static_cast<int>(kPrecondError));
    }
    if (rank == 0 && cbad != INT_MAX) {
      if (a.first || a.bad_layer[sub] == 0) a.bad_layer[sub] = cbad;
      atomicMax(a.status, static_cast<int>(kPrecondError));
    }
  }
}

}  // namespace ddmgnn
