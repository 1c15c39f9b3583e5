// Host-side (setup-time) builders: batched subdomain graph layout and the
// constant-bank weight packing.
//
// build_host_layout replaces the reference's per-subdomain template
// construction — build_local_graphs (pkg/src/ddmgnn/hybrid.py:36-46) =
// extract_local_matrix (asm.py:28-32, A[idx][:, idx]) + local_graph_from_matrix
// (dss.py:173-186) — and the partition-of-unity bookkeeping of
// _finish_decomposition (decomp.py:180-193) with one O(V + E) pass in C++,
// parallel over subdomains (OpenMP).  Edges are the structural off-diagonal
// pattern of A restricted to the subdomain, both directions, in ascending
// (src, dst) local order — exactly the reference's lexsort order because local
// node order is ascending global DOF order.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "ddmgnn_internal.h"
#include "gnn_cfg.h"

namespace ddmgnn {

int build_host_layout(int n, const int64_t* indptr, const int32_t* indices, const double* coords,
                      int K, const int64_t* sub_ptr, const int64_t* sub_idx, HostLayout* out,
                      std::string* err) {
  HostLayout& L = *out;
  if (K <= 0) {
    *err = "decomposition has no subdomains";
    return kValueError;
  }
  const long long V64 = sub_ptr[K];
  if (V64 >= (1ll << 31)) {
    *err = "total subdomain size exceeds 2^31";
    return kValueError;
  }
  L.n = n;
  L.K = K;
  L.V = static_cast<int>(V64);
  L.sub_ptr.resize(K + 1);
  L.idx.resize(L.V);
  std::vector<double> mult(n, 0.0);
  int k_max = 0;
  for (int i = 0; i < K; ++i) {
    const long long b = sub_ptr[i], e = sub_ptr[i + 1];
    if (e < b) {
      *err = "sub_ptr must be nondecreasing";
      return kValueError;
    }
    L.sub_ptr[i] = static_cast<int>(b);
    if (e - b > k_max) k_max = static_cast<int>(e - b);
    for (long long p = b; p < e; ++p) {
      const long long g = sub_idx[p];
      if (g < 0 || g >= n) {
        *err = "subdomain index out of range";
        return kValueError;
      }
      if (p > b && g <= sub_idx[p - 1]) {
        *err = "subdomain index arrays must be strictly ascending";
        return kValueError;
      }
      L.idx[p] = static_cast<int>(g);
      mult[g] += 1.0;  // decomp.py:186-187
    }
  }
  L.sub_ptr[K] = L.V;
  L.k_max = k_max;
  for (int j = 0; j < n; ++j) {
    if (mult[j] == 0.0) {
      *err = "subdomains do not cover all DOFs";  // decomp.py:188-189
      return kValueError;
    }
  }
  L.pou.resize(n);
  for (int j = 0; j < n; ++j) L.pou[j] = 1.0 / mult[j];  // decomp.py:190

  // ---- pass 1: local out-degree of every batched node ----
  L.deg.assign(L.V, 0);
  int deg_overflow = 0;
#pragma omp parallel
  {
    std::vector<int> loc(n, -1);
#pragma omp for schedule(dynamic, 4)
    for (int i = 0; i < K; ++i) {
      const int b = L.sub_ptr[i], e = L.sub_ptr[i + 1];
      for (int p = b; p < e; ++p) loc[L.idx[p]] = p - b;
      for (int p = b; p < e; ++p) {
        const int g = L.idx[p];
        int cnt = 0;
        for (long long jj = indptr[g]; jj < indptr[g + 1]; ++jj) {
          const int c = indices[jj];
          if (c != g && loc[c] >= 0) ++cnt;
        }
        if (cnt > 65535) {
#pragma omp atomic write
          deg_overflow = 1;
          cnt = 65535;
        }
        L.deg[p] = static_cast<uint16_t>(cnt);
      }
      for (int p = b; p < e; ++p) loc[L.idx[p]] = -1;
    }
  }
  if (deg_overflow) {
    *err = "local node degree exceeds 65535";
    return kValueError;
  }

  // ---- SELL-32 slices ----
  L.slice_base.resize(K);
  int S = 0;
  for (int i = 0; i < K; ++i) {
    L.slice_base[i] = S;
    S += (L.sub_ptr[i + 1] - L.sub_ptr[i] + 31) / 32;
  }
  L.S = S;
  L.slice_off.resize(S + 1);
  long long off = 0, E = 0;
  for (int i = 0; i < K; ++i) {
    const int b = L.sub_ptr[i], k = L.sub_ptr[i + 1] - b;
    for (int q = 0; q * 32 < k; ++q) {
      int w = 0;
      for (int t = q * 32; t < std::min(k, q * 32 + 32); ++t) {
        w = std::max<int>(w, L.deg[b + t]);
        E += L.deg[b + t];
      }
      L.slice_off[L.slice_base[i] + q] = static_cast<int>(off);
      off += 32ll * w;
      if (off >= (1ll << 31)) {
        *err = "padded edge count exceeds 2^31";
        return kValueError;
      }
    }
  }
  L.slice_off[S] = static_cast<int>(off);
  L.E = E;
  L.E_pad = off;
  L.edges.assign(static_cast<size_t>(off) * 2, 0.f);
  L.reach.assign(K, 0);
  L.xy.assign(2ull * L.V, 0.f);

  // ---- pass 2: edge records {|d|, dst} (dss.py:177-185) and centred coordinates ----
  // edge_vec = coords[dst] - coords[src] (dss.py:184) enters the model only
  // linearly (W1cat rows 2d, 2d+1), so the kernel folds it into the per-node
  // projections; the node coordinates are stored relative to the subdomain's
  // bounding-box centre so the fp32 difference keeps ~1e-6 relative accuracy.
#pragma omp parallel
  {
    std::vector<int> loc(n, -1);
#pragma omp for schedule(dynamic, 4)
    for (int i = 0; i < K; ++i) {
      const int b = L.sub_ptr[i], e = L.sub_ptr[i + 1];
      double lo[2] = {HUGE_VAL, HUGE_VAL}, hi[2] = {-HUGE_VAL, -HUGE_VAL};
      for (int p = b; p < e; ++p) {
        const int g = L.idx[p];
        loc[g] = p - b;
        for (int a = 0; a < 2; ++a) {
          lo[a] = std::min(lo[a], coords[2 * g + a]);
          hi[a] = std::max(hi[a], coords[2 * g + a]);
        }
      }
      const double cx = 0.5 * (lo[0] + hi[0]), cy = 0.5 * (lo[1] + hi[1]);
      // padding records (SELL slots past a node's degree, lanes past k) point at the
      // kernel's dummy Q row k with |d| = 0
      {
        const int kk = e - b, ns = (kk + 31) / 32;
        const long long r0 = L.slice_off[L.slice_base[i]], r1 = L.slice_off[L.slice_base[i] + ns];
        for (long long r = r0; r < r1; ++r) {
          L.edges[2 * r] = 0.f;
          std::memcpy(&L.edges[2 * r + 1], &kk, 4);
        }
      }
      int reach = 0;
      for (int p = b; p < e; ++p) {
        const int a = p - b, g = L.idx[p];
        L.xy[2ull * p] = static_cast<float>(coords[2 * g] - cx);
        L.xy[2ull * p + 1] = static_cast<float>(coords[2 * g + 1] - cy);
        const long long base = L.slice_off[L.slice_base[i] + (a >> 5)] + (a & 31);
        int slot = 0;
        for (long long jj = indptr[g]; jj < indptr[g + 1]; ++jj) {
          const int c = indices[jj];
          if (c == g || loc[c] < 0) continue;
          const double dx = coords[2 * c] - coords[2 * g];
          const double dy = coords[2 * c + 1] - coords[2 * g + 1];
          float* rec = &L.edges[static_cast<size_t>(base + 32ll * slot) * 2];
          rec[0] = static_cast<float>(std::hypot(dx, dy));
          int dst = loc[c];
          std::memcpy(&rec[1], &dst, 4);
          reach = std::max(reach, std::abs((dst >> 5) - (a >> 5)));
          ++slot;
        }
      }
      L.reach[i] = reach;
      for (int p = b; p < e; ++p) loc[L.idx[p]] = -1;
    }
  }

  // ---- transpose map: per DOF, (batched position, subdomain) in ascending subdomain ----
  L.tptr.assign(n + 1, 0);
  for (int p = 0; p < L.V; ++p) L.tptr[L.idx[p] + 1]++;
  for (int j = 0; j < n; ++j) L.tptr[j + 1] += L.tptr[j];
  L.tent.resize(2ull * L.V);
  {
    std::vector<int> cur(L.tptr.begin(), L.tptr.end() - 1);
    for (int i = 0; i < K; ++i)
      for (int p = L.sub_ptr[i]; p < L.sub_ptr[i + 1]; ++p) {
        const int slot = cur[L.idx[p]]++;
        L.tent[2ull * slot] = p;
        L.tent[2ull * slot + 1] = i;
      }
  }

  // ---- longest-processing-time order of subdomains (descending size) ----
  L.order.resize(K);
  std::iota(L.order.begin(), L.order.end(), 0);
  std::stable_sort(L.order.begin(), L.order.end(), [&](int x, int y) {
    return (L.sub_ptr[x + 1] - L.sub_ptr[x]) > (L.sub_ptr[y + 1] - L.sub_ptr[y]);
  });
  return kOk;
}

// Pack the reference's flat float64 parameters (dss.py:93-99 order: per layer
// phi_out, phi_in, psi, dec, each (w1, b1, w2, b2)) into fp32 constant banks.
// Per-layer bank layout (gnn_cfg.h, rows padded to 4 floats); W1cat is the
// reference's stacked hidden layer of both message MLPs (dss.py:281-290, the
// in-MLP's dx,dy rows negated), rows [h_src (d), h_dst (d), dx, dy, |d|]:
//   WQ  [d+2][2d]  = [W1cat h_dst rows ; +W1cat dx row ; +W1cat dy row]
//   WP  [d+2][2d]  = [W1cat h_src rows ; -W1cat dx row ; -W1cat dy row]
//   b1  [2d], WL [2d] = W1cat |d| row
//   WU  [3d+2][d]  = [Wp1 h rows ; Wp1 c row ; bdeg ; Mo ; Mi]
//         bdeg = b2o . Wp1[phi_o rows] + b2i . Wp1[phi_i rows]      (x node degree)
//         Mo   = e * W2o . Wp1[phi_o rows],  Mi = e * W2i . Wp1[phi_i rows]
//   bp1 [d], WP2 [d][d] = 0.5 * Wp2, bp2 [d]
// (WP2's 0.5 pairs with the kernel's node relu(x) = (x + |x|) / 2; e = 1 when the
// edge loop sums max(x, 0), 0.5 when it sums x + |x|, gnn_edge_relu_plain()).  The folded
// products are formed in fp64 and rounded once.  The FINAL layer's decoder
// (dss.py:327; only the last output is consumed by hybrid.py:124) sits at the end
// of every bank: Wd1[d][d] bd1[d] wd2[d] bd2.
int pack_model(int k_bar, int d, double alpha, const double* params, long long n_params,
               PackedModel* out, std::string* err) {
  if (k_bar < 1 || d < 1) {
    *err = "k_bar and d must be >= 1";
    return kValueError;
  }
  int o[kBankOffsets];
  if (!gnn_bank_offsets(d, o)) {
    *err = "latent dimension d=" + std::to_string(d) +
           " has no compiled kernel (supported: 3, 4, 5, 10, 20)";
    return kValueError;
  }
  const long long expect = static_cast<long long>(k_bar) * (11ll * d * d + 15ll * d + 1);
  if (n_params != expect) {
    *err = "weight block size mismatch: expected " + std::to_string(expect * 8) +
           " bytes for k_bar=" + std::to_string(k_bar) + ", d=" + std::to_string(d) + ", got " +
           std::to_string(n_params * 8);
    return kValueError;
  }
  enum { WQ, WP, B1, WL, WU, BP1, WP2, BP2, STRIDE, D2P, DP, DW1, DB1, DW2, DB2, LMAX };
  const int D = d;
  const int lmax = o[LMAX], stride = o[STRIDE], d2p = o[D2P], dp = o[DP];
  PackedModel& M = *out;
  M.k_bar = k_bar;
  M.d = d;
  M.lmax = lmax;
  M.stride = stride;
  M.dec_off = o[DW1];
  M.alpha = static_cast<float>(alpha);
  const int nch = (k_bar + lmax - 1) / lmax;
  M.bank.assign(static_cast<size_t>(nch) * kConstFloats, 0.f);

  const double* p = params;
  const double* last_dec = nullptr;
  auto f = [](double v) { return static_cast<float>(v); };
  for (int l = 0; l < k_bar; ++l) {
    const double* w1o = p; p += (2 * D + 3) * D;
    const double* b1o = p; p += D;
    const double* w2o = p; p += D * D;
    const double* b2o = p; p += D;
    const double* w1i = p; p += (2 * D + 3) * D;
    const double* b1i = p; p += D;
    const double* w2i = p; p += D * D;
    const double* b2i = p; p += D;
    const double* wp1 = p; p += (3 * D + 1) * D;
    const double* bp1 = p; p += D;
    const double* wp2 = p; p += D * D;
    const double* bp2 = p; p += D;
    last_dec = p;
    p += D * D + D + D + 1;
    float* B = &M.bank[static_cast<size_t>(l / lmax) * kConstFloats + (l % lmax) * stride];
    auto w1cat = [&](int row, int j) -> double {  // (2D+3) x 2D, dss.py:288-290
      if (j < D) return w1o[row * D + j];
      double v = w1i[row * D + (j - D)];
      if (row == 2 * D || row == 2 * D + 1) v = -v;
      return v;
    };
    for (int j = 0; j < 2 * D; ++j) {
      for (int m = 0; m < D; ++m) {
        B[o[WQ] + m * d2p + j] = f(w1cat(D + m, j));
        B[o[WP] + m * d2p + j] = f(w1cat(m, j));
      }
      for (int a = 0; a < 2; ++a) {
        B[o[WQ] + (D + a) * d2p + j] = f(w1cat(2 * D + a, j));
        B[o[WP] + (D + a) * d2p + j] = f(-w1cat(2 * D + a, j));
      }
      B[o[B1] + j] = f(j < D ? b1o[j] : b1i[j - D]);
      B[o[WL] + j] = f(w1cat(2 * D + 2, j));
    }
    // psi first layer (3D+1 inputs [h, c, phi_o, phi_i], dss.py:293-299) with the
    // messages' second layer folded in
    const double edge_scale = gnn_edge_relu_plain() ? 1.0 : 0.5;
    const double* wp1_o = wp1 + (D + 1) * D;      // rows of phi_o
    const double* wp1_i = wp1 + (2 * D + 1) * D;  // rows of phi_i
    for (int j = 0; j < D; ++j) {
      for (int m = 0; m <= D; ++m) B[o[WU] + m * dp + j] = f(wp1[m * D + j]);  // h rows, c row
      double bd = 0.0;
      for (int q = 0; q < D; ++q) bd += b2o[q] * wp1_o[q * D + j] + b2i[q] * wp1_i[q * D + j];
      B[o[WU] + (D + 1) * dp + j] = f(bd);
      for (int m = 0; m < D; ++m) {
        double mo = 0.0, mi = 0.0;
        for (int q = 0; q < D; ++q) {
          mo += w2o[m * D + q] * wp1_o[q * D + j];
          mi += w2i[m * D + q] * wp1_i[q * D + j];
        }
        B[o[WU] + (D + 2 + m) * dp + j] = f(edge_scale * mo);
        B[o[WU] + (2 * D + 2 + m) * dp + j] = f(edge_scale * mi);
      }
      B[o[BP1] + j] = f(bp1[j]);
      B[o[BP2] + j] = f(bp2[j]);
      for (int m = 0; m < D; ++m) B[o[WP2] + m * dp + j] = f(0.5 * wp2[m * D + j]);
    }
  }
  // decoder of the final layer: w1 [D][D], b1 [D], w2 [D][1], b2 [1]
  const double* dw1 = last_dec;
  const double* db1 = dw1 + D * D;
  const double* dw2 = db1 + D;
  const double* db2 = dw2 + D;
  for (int c = 0; c < nch; ++c) {
    float* B = &M.bank[static_cast<size_t>(c) * kConstFloats];
    for (int m = 0; m < D; ++m)
      for (int j = 0; j < D; ++j) B[o[DW1] + m * dp + j] = static_cast<float>(dw1[m * D + j]);
    for (int j = 0; j < D; ++j) {
      B[o[DB1] + j] = static_cast<float>(db1[j]);
      B[o[DW2] + j] = static_cast<float>(dw2[j]);
    }
    B[o[DB2]] = static_cast<float>(db2[0]);
  }
  return kOk;
}

}  // namespace ddmgnn
