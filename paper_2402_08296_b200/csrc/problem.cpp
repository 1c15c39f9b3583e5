// Native input producers for the DDM-GNN path (host-only, no CUDA): the parts of
// the reference's problem setup that are O(N) / O(K*N) Python loops, ported
// bit-exactly so that 1M- and 10M-node problems can be built on the GPU host.
//
//   ddmp_blob_triangles   mesh.py:131-150,196-201  (ring fan + _zip_rings)
//   ddmp_boundary_flags   mesh.py:71-87            (edges used by one triangle)
//   ddmp_assemble_*       fem.py:120-165           (dict accumulation in triangle
//                                                   order, Dirichlet elimination in
//                                                   key-insertion order, CSR)
//   ddmp_partition        decomp.py:92-159         (farthest-point seeds, smallest-
//                                                   region-first BFS growth, one
//                                                   smoothing pass)
//   ddmp_add_overlap_*    decomp.py:196-216        (BFS layers, sorted subdomains)
//
// Floating-point work that the reference does with numpy ufuncs (coordinates,
// element matrices, load vector) stays in numpy on the caller's side, so every
// rounding matches the reference; this file only reproduces the loops and their
// accumulation ORDER.  Compiled with -ffp-contract=off (no FMA contraction).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <deque>
#include <numeric>
#include <set>
#include <string>
#include <utility>
#include <vector>

namespace {

thread_local std::string g_perr;

// Sorted-unique neighbour lists (self included) from triangles.
struct Pattern {
  std::vector<int64_t> ptr;
  std::vector<int32_t> col;
  int64_t find(int64_t i, int64_t j) const {
    auto b = col.begin() + ptr[i], e = col.begin() + ptr[i + 1];
    auto it = std::lower_bound(b, e, static_cast<int32_t>(j));
    return it - col.begin();
  }
};

Pattern build_pattern(int64_t n, int64_t T, const int64_t* tris) {
  Pattern P;
  std::vector<int64_t> cnt(n + 1, 0);
  for (int64_t t = 0; t < 3 * T; ++t) cnt[tris[t] + 1] += 3;
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  std::vector<int32_t> tmp(cnt[n]);
  std::vector<int64_t> cur(cnt.begin(), cnt.end() - 1);
  for (int64_t t = 0; t < T; ++t)
    for (int a = 0; a < 3; ++a) {
      const int64_t i = tris[3 * t + a];
      for (int b = 0; b < 3; ++b) tmp[cur[i]++] = static_cast<int32_t>(tris[3 * t + b]);
    }
  P.ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    auto b = tmp.begin() + cnt[i], e = tmp.begin() + cnt[i + 1];
    std::sort(b, e);
    P.ptr[i + 1] = std::unique(b, e) - b;
  }
  for (int64_t i = 0; i < n; ++i) P.ptr[i + 1] += P.ptr[i];
  P.col.resize(P.ptr[n]);
  for (int64_t i = 0; i < n; ++i)
    std::copy(tmp.begin() + cnt[i], tmp.begin() + cnt[i] + (P.ptr[i + 1] - P.ptr[i]),
              P.col.begin() + P.ptr[i]);
  return P;
}

struct Assembly {
  int64_t n_int = 0;
  std::vector<int64_t> indptr;
  std::vector<int32_t> indices;
  std::vector<double> data;
  std::vector<double> b;
};

// max segment tree over d (leftmost index of the maximum, like np.argmax)
struct ArgMaxTree {
  int64_t size = 1;
  std::vector<int64_t> val;  // d value
  std::vector<int64_t> idx;
  explicit ArgMaxTree(const std::vector<int64_t>& d) {
    const int64_t n = static_cast<int64_t>(d.size());
    while (size < n) size <<= 1;
    val.assign(2 * size, INT64_MIN);
    idx.assign(2 * size, INT64_MAX);
    for (int64_t i = 0; i < n; ++i) {
      val[size + i] = d[i];
      idx[size + i] = i;
    }
    for (int64_t p = size - 1; p >= 1; --p) pull(p);
  }
  void pull(int64_t p) {
    const int64_t l = 2 * p, r = 2 * p + 1;
    if (val[l] >= val[r]) {  // ties -> left (smaller index)
      val[p] = val[l];
      idx[p] = idx[l];
    } else {
      val[p] = val[r];
      idx[p] = idx[r];
    }
  }
  void set(int64_t i, int64_t v) {
    int64_t p = size + i;
    val[p] = v;
    for (p >>= 1; p >= 1; p >>= 1) pull(p);
  }
  int64_t argmax() const { return idx[1]; }
};

inline void neighbors_bfs(int64_t n, const int64_t* indptr, const int32_t* indices, int64_t src,
                          std::vector<int64_t>& dist) {
  dist.assign(n, -1);
  std::vector<int32_t> q;
  q.reserve(n);
  dist[src] = 0;
  q.push_back(static_cast<int32_t>(src));
  for (size_t h = 0; h < q.size(); ++h) {
    const int64_t u = q[h];
    for (int64_t t = indptr[u]; t < indptr[u + 1]; ++t) {
      const int64_t v = indices[t];
      if (v == u) continue;
      if (dist[v] < 0) {
        dist[v] = dist[u] + 1;
        q.push_back(static_cast<int32_t>(v));
      }
    }
  }
}

}  // namespace

extern "C" {

const char* ddmp_last_error(void) { return g_perr.c_str(); }

// mesh.py:196-201 — returns the triangle count; writes (T,3) when out != NULL.
int64_t ddmp_blob_triangles(int64_t n_rings, const int64_t* ring_sizes, int64_t* out) {
  std::vector<int64_t> start(n_rings);
  int64_t next = 1;
  for (int64_t j = 0; j < n_rings; ++j) {
    start[j] = next;
    next += ring_sizes[j];
  }
  int64_t T = 0;
  auto emit = [&](int64_t a, int64_t b, int64_t c) {
    if (out) {
      out[3 * T] = a;
      out[3 * T + 1] = b;
      out[3 * T + 2] = c;
    }
    ++T;
  };
  const int64_t n0 = ring_sizes[0];
  for (int64_t i = 0; i < n0; ++i) emit(0, start[0] + i, start[0] + (i + 1) % n0);
  for (int64_t j = 1; j < n_rings; ++j) {  // _zip_rings(rings[j-1], rings[j]), mesh.py:131-150
    const int64_t n_in = ring_sizes[j - 1], n_out = ring_sizes[j];
    const int64_t si = start[j - 1], so = start[j];
    int64_t i = 0, k = 0;
    while (i < n_in || k < n_out) {
      const bool adv_inner = i < n_in && (k == n_out || (i + 1) * n_out <= (k + 1) * n_in);
      if (adv_inner) {
        emit(si + i % n_in, so + k % n_out, si + (i + 1) % n_in);
        ++i;
      } else {
        emit(si + i % n_in, so + k % n_out, so + (k + 1) % n_out);
        ++k;
      }
    }
  }
  return T;
}

// mesh.py:80-87
int ddmp_boundary_flags(int64_t n, int64_t T, const int64_t* tris, uint8_t* flags) {
  Pattern P = build_pattern(n, T, tris);
  std::vector<int32_t> cnt(P.col.size(), 0);
  for (int64_t t = 0; t < T; ++t) {
    const int64_t v[3] = {tris[3 * t], tris[3 * t + 1], tris[3 * t + 2]};
    for (int e = 0; e < 3; ++e) {
      int64_t a = v[e], b = v[(e + 1) % 3];
      if (a > b) std::swap(a, b);
      cnt[P.find(a, b)]++;
    }
  }
  std::memset(flags, 0, n);
  for (int64_t a = 0; a < n; ++a)
    for (int64_t p = P.ptr[a]; p < P.ptr[a + 1]; ++p) {
      const int64_t b = P.col[p];
      if (b > a && cnt[p] == 1) flags[a] = flags[b] = 1;
    }
  return 0;
}

// fem.py:120-165.  k_el: (T,3,3) element matrices from numpy; load: np.bincount
// load vector; g_full: Dirichlet values on all nodes (0 at interior nodes).
void* ddmp_assemble(int64_t n, int64_t T, const int64_t* tris, const double* k_el,
                    const uint8_t* boundary, const double* load, const double* g_full) {
  auto* A = new Assembly();
  Pattern P = build_pattern(n, T, tris);
  std::vector<int64_t> iof(n, -1);
  int64_t n_int = 0;
  for (int64_t i = 0; i < n; ++i)
    if (!boundary[i]) iof[i] = n_int++;
  A->n_int = n_int;
  std::vector<double> acc(P.col.size(), 0.0);
  std::vector<int64_t> first(P.col.size(), -1);
  int64_t counter = 0;
  for (int64_t t = 0; t < T; ++t)
    for (int li = 0; li < 3; ++li) {
      const int64_t gi = tris[3 * t + li];
      for (int lj = 0; lj < 3; ++lj) {
        const int64_t p = P.find(gi, tris[3 * t + lj]);
        if (first[p] < 0) first[p] = counter++;
        acc[p] = acc[p] + k_el[9 * t + 3 * li + lj];  // acc.get(key, 0.0) + kt[li, lj]
      }
    }
  A->b.resize(n_int);
  A->indptr.assign(n_int + 1, 0);
  for (int64_t gi = 0; gi < n; ++gi) {
    const int64_t ii = iof[gi];
    if (ii < 0) continue;
    int64_t c = 0;
    for (int64_t p = P.ptr[gi]; p < P.ptr[gi + 1]; ++p) c += iof[P.col[p]] >= 0;
    A->indptr[ii + 1] = c;
  }
  for (int64_t i = 0; i < n_int; ++i) A->indptr[i + 1] += A->indptr[i];
  A->indices.resize(A->indptr[n_int]);
  A->data.resize(A->indptr[n_int]);
  std::vector<std::pair<int64_t, int64_t>> bnd;  // (first occurrence, pattern pos)
  for (int64_t gi = 0; gi < n; ++gi) {
    const int64_t ii = iof[gi];
    if (ii < 0) continue;
    int64_t o = A->indptr[ii];
    bnd.clear();
    for (int64_t p = P.ptr[gi]; p < P.ptr[gi + 1]; ++p) {
      const int64_t jj = iof[P.col[p]];
      if (jj >= 0) {
        A->indices[o] = static_cast<int32_t>(jj);
        A->data[o] = acc[p];
        ++o;
      } else {
        bnd.emplace_back(first[p], p);
      }
    }
    // b_red[ii] -= v * g_full[gj] in dict insertion order (fem.py:149-160)
    std::sort(bnd.begin(), bnd.end());
    double bi = load[gi];
    for (const auto& e : bnd) bi = bi - acc[e.second] * g_full[P.col[e.second]];
    A->b[ii] = bi;
  }
  return A;
}

void ddmp_assemble_sizes(void* h, int64_t* n_int, int64_t* nnz) {
  auto* A = static_cast<Assembly*>(h);
  *n_int = A->n_int;
  *nnz = static_cast<int64_t>(A->indices.size());
}

void ddmp_assemble_copy(void* h, int64_t* indptr, int32_t* indices, double* data, double* b) {
  auto* A = static_cast<Assembly*>(h);
  std::copy(A->indptr.begin(), A->indptr.end(), indptr);
  std::copy(A->indices.begin(), A->indices.end(), indices);
  std::copy(A->data.begin(), A->data.end(), data);
  std::copy(A->b.begin(), A->b.end(), b);
}

void ddmp_assemble_free(void* h) { delete static_cast<Assembly*>(h); }

// decomp.py:92-159.  `start` = int(np.random.default_rng(seed).integers(n)),
// drawn by the caller with numpy.  Returns 0, or 1 with ddmp_last_error().
int ddmp_partition(int64_t n, const int64_t* indptr, const int32_t* indices, int64_t target_size,
                   int64_t start, int64_t* owner) {
  if (!(1 <= target_size && target_size <= n)) {
    g_perr = "target_size must be in [1, " + std::to_string(n) + "], got " +
             std::to_string(target_size);
    return 1;
  }
  std::vector<int64_t> d;
  neighbors_bfs(n, indptr, indices, 0, d);
  for (int64_t i = 0; i < n; ++i)
    if (d[i] < 0) {
      g_perr = "adjacency graph is not connected";
      return 1;
    }
  // k = int(round(n / target_size)) with round-half-even (Python round)
  const double q = static_cast<double>(n) / static_cast<double>(target_size);
  double fl = static_cast<double>(static_cast<int64_t>(q));
  double frac = q - fl;
  int64_t k = static_cast<int64_t>(fl);
  if (frac > 0.5 || (frac == 0.5 && (k % 2 == 1))) ++k;
  k = std::min(std::max<int64_t>(k, 1), n);

  neighbors_bfs(n, indptr, indices, start, d);
  auto argmax = [&](const std::vector<int64_t>& v) {
    return static_cast<int64_t>(std::max_element(v.begin(), v.end()) - v.begin());
  };
  std::vector<int64_t> seeds{argmax(d)};
  neighbors_bfs(n, indptr, indices, seeds[0], d);
  {
    // d = minimum(d, bfs(nxt)) by a BFS pruned at nodes that do not improve
    // (exact: d is a graph distance to the seed set, so it is 1-Lipschitz)
    ArgMaxTree tree(d);
    std::vector<int64_t> nd(n, -1);
    std::vector<int32_t> qu;
    std::vector<int32_t> touched;
    while (static_cast<int64_t>(seeds.size()) < k) {
      const int64_t nxt = tree.argmax();
      seeds.push_back(nxt);
      qu.clear();
      touched.clear();
      nd[nxt] = 0;
      touched.push_back(static_cast<int32_t>(nxt));
      qu.push_back(static_cast<int32_t>(nxt));
      if (d[nxt] != 0) {
        d[nxt] = 0;
        tree.set(nxt, 0);
      }
      for (size_t h = 0; h < qu.size(); ++h) {
        const int64_t u = qu[h];
        for (int64_t t = indptr[u]; t < indptr[u + 1]; ++t) {
          const int64_t v = indices[t];
          if (v == u || nd[v] >= 0) continue;
          const int64_t dv = nd[u] + 1;
          nd[v] = dv;
          touched.push_back(static_cast<int32_t>(v));
          if (dv < d[v]) {
            d[v] = dv;
            tree.set(v, dv);
            qu.push_back(static_cast<int32_t>(v));
          }
        }
      }
      for (int32_t v : touched) nd[v] = -1;
    }
  }

  // region growth (decomp.py:128-145)
  std::fill(owner, owner + n, -1);
  std::vector<int64_t> sizes(k, 0);
  std::vector<std::deque<int32_t>> queues(k);
  for (int64_t r = 0; r < k; ++r) {
    queues[r].push_back(static_cast<int32_t>(seeds[r]));
    owner[seeds[r]] = r;
    sizes[r] = 1;
  }
  // the reference assigns owner in seed order; a later seed overwrites an earlier
  // one if seeds coincide (sizes stay 1 each) — reproduced by the loop above.
  std::set<std::pair<int64_t, int64_t>> active;
  for (int64_t r = 0; r < k; ++r) active.insert({sizes[r], r});
  while (!active.empty()) {
    const int64_t r = active.begin()->second;
    auto& queue = queues[r];
    bool grew = false;
    const int64_t old = sizes[r];
    while (!queue.empty() && !grew) {
      const int64_t u = queue.front();
      queue.pop_front();
      for (int64_t t = indptr[u]; t < indptr[u + 1]; ++t) {
        const int64_t v = indices[t];
        if (v == u) continue;
        if (owner[v] < 0) {
          owner[v] = r;
          sizes[r]++;
          queue.push_back(static_cast<int32_t>(v));
          grew = true;
        }
      }
    }
    active.erase({old, r});
    if (!queue.empty() || grew) active.insert({sizes[r], r});
  }

  // smoothing pass (decomp.py:147-158) with _connected_without (:162-177)
  std::vector<std::vector<int32_t>> members(k);
  std::vector<int64_t> where(n);
  for (int64_t u = 0; u < n; ++u) {
    where[u] = static_cast<int64_t>(members[owner[u]].size());
    members[owner[u]].push_back(static_cast<int32_t>(u));
  }
  std::vector<int64_t> stamp(n, -1);
  std::vector<int32_t> stack;
  int64_t stamp_id = 0;
  std::vector<int64_t> nbr_regions;
  for (int64_t u = 0; u < n; ++u) {
    const int64_t r = owner[u];
    if (sizes[r] <= 1) continue;
    nbr_regions.clear();
    for (int64_t t = indptr[u]; t < indptr[u + 1]; ++t) {
      const int64_t v = indices[t];
      if (v == u) continue;
      if (owner[v] != r) nbr_regions.push_back(owner[v]);
    }
    int64_t best = -1;
    for (int64_t r2 : nbr_regions) {
      if (!(sizes[r2] + 1 < sizes[r])) continue;
      if (best < 0 || sizes[r2] < sizes[best] || (sizes[r2] == sizes[best] && r2 < best)) best = r2;
    }
    if (best < 0) continue;
    // connected_without(region r, drop u)
    const auto& mem = members[r];
    int64_t seed_node = -1;
    for (int32_t m : mem)
      if (m != u) {
        seed_node = m;
        break;
      }
    bool connected = false;
    if (seed_node >= 0) {
      ++stamp_id;
      stamp[u] = stamp_id;  // excluded
      stamp[seed_node] = stamp_id;
      stack.clear();
      stack.push_back(static_cast<int32_t>(seed_node));
      int64_t seen = 1;
      while (!stack.empty()) {
        const int64_t x = stack.back();
        stack.pop_back();
        for (int64_t t = indptr[x]; t < indptr[x + 1]; ++t) {
          const int64_t v = indices[t];
          if (v == x || owner[v] != r || stamp[v] == stamp_id) continue;
          stamp[v] = stamp_id;
          ++seen;
          stack.push_back(static_cast<int32_t>(v));
        }
      }
      connected = seen == static_cast<int64_t>(mem.size()) - 1;
    }
    if (connected) {
      // move u from r to best
      auto& mr = members[r];
      const int64_t w = where[u];
      const int32_t last = mr.back();
      mr[w] = last;
      where[last] = w;
      mr.pop_back();
      where[u] = static_cast<int64_t>(members[best].size());
      members[best].push_back(static_cast<int32_t>(u));
      owner[u] = best;
      sizes[r]--;
      sizes[best]++;
    }
  }
  return 0;
}

// decomp.py:196-216.  Two calls: sizes (sub_idx == NULL) then fill.
struct OverlapResult {
  std::vector<int64_t> ptr;
  std::vector<int64_t> idx;
};

void* ddmp_add_overlap(int64_t n, const int64_t* indptr, const int32_t* indices,
                       const int64_t* owner, int64_t overlap) {
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) k = std::max(k, owner[i] + 1);
  std::vector<std::vector<int32_t>> mem(k);
  for (int64_t i = 0; i < n; ++i) mem[owner[i]].push_back(static_cast<int32_t>(i));
  std::vector<std::vector<int64_t>> subs(k);
#pragma omp parallel
  {
    std::vector<int32_t> depth(n, -1);
    std::vector<int32_t> q;
#pragma omp for schedule(dynamic, 8)
    for (int64_t r = 0; r < k; ++r) {
      q.assign(mem[r].begin(), mem[r].end());
      for (int32_t u : q) depth[u] = 0;
      for (size_t h = 0; h < q.size(); ++h) {
        const int64_t u = q[h];
        if (depth[u] == overlap) continue;
        for (int64_t t = indptr[u]; t < indptr[u + 1]; ++t) {
          const int64_t v = indices[t];
          if (v == u) continue;
          if (depth[v] < 0) {
            depth[v] = depth[u] + 1;
            q.push_back(static_cast<int32_t>(v));
          }
        }
      }
      std::vector<int64_t> s(q.begin(), q.end());
      std::sort(s.begin(), s.end());
      for (int32_t u : q) depth[u] = -1;
      subs[r] = std::move(s);
    }
  }
  auto* R = new OverlapResult();
  R->ptr.assign(k + 1, 0);
  for (int64_t r = 0; r < k; ++r) R->ptr[r + 1] = R->ptr[r] + static_cast<int64_t>(subs[r].size());
  R->idx.resize(R->ptr[k]);
  for (int64_t r = 0; r < k; ++r) std::copy(subs[r].begin(), subs[r].end(), R->idx.begin() + R->ptr[r]);
  return R;
}

void ddmp_overlap_sizes(void* h, int64_t* k, int64_t* total) {
  auto* R = static_cast<OverlapResult*>(h);
  *k = static_cast<int64_t>(R->ptr.size()) - 1;
  *total = R->ptr.back();
}

void ddmp_overlap_copy(void* h, int64_t* ptr, int64_t* idx) {
  auto* R = static_cast<OverlapResult*>(h);
  std::copy(R->ptr.begin(), R->ptr.end(), ptr);
  std::copy(R->idx.begin(), R->idx.end(), idx);
}

void ddmp_overlap_free(void* h) { delete static_cast<OverlapResult*>(h); }

}  // extern "C"
