"""CPU oracle for the DDM-GNN hot path — TEST INFRASTRUCTURE ONLY.

This module is the *checker*, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2402_08296_b200``) never imports anything under ``oracle/``.

It restates, in float64 numpy/scipy, the reference package ``ddmgnn`` 0.1.0
(read-only at /root/reference; citations are ``pkg/src/ddmgnn/<file>:<line>``):

* ``local_graph``        — asm.py:28-32 (extract_local_matrix) + dss.py:173-186
                           (local_graph_from_matrix)
* ``finish_decomposition`` — decomp.py:180-193 (_finish_decomposition) +
                           decomp.py:238-246 (nicolaides)
* ``coarse_matrix``      — asm.py:35-41
* ``forward``            — dss.py:257-258, 273-299, 302-329
* ``apply_ddm_gnn``      — hybrid.py:100-136 (two-level) and the one-level
                           restatement (same lines with z initialised to zero
                           instead of hybrid.py:117; SURVEY.md finding 2)
* ``pcg``                — sparse.py:76-127
* ``load_model``/``model_layers`` — dss.py:93-99, 547-571 (dss-v1 format)

Parity pinning: the restatement is checked against golden vectors produced by
the reference itself (tests/golden/make_golden.py imports /root/reference and
commits the outputs); see tests/test_oracle_golden.py.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse as sp

# ---------------------------------------------------------------------------
# model format (dss.py:54-99, 530-571)


@dataclass
class OracleModel:
    k_bar: int
    d: int
    alpha: float
    seed: int
    # per layer: dict name -> (w1, b1, w2, b2) for phi_out, phi_in, psi, dec
    layers: list


def _mlp_shapes(d: int):
    """Canonical per-layer MLP shapes in serialization order (dss.py:93-99, 117-123)."""
    return (
        ("phi_out", 2 * d + 3, d, d),
        ("phi_in", 2 * d + 3, d, d),
        ("psi", 3 * d + 1, d, d),
        ("dec", d, d, 1),
    )


def model_from_flat(k_bar: int, d: int, alpha: float, seed: int, flat: np.ndarray) -> OracleModel:
    """Split a flat float64 parameter vector in `_param_arrays` order (dss.py:93-99)."""
    flat = np.asarray(flat, dtype=np.float64)
    pos = 0
    layers = []
    for _ in range(k_bar):
        layer = {}
        for name, n_in, n_hid, n_out in _mlp_shapes(d):
            w1 = flat[pos : pos + n_in * n_hid].reshape(n_in, n_hid); pos += n_in * n_hid
            b1 = flat[pos : pos + n_hid]; pos += n_hid
            w2 = flat[pos : pos + n_hid * n_out].reshape(n_hid, n_out); pos += n_hid * n_out
            b2 = flat[pos : pos + n_out]; pos += n_out
            layer[name] = (w1, b1, w2, b2)
        layers.append(layer)
    if pos != flat.size:
        raise ValueError("flat parameter vector has the wrong length")
    return OracleModel(k_bar, d, alpha, seed, layers)


def load_model(path: str) -> OracleModel:
    """dss-v1 reader (dss.py:547-571)."""
    with open(path, "rb") as fh:
        header = json.loads(fh.readline().decode("ascii"))
        blob = fh.read()
    if header.get("format") != "dss-v1":
        raise ValueError("unsupported model format")
    return model_from_flat(int(header["k_bar"]), int(header["d"]), float(header["alpha"]),
                           int(header["seed"]), np.frombuffer(blob, dtype="<f8"))


def init_model_flat(k_bar: int, d: int, seed: int) -> np.ndarray:
    """Xavier-uniform init in the reference draw order (dss.py:102-127)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(k_bar):
        for _name, n_in, n_hid, n_out in _mlp_shapes(d):
            a1 = np.sqrt(6.0 / (n_in + n_hid))
            w1 = rng.uniform(-a1, a1, (n_in, n_hid))
            a2 = np.sqrt(6.0 / (n_hid + n_out))
            w2 = rng.uniform(-a2, a2, (n_hid, n_out))
            out += [w1.ravel(), np.zeros(n_hid), w2.ravel(), np.zeros(n_out)]
    return np.concatenate(out)


# ---------------------------------------------------------------------------
# decomposition + local graphs


def finish_decomposition(subdomains, n: int):
    """PoU weights and R0 (decomp.py:180-193, 238-246)."""
    multiplicity = np.zeros(n)
    for sub in subdomains:
        multiplicity[sub] += 1.0
    if np.any(multiplicity == 0):
        raise ValueError("subdomains do not cover all DOFs")
    weights = [1.0 / multiplicity[sub] for sub in subdomains]
    rows = np.concatenate([np.full(s.size, r) for r, s in enumerate(subdomains)])
    cols = np.concatenate(subdomains)
    vals = np.concatenate(weights)
    r0 = sp.csr_matrix((vals, (rows, cols)), shape=(len(subdomains), n))
    r0.sort_indices()
    return weights, r0


@dataclass
class OracleGraph:
    coords: np.ndarray
    edges: np.ndarray      # (E, 2) lexsorted (src, dst)
    edge_vec: np.ndarray   # (E, 2)
    edge_len: np.ndarray   # (E,)
    a_local: sp.csr_matrix

    @property
    def node_count(self) -> int:
        return self.coords.shape[0]


def local_graph(a: sp.csr_matrix, idx: np.ndarray, coords: np.ndarray) -> OracleGraph:
    """asm.py:28-32 then dss.py:173-186."""
    a_loc = a[idx, :][:, idx].tocsr()
    a_loc.sort_indices()
    coo = a_loc.tocoo()
    mask = coo.row != coo.col
    src = coo.row[mask].astype(np.int64)
    dst = coo.col[mask].astype(np.int64)
    order = np.lexsort((dst, src))
    edges = np.column_stack((src[order], dst[order]))
    c = np.asarray(coords, dtype=float)[idx]
    edge_vec = c[edges[:, 1]] - c[edges[:, 0]]
    edge_len = np.hypot(edge_vec[:, 0], edge_vec[:, 1])
    return OracleGraph(c, edges, edge_vec, edge_len, a_loc)


def coarse_matrix(a: sp.csr_matrix, r0: sp.csr_matrix) -> np.ndarray:
    """asm.py:35-41 (rank check + dense R0 A R0^T)."""
    gram = (r0 @ r0.T).toarray()
    if np.linalg.matrix_rank(gram) < r0.shape[0]:
        raise RuntimeError("coarse rows are rank deficient")
    return (r0 @ a @ r0.T).toarray()


# ---------------------------------------------------------------------------
# forward (dss.py:257-329), float64


def _mlp(p, x):
    w1, b1, w2, b2 = p
    return np.maximum(x @ w1 + b1, 0.0) @ w2 + b2


def forward(model: OracleModel, graphs, c_list, return_all: bool = False):
    """Batched forward over concatenated graphs (dss.py:197-222, 302-329).

    Returns the final decoded output (concatenated); raises the reference's
    RuntimeError on a non-finite latent state.
    """
    d = model.d
    counts = [g.node_count for g in graphs]
    offs = np.concatenate(([0], np.cumsum(counts)))
    n_nodes = int(offs[-1])
    edges = np.vstack([g.edges + o for g, o in zip(graphs, offs[:-1])])
    edge_vec = np.vstack([g.edge_vec for g in graphs])
    edge_len = np.concatenate([g.edge_len for g in graphs])
    c = np.concatenate(c_list)
    n_edges = edges.shape[0]
    scatter_src = sp.csr_matrix((np.ones(n_edges), (edges[:, 0], np.arange(n_edges))),
                                shape=(n_nodes, n_edges))
    src, dst = edges[:, 0], edges[:, 1]
    x_edge = np.empty((n_edges, 2 * d + 3))
    x_edge[:, 2 * d : 2 * d + 2] = edge_vec
    x_edge[:, 2 * d + 2] = edge_len
    h = np.zeros((n_nodes, d))
    outputs = []
    for k, layer in enumerate(model.layers, start=1):
        np.take(h, src, axis=0, out=x_edge[:, :d])
        np.take(h, dst, axis=0, out=x_edge[:, d : 2 * d])
        w_out, b_out = layer["phi_out"][0], layer["phi_out"][1]
        w_in = layer["phi_in"][0].copy()
        w_in[2 * d : 2 * d + 2] *= -1.0
        w1_cat = np.hstack((w_out, w_in))
        b1_cat = np.concatenate((b_out, layer["phi_in"][1]))
        z_cat = x_edge @ w1_cat
        z_cat += b1_cat
        np.maximum(z_cat, 0.0, out=z_cat)
        m_out = z_cat[:, :d] @ layer["phi_out"][2] + layer["phi_out"][3]
        m_in = z_cat[:, d:] @ layer["phi_in"][2] + layer["phi_in"][3]
        phi_o = scatter_src @ m_out
        phi_i = scatter_src @ m_in
        x_node = np.empty((n_nodes, 3 * d + 1))
        x_node[:, :d] = h
        x_node[:, d] = c
        x_node[:, d + 1 : 2 * d + 1] = phi_o
        x_node[:, 2 * d + 1 :] = phi_i
        h = h + model.alpha * _mlp(layer["psi"], x_node)
        if not np.all(np.isfinite(h)):
            raise RuntimeError(f"non-finite latent state at message-passing iteration {k}")
        outputs.append(_mlp(layer["dec"], h)[:, 0])
    return outputs if return_all else outputs[-1]


# ---------------------------------------------------------------------------
# preconditioner apply (hybrid.py:49-136)


class OraclePreconditioner:
    """Restatement of build_ddm_gnn (hybrid.py:84-97) + apply (hybrid.py:112-136)."""

    def __init__(self, a, coords, subdomains, model: OracleModel, level: str = "two",
                 batch_nodes_cap: int = 100_000):
        self.a = a.tocsr()
        self.n = a.shape[0]
        self.subdomains = [np.asarray(s, dtype=np.int64) for s in subdomains]
        self.weights, self.r0 = finish_decomposition(self.subdomains, self.n)
        self.templates = [local_graph(self.a, s, coords) for s in self.subdomains]
        self.model = model
        self.level = level
        self.cap = batch_nodes_cap
        self.coarse = None
        if level == "two":
            cm = coarse_matrix(self.a, self.r0)
            self.coarse = scipy.linalg.lu_factor(cm, check_finite=False)

    def coarse_term(self, r):
        return self.r0.T @ scipy.linalg.lu_solve(self.coarse, self.r0 @ r, check_finite=False)

    def __call__(self, r):
        return self.apply(r)

    def apply(self, r):
        r = np.asarray(r, dtype=float)
        if r.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got shape {r.shape}")
        z = self.coarse_term(r) if self.level == "two" else np.zeros(self.n)
        loaded = []
        for i, idx in enumerate(self.subdomains):        # hybrid.py:100-109
            r_i = r[idx]
            scale = float(np.linalg.norm(r_i))
            if scale == 0.0:
                continue
            loaded.append((i, r_i / scale, scale))
        solutions = {}
        batches = plan_batches([self.templates[i].node_count for i, _, _ in loaded], self.cap)
        for members in batches:                           # hybrid.py:121-131
            graphs = [self.templates[loaded[m][0]] for m in members]
            out = forward(self.model, graphs, [loaded[m][1] for m in members])
            offs = np.concatenate(([0], np.cumsum([g.node_count for g in graphs])))
            for m, s0, s1 in zip(members, offs[:-1], offs[1:]):
                local = out[s0:s1]
                if not np.all(np.isfinite(local)):
                    raise RuntimeError(f"non-finite model output in subdomain {loaded[m][0]}")
                solutions[loaded[m][0]] = local
        for i, _c, scale in loaded:                       # hybrid.py:133-135
            z[self.subdomains[i]] += scale * solutions[i]
        return z


def plan_batches(node_counts, cap: int):
    """hybrid.py:49-68."""
    if cap < 1:
        raise ValueError("batch node cap must be >= 1")
    batches, current, load = [], [], 0
    for i, count in enumerate(node_counts):
        if current and load + count > cap:
            batches.append(current)
            current, load = [], 0
        current.append(i)
        load += count
    if current:
        batches.append(current)
    return batches


# ---------------------------------------------------------------------------
# PCG (sparse.py:76-127)


def pcg(a, b, precond, tol: float, max_iter: int, u0=None, flexible: bool = False):
    """Returns (u, iterations, history, converged).

    ``flexible=True`` is the opt-in flexible CG (Polak-Ribiere beta,
    beta = <r_k+1, z_k+1 - z_k> / <r_k, z_k>; Notay 2000) that the
    reference does NOT have (SURVEY.md finding 3): the SURVEY's flexible-CG
    probe recipe (appendix).  Every other line is sparse.py:76-127; with a
    linear SPD preconditioner it equals PCG in exact arithmetic."""
    if tol <= 0:
        raise ValueError("tol must be positive")
    b = np.asarray(b, dtype=float)
    n = b.shape[0]
    u = np.zeros(n) if u0 is None else np.asarray(u0, dtype=float).copy()
    norm_b = float(np.linalg.norm(b))
    if norm_b == 0.0:
        return np.zeros(n), 0, [0.0], True
    r = b - a @ u
    history = [float(np.linalg.norm(r)) / norm_b]
    if history[0] < tol:
        return u, 0, history, True
    z = precond(r) if precond is not None else r
    p = z.copy()
    rho = float(r @ z)
    iterations = 0
    converged = False
    for _ in range(max_iter):
        q = a @ p
        pq = float(p @ q)
        if pq <= 0:
            raise RuntimeError("matrix not SPD: <p, Ap> <= 0")
        alpha = rho / pq
        u = u + alpha * p
        r = r - alpha * q
        rel = float(np.linalg.norm(r)) / norm_b
        if not np.isfinite(rel):
            raise RuntimeError(f"non-finite residual at iteration {iterations + 1}")
        history.append(rel)
        iterations += 1
        if rel < tol:
            converged = True
            break
        z_old = z
        z = precond(r) if precond is not None else r
        rho_next = float(r @ z)
        beta = (float(r @ (z - z_old)) if flexible else rho_next) / rho
        rho = rho_next
        p = z + beta * p
    return u, iterations, history, converged


def gnn_flops(k_bar: int, d: int, v: int, e: int) -> float:
    """Minimal factorised FP32 flop count of one GNN apply."""
    per_node = 8 * d * d + 2 * d + 4 * d * d + 4 * d + 2 * (3 * d + 1) * d + 2 * d * d + 2 * d + 2 * d
    per_edge = 2 * d * 8
    return float(k_bar * (per_node * v + per_edge * e) + (2 * d * d + 2 * d) * v)
