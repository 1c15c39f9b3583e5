"""Multi-process CPU oracle of the DDM-GNN apply — TEST INFRASTRUCTURE ONLY.

Same arithmetic as ``oracle.ddm_oracle.OraclePreconditioner`` (the float64
restatement of the reference's ``apply_ddm_gnn``, hybrid.py:112-136, pinned
to reference goldens by tests/test_oracle_golden.py), spread over the host's
cores so that a full apply at BASELINE configs B/C (1.4M subdomain nodes at C)
takes seconds instead of half a minute:

* the K subdomains are split into contiguous slices, one per worker process
  (fork: the workers share A, coords and the subdomain index arrays copy-on-
  write); each worker builds its own templates (asm.py:28-32, dss.py:173-186)
  once and runs ``forward`` (dss.py:302-329) over its slice in
  ``plan_batches`` batches (hybrid.py:49-68, cap 100,000 nodes) on ONE BLAS
  thread, exactly as the reference does for its batches;
* the parent does what the reference does outside ``forward``: the coarse
  term ``r0.T @ lu_solve(r0 @ r)`` (hybrid.py:117, sparse.py:158-164) and the
  gluing ``z[idx_i] += s_i * sol_i`` in ascending subdomain order
  (hybrid.py:133-135), so z is the serial oracle's z (bitwise for the
  gluing; the per-batch GEMMs are row-independent, tests/test_hybrid.py:101-108
  of the reference checks batch invariance bitwise).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs use this module; the product package never imports oracle/.
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np
import scipy.linalg

from . import ddm_oracle as orc

_STATE = {}


def _worker(conn, lo, hi, offs):
    """Worker loop over subdomains [lo, hi).  Commands: ("apply",) ->
    reads r from the shared buffer, writes s_i and s_i*sol_i for its slice;
    ("model", flat, k_bar, d, alpha) -> swap weights; ("stop",)."""
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:  # pragma: no cover - threadpoolctl is part of the image
        pass
    st = _STATE
    a, coords, subs = st["a"], st["coords"], st["subs"]
    r_sh, out_sh, sc_sh = st["r"], st["out"], st["scale"]
    cap = st["cap"]
    model = st["model"]
    templates = {i: orc.local_graph(a, subs[i], coords) for i in range(lo, hi)}
    conn.send(("ready",))
    while True:
        msg = conn.recv()
        if msg[0] == "stop":
            conn.close()
            return
        if msg[0] == "model":
            model = orc.model_from_flat(msg[2], msg[3], msg[4], 0, msg[1])
            conn.send(("ok",))
            continue
        try:
            r = np.frombuffer(r_sh, dtype=np.float64)
            out = np.frombuffer(out_sh, dtype=np.float64)
            sc = np.frombuffer(sc_sh, dtype=np.float64)
            loaded = []
            for i in range(lo, hi):                         # hybrid.py:100-109
                r_i = r[subs[i]]
                s = float(np.linalg.norm(r_i))
                sc[i] = s
                if s == 0.0:
                    continue
                loaded.append((i, r_i / s, s))
            batches = orc.plan_batches([templates[i].node_count for i, _, _ in loaded], cap)
            for members in batches:                         # hybrid.py:121-131
                graphs = [templates[loaded[m][0]] for m in members]
                res = orc.forward(model, graphs, [loaded[m][1] for m in members])
                o = 0
                for m in members:
                    i, _c, s = loaded[m]
                    k = subs[i].size
                    local = res[o:o + k]
                    o += k
                    if not np.all(np.isfinite(local)):
                        raise RuntimeError(f"non-finite model output in subdomain {i}")
                    out[offs[i]:offs[i] + k] = s * local
            conn.send(("ok",))
        except Exception as exc:  # report, keep serving
            conn.send(("err", type(exc).__name__, str(exc)))


class ParallelOracle:
    """Restatement of build_ddm_gnn + apply_ddm_gnn (hybrid.py:84-136) over
    ``workers`` processes.  ``level`` "two" adds the coarse term (the
    reference); "one" starts from zeros (SURVEY.md finding 2)."""

    def __init__(self, a, coords, subdomains, model: orc.OracleModel, level: str = "two",
                 workers: int | None = None, batch_nodes_cap: int = 100_000):
        self.a = a.tocsr()
        self.n = self.a.shape[0]
        self.subs = [np.asarray(s, dtype=np.int64) for s in subdomains]
        self.level = level
        k = len(self.subs)
        sizes = np.array([s.size for s in self.subs], dtype=np.int64)
        self.offs = np.concatenate(([0], np.cumsum(sizes)))
        self.coarse = None
        self.weights, self.r0 = orc.finish_decomposition(self.subs, self.n)
        if level == "two":
            self.coarse = scipy.linalg.lu_factor(orc.coarse_matrix(self.a, self.r0),
                                                 check_finite=False)
        nw = max(1, min(workers or os.cpu_count() or 1, k))
        # contiguous slices balanced by subdomain nodes
        cuts = np.searchsorted(self.offs, np.linspace(0, self.offs[-1], nw + 1)[1:-1])
        bounds = np.unique(np.concatenate(([0], cuts, [k])))
        self._r = mp.RawArray("d", self.n)
        self._out = mp.RawArray("d", int(self.offs[-1]))
        self._scale = mp.RawArray("d", k)
        _STATE.update(a=self.a, coords=np.asarray(coords, dtype=float), subs=self.subs,
                      r=self._r, out=self._out, scale=self._scale, cap=batch_nodes_cap,
                      model=model)
        ctx = mp.get_context("fork")
        self._procs, self._conns = [], []
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            parent, child = ctx.Pipe()
            p = ctx.Process(target=_worker, args=(child, int(lo), int(hi), self.offs), daemon=True)
            p.start()
            child.close()
            self._procs.append(p)
            self._conns.append(parent)
        _STATE.clear()
        for c in self._conns:
            c.recv()
        self.workers = len(self._procs)

    # ------------------------------------------------------------------
    def set_model(self, model: orc.OracleModel):
        flat = np.concatenate([np.concatenate([x.ravel() for x in layer[nm]])
                               for layer in model.layers
                               for nm in ("phi_out", "phi_in", "psi", "dec")])
        for c in self._conns:
            c.send(("model", flat, model.k_bar, model.d, model.alpha))
        for c in self._conns:
            c.recv()

    def coarse_term(self, r):
        return self.r0.T @ scipy.linalg.lu_solve(self.coarse, self.r0 @ r, check_finite=False)

    def __call__(self, r):
        return self.apply(r)

    def apply(self, r, level: str | None = None):
        level = level or self.level
        r = np.asarray(r, dtype=float)
        if r.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got shape {r.shape}")
        np.frombuffer(self._r, dtype=np.float64)[:] = r
        for c in self._conns:
            c.send(("apply",))
        errs = [c.recv() for c in self._conns]
        for e in errs:
            if e[0] == "err":
                raise (RuntimeError if e[1] == "RuntimeError" else ValueError)(e[2])
        if level == "two":
            if self.coarse is None:
                raise ValueError("two-level apply needs the coarse factorisation")
            z = self.coarse_term(r)
        else:
            z = np.zeros(self.n)
        out = np.frombuffer(self._out, dtype=np.float64)
        sc = np.frombuffer(self._scale, dtype=np.float64)
        for i, idx in enumerate(self.subs):                 # hybrid.py:133-135
            if sc[i] == 0.0:
                continue
            z[idx] += out[self.offs[i]:self.offs[i + 1]]
        return z

    def close(self):
        for c in self._conns:
            try:
                c.send(("stop",))
            except (OSError, BrokenPipeError):
                pass
        for p in self._procs:
            p.join(timeout=10)
            if p.is_alive():
                p.kill()
        self._procs, self._conns = [], []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
