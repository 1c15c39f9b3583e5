"""GPU training of DSS weights (last item) — the reference's
dataset harvesting (dataset.py:95-121) and training loop (dss.py:337-478,
train: Adam with global-norm clipping and plateau lr scheduling) on the GPU.

This is an offline tool around the product path, not part of it: it uses
PyTorch autograd on device tensors for the training arithmetic (fp64, the
reference's precision), the device-resident DDM-LU preconditioner
(`build_asm`) and PCG of this package for harvesting, and writes dss-v1 weight
files that `load_model` / `build_ddm_gnn` consume.

    harvest(problem, tol, max_iter)    -> list of (subdomain, c) local problems
    Trainer(k_bar, d).fit(train, val)  -> DssModel + per-epoch log
"""

from __future__ import annotations

import copy
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .asm import build_asm, extract_local_matrix
from .dss import DssModel
from .sparse import pcg

__all__ = ["LocalProblem", "harvest", "Trainer"]


@dataclass
class LocalProblem:
    """One training sample: a subdomain graph with its normalised residual c
    (hybrid.py:103-108 / dataset.py:108-114)."""

    edges: np.ndarray      # (E, 2) lexsorted local (src, dst)
    edge_vec: np.ndarray   # (E, 2)
    edge_len: np.ndarray   # (E,)
    a_local: sp.csr_matrix
    c: np.ndarray

    @property
    def node_count(self) -> int:
        return self.c.shape[0]


def _template(a, coords, idx):
    """Local graph of one subdomain (asm.py:28-32 + dss.py:173-186)."""
    a_loc = extract_local_matrix(a, idx)
    coo = a_loc.tocoo()
    m = coo.row != coo.col
    src, dst = coo.row[m].astype(np.int64), coo.col[m].astype(np.int64)
    order = np.lexsort((dst, src))
    edges = np.column_stack((src[order], dst[order]))
    c = np.asarray(coords)[idx]
    vec = c[edges[:, 1]] - c[edges[:, 0]]
    return edges, vec, np.hypot(vec[:, 0], vec[:, 1]), a_loc


def harvest(problem, tol: float = 1e-6, max_iter: int = 500, every: int = 1,
            max_samples: int | None = None, rng: np.random.Generator | None = None):
    """Solve with PCG + the exact two-level preconditioner and sample every
    subdomain's normalised residual at every application (dataset.py:95-121).
    Returns [] when the solve does not converge."""
    a, dec = problem.system.a, problem.dec
    asm2 = build_asm(a, dec, "two")
    templates = [_template(a, problem.coords, idx) for idx in dec.subdomains]
    residuals = []
    counter = {"it": 0}

    def harvesting_precond(r):
        if counter["it"] % every == 0:
            residuals.append(np.array(r, copy=True))
        counter["it"] += 1
        return asm2(r)

    _u, rep = pcg(a, problem.system.b, harvesting_precond, tol, max_iter)
    if not rep.converged:
        return []
    out = []
    for r in residuals:
        for i, idx in enumerate(dec.subdomains):
            ri = r[idx]
            s = float(np.linalg.norm(ri))
            if s > 0.0:
                e, v, ln, al = templates[i]
                out.append(LocalProblem(e, v, ln, al, ri / s))
    if max_samples is not None and len(out) > max_samples:
        rng = rng or np.random.default_rng(0)
        out = [out[j] for j in rng.choice(len(out), max_samples, replace=False)]
    return out


class _Batch:
    """Concatenated graphs on the device (dss.py:197-222)."""

    def __init__(self, samples, device):
        import torch

        counts = [s.node_count for s in samples]
        offs = np.concatenate(([0], np.cumsum(counts)))
        n = int(offs[-1])
        edges = np.vstack([s.edges + o for s, o in zip(samples, offs[:-1])])
        t = lambda x, dt=torch.float64: torch.as_tensor(x, dtype=dt, device=device)  # noqa: E731
        self.n = n
        self.src = t(edges[:, 0], torch.long)
        self.dst = t(edges[:, 1], torch.long)
        self.geo = t(np.column_stack((np.vstack([s.edge_vec for s in samples]),
                                      np.concatenate([s.edge_len for s in samples]))))
        self.c = t(np.concatenate([s.c for s in samples]))
        blk = sp.block_diag([s.a_local for s in samples], format="csr")
        self.a = torch.sparse_csr_tensor(t(blk.indptr, torch.long), t(blk.indices, torch.long),
                                         t(blk.data), size=(n, n), check_invariants=False)
        # 1/k_i per node: residual_loss is a per-graph mean (dss.py:330-336)
        self.inv_k = t(np.repeat(1.0 / np.asarray(counts, dtype=np.float64), counts))


class Trainer:
    """The reference's training recipe (dss.py:383-478) with autograd on the GPU."""

    def __init__(self, model: DssModel, device: int = 0):
        import torch

        self.d, self.k_bar, self.alpha = model.d, model.k_bar, model.alpha
        self.device = torch.device("cuda", device)
        self.model = copy.deepcopy(model)
        self.params = [torch.tensor(p, dtype=torch.float64, device=self.device,
                                    requires_grad=True) for p in _arrays(self.model)]

    # --- forward (dss.py:302-329) -----------------------------------------------------
    def _forward_loss(self, b: _Batch):
        import torch

        d = self.d
        h = torch.zeros((b.n, d), dtype=torch.float64, device=self.device)
        total = torch.zeros((), dtype=torch.float64, device=self.device)
        p = iter(self.params)
        for _k in range(self.k_bar):
            w1o, b1o, w2o, b2o = next(p), next(p), next(p), next(p)
            w1i, b1i, w2i, b2i = next(p), next(p), next(p), next(p)
            wp1, bp1, wp2, bp2 = next(p), next(p), next(p), next(p)
            wd1, bd1, wd2, bd2 = next(p), next(p), next(p), next(p)
            x_edge = torch.cat((h[b.src], h[b.dst], b.geo), dim=1)
            sign = torch.ones(2 * d + 3, 1, dtype=torch.float64, device=self.device)
            sign[2 * d:2 * d + 2] = -1.0  # in-MLP sees the reversed relative position
            z_o = torch.relu(x_edge @ w1o + b1o)
            z_i = torch.relu(x_edge @ (w1i * sign) + b1i)
            m_o = z_o @ w2o + b2o
            m_i = z_i @ w2i + b2i
            phi_o = torch.zeros((b.n, d), dtype=torch.float64, device=self.device).index_add(0, b.src, m_o)
            phi_i = torch.zeros((b.n, d), dtype=torch.float64, device=self.device).index_add(0, b.src, m_i)
            x_node = torch.cat((h, b.c[:, None], phi_o, phi_i), dim=1)
            h = h + self.alpha * (torch.relu(x_node @ wp1 + bp1) @ wp2 + bp2)
            out = (torch.relu(h @ wd1 + bd1) @ wd2 + bd2)[:, 0]
            res = torch.mv(b.a, out) - b.c
            total = total + (b.inv_k * res * res).sum()  # training_loss (dss.py:339-345)
        return total

    def evaluate(self, samples, batch_size: int = 100) -> float:
        import torch

        if not samples:
            return float("nan")
        with torch.no_grad():
            tot = 0.0
            for s in range(0, len(samples), batch_size):
                tot += float(self._forward_loss(_Batch(samples[s:s + batch_size], self.device)))
        return tot / len(samples)

    def fit(self, train, val, epochs: int, lr: float = 1e-2, batch_size: int = 100,
            clip_norm: float = 1e-2, factor: float = 0.1, patience: int = 10,
            min_lr: float = 1e-5, seed: int = 0, log_every: int = 0, on_epoch=None):
        """Adam + global-norm clipping + plateau schedule, as dss.py:392-469."""
        import torch

        if not train:
            raise ValueError("empty training set")
        beta1, beta2, eps = 0.9, 0.999, 1e-8
        m_state = [torch.zeros_like(p) for p in self.params]
        v_state = [torch.zeros_like(p) for p in self.params]
        rng = np.random.default_rng(seed)
        step, best, bad, log = 0, np.inf, 0, []
        batches_val = val
        for epoch in range(epochs):
            order = rng.permutation(len(train))
            loss_sum = 0.0
            for start in range(0, len(order), batch_size):
                chunk = [train[i] for i in order[start:start + batch_size]]
                b = _Batch(chunk, self.device)
                loss = self._forward_loss(b)
                if not torch.isfinite(loss):
                    raise RuntimeError(f"non-finite loss at epoch {epoch}")
                loss_sum += float(loss.detach())
                grads = torch.autograd.grad(loss, self.params)
                with torch.no_grad():
                    grads = [g / len(chunk) for g in grads]
                    gnorm = float(torch.sqrt(sum((g * g).sum() for g in grads)))
                    if gnorm > clip_norm and gnorm > 0:
                        grads = [g * (clip_norm / gnorm) for g in grads]
                    step += 1
                    bc1, bc2 = 1.0 - beta1 ** step, 1.0 - beta2 ** step
                    for p, m, v, g in zip(self.params, m_state, v_state, grads):
                        m.mul_(beta1).add_((1.0 - beta1) * g)
                        v.mul_(beta2).add_((1.0 - beta2) * g * g)
                        p.sub_(lr * (m / bc1) / (torch.sqrt(v / bc2) + eps))
            train_loss = loss_sum / len(train)
            val_loss = self.evaluate(batches_val, batch_size)
            log.append((epoch, train_loss, val_loss, lr))
            if log_every and epoch % log_every == 0:
                print(f"epoch {epoch} train {train_loss:.4e} val {val_loss:.4e} lr {lr:g}",
                      flush=True)
            if on_epoch is not None:  # e.g. solver-aware checkpoint selection
                on_epoch(epoch, self.to_model)
            if val:
                if val_loss < best:
                    best, bad = val_loss, 0
                else:
                    bad += 1
                    if bad > patience:
                        new_lr = max(lr * factor, min_lr)
                        if new_lr < lr:
                            lr = new_lr
                        bad = 0
        return self.to_model(), log

    def to_model(self) -> DssModel:
        m = copy.deepcopy(self.model)
        for dst, src in zip(_arrays(m), self.params):
            dst[...] = src.detach().cpu().numpy().reshape(dst.shape)
        return m


def _arrays(model: DssModel):
    """Parameter arrays in the reference's _param_arrays order (dss.py:93-99)."""
    out = []
    for w in model.layers:
        for mlp in (w.phi_out, w.phi_in, w.psi, w.dec):
            out.extend([mlp.w1, mlp.b1, mlp.w2, mlp.b2])
    return out
