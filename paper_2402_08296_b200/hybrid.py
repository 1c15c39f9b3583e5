"""DDM-GNN preconditioner on B200: the drop-in for pkg/src/ddmgnn/hybrid.py.

    build_ddm_gnn(a, coords, dec, model, batch_nodes_cap=100_000)   hybrid.py:84-97
    DdmGnnPreconditioner.__call__(r) -> z                          hybrid.py:71-81
    apply_ddm_gnn(p, r) -> z                                       hybrid.py:112-136
    plan_batches(node_counts, cap)                                 hybrid.py:49-68

Same signatures, argument meaning and error behaviour as the reference, with
one addition: ``level`` ("two" = the reference's two-level operator, default;
"one" = local GNN solves only, the one-level variant BASELINE config B asks
for).  Everything per-apply runs in CUDA kernels for sm_100a through the C ABI
(include/ddmgnn_b200.h): fused restriction + message passing + decoder per
subdomain, dense coarse solve, gather-based prolongation.  ``r`` may be a numpy
array (host round trip, the reference's calling convention) or a CUDA float64
torch tensor (zero-copy, returns a CUDA tensor).  There is no CPU fallback.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import _lib
from .asm import coarse_inverse, coarse_matrix
from .decomp import Decomposition
from .dss import DssModel, flat_params
from .sparse import private_copy

__all__ = ["DdmGnnPreconditioner", "build_ddm_gnn", "apply_ddm_gnn", "plan_batches",
           "LocalGraphView"]

_LEVELS = {"one": _lib.LEVEL_ONE, "two": _lib.LEVEL_TWO}


def plan_batches(node_counts, cap: int) -> list:
    """Greedy in-order packing of graphs into batches of at most ``cap`` nodes.

    Kept for API parity (hybrid.py:49-68).  The device path processes every
    subdomain in one launch; results never depend on the cap, which only fixes
    the order in which the reference would report non-finite states.
    """
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


class LocalGraphView:
    """Read-back of one subdomain graph as built on the device (parity checks)."""

    def __init__(self, src, dst, vec):
        self.edges = np.column_stack((src.astype(np.int64), dst.astype(np.int64)))
        self.edge_vec = vec[:, :2]
        self.edge_len = vec[:, 2]


class DdmGnnPreconditioner:
    """Device-resident DDM-GNN operator (hybrid.py:71-81)."""

    def __init__(self, ctx: _lib.Context, a, dec: Decomposition, model: DssModel, level: str,
                 batch_nodes_cap: int, coarse: np.ndarray | None):
        self._ctx = ctx
        self.a = a
        self.dec = dec
        self.model = model
        self.level = level
        self.batch_nodes_cap = batch_nodes_cap
        self.coarse_matrix = coarse
        self._level_code = _LEVELS[level]

    @property
    def context(self) -> _lib.Context:
        return self._ctx

    @property
    def n(self) -> int:
        return self.dec.n_dofs

    def info(self) -> dict:
        return self._ctx.info()

    def local_graph(self, i: int) -> LocalGraphView:
        return LocalGraphView(*self._ctx.export_local_graph(i))

    def reload_model(self, model: DssModel | None = None) -> None:
        """Re-upload weights (after editing ``self.model`` in place)."""
        if model is not None:
            self.model = model
        m = self.model
        self._ctx.set_model(m.k_bar, m.d, m.alpha, flat_params(m))

    def __call__(self, r):
        return apply_ddm_gnn(self, r)


def build_ddm_gnn(a: sp.csr_matrix, coords: np.ndarray, dec: Decomposition, model: DssModel,
                  batch_nodes_cap: int = 100_000, level: str = "two",
                  device: int = 0) -> DdmGnnPreconditioner:
    """Precompute the device layout and factorise the coarse matrix (hybrid.py:84-97)."""
    if level not in _LEVELS:
        raise ValueError(f"level must be 'one' or 'two', got {level!r}")
    if batch_nodes_cap < 1:
        raise ValueError("batch node cap must be >= 1")
    a = sp.csr_matrix(a)
    if not a.has_sorted_indices:
        a = a.copy()
        a.sort_indices()
    coords = np.asarray(coords, dtype=float)
    if coords.shape != (dec.n_dofs, 2):
        raise ValueError(f"expected coords of shape ({dec.n_dofs}, 2)")
    ctx = _lib.Context(device)
    ctx.set_matrix(a)
    ctx.set_geometry(coords)
    ctx.set_decomposition(dec.subdomains)
    ctx.set_batch_cap(batch_nodes_cap)
    ctx.build()
    ctx.set_model(model.k_bar, model.d, model.alpha, flat_params(model))
    cm = None
    if level == "two":
        # the reference always factorises the coarse matrix (hybrid.py:93-96)
        try:
            cm = coarse_matrix(a, dec)
            inv = coarse_inverse(cm)
        except RuntimeError as exc:
            msg = str(exc)
            raise RuntimeError(msg if msg.startswith("singular coarse matrix")
                               else f"singular coarse matrix: {msg}") from exc
        ctx.set_coarse_inverse(inv)
    # private copy: pcg() recognises "its" matrix by content, not identity
    return DdmGnnPreconditioner(ctx, private_copy(a), dec, model, level, batch_nodes_cap, cm)


def _is_torch_cuda(x) -> bool:
    t = type(x)
    return t.__module__.startswith("torch") and getattr(x, "is_cuda", False)


def apply_ddm_gnn(p: DdmGnnPreconditioner, r):
    """z = M r (hybrid.py:112-136), computed on the GPU."""
    n = p.n
    if _is_torch_cuda(r):
        import torch

        if r.shape != (n,):
            raise ValueError(f"expected vector of length {n}, got shape {tuple(r.shape)}")
        r = r.to(dtype=torch.float64).contiguous()
        z = torch.empty_like(r)
        # torch's default stream is the legacy NULL stream: pass cudaStreamLegacy (0x1)
        stream = torch.cuda.current_stream(r.device).cuda_stream or _lib.LEGACY_STREAM
        p.context.apply_device(r.data_ptr(), z.data_ptr(), p._level_code, stream, True)
        return z
    r = np.asarray(r, dtype=float)
    if r.shape != (n,):
        raise ValueError(f"expected vector of length {n}, got shape {r.shape}")
    return p.context.apply_host(r, p._level_code)
