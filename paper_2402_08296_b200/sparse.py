"""Device-resident Krylov solve: the drop-in for pkg/src/ddmgnn/sparse.py.

    pcg(a, b, precond, tol, max_iter, u0=None) -> (u, SolveReport)   sparse.py:76-127
    cg(a, b, tol, max_iter, u0=None)                                 sparse.py:130-132
    SolveReport                                                      sparse.py:31-53

The recurrence is the reference's Algorithm 1 exactly (standard PCG,
beta = rho_{k+1}/rho_k; ``flexible=True`` opts into flexible CG, Polak-Ribiere
beta = <r_{k+1}, z_{k+1} - z_k>/rho_k, which the reference does not have), run
on the GPU in fp64: CSR SpMV fused with <p,Ap>,
fused axpy + norm, the preconditioner kernels, all captured in a CUDA graph.
``precond`` may be
  * a DdmGnnPreconditioner built on the same matrix -> fully on device;
  * None -> plain CG on device;
  * any other callable r -> z -> the Krylov loop stays on the device and the
    callable is invoked on host copies of r (the reference's operator hook).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib

__all__ = ["SolveReport", "validate_csr", "pcg", "fcg", "cg", "Ic0Preconditioner", "ic0"]


@dataclass
class SolveReport:
    """Iteration record of one Krylov solve (sparse.py:31-53)."""

    iterations: int
    residual_history: list
    converged: bool
    final_relres: float
    tolerance: float = field(default=0.0, repr=False)

    def to_json(self) -> str:
        return json.dumps({"iterations": self.iterations, "converged": self.converged,
                           "final_relres": self.final_relres,
                           "residual_history": self.residual_history})


def validate_csr(a: sp.csr_matrix) -> None:
    """CSR structural invariants (sparse.py:56-67)."""
    n_rows, n_cols = a.shape
    indptr, indices = a.indptr, a.indices
    if indptr[0] != 0 or indptr[-1] != a.nnz or len(indptr) != n_rows + 1:
        raise ValueError("malformed indptr")
    if np.any(np.diff(indptr) < 0):
        raise ValueError("indptr not nondecreasing")
    d = np.diff(indices)
    row_of = np.repeat(np.arange(n_rows), np.diff(indptr))
    same_row = row_of[1:] == row_of[:-1]
    # the reference scans rows in order and reports the first row that breaks
    # either rule (sparse.py:64-67)
    bad_rows = np.zeros(n_rows, dtype=bool)
    bad_rows[row_of[1:][same_row & (d <= 0)]] = True
    bad_rows[row_of[(indices < 0) | (indices >= n_cols)]] = True
    if np.any(bad_rows):
        r = int(np.argmax(bad_rows))
        raise ValueError(f"row {r}: columns not strictly increasing in range")


_solver_cache: dict = {}


def private_copy(a: sp.csr_matrix) -> sp.csr_matrix:
    """A CSR copy that shares no array with the caller's matrix: device contexts
    remember the matrix they hold through it, so an in-place edit of the caller's
    ``a.data`` is seen as a different matrix (the reference recomputes ``a @ p``
    on every call, sparse.py:107)."""
    return sp.csr_matrix((a.data.copy(), a.indices.copy(), a.indptr.copy()), shape=a.shape)


def _same_matrix(a, b) -> bool:
    return (a.shape == b.shape and a.nnz == b.nnz and np.array_equal(a.indptr, b.indptr)
            and np.array_equal(a.indices, b.indices) and np.array_equal(a.data, b.data))


def _solver_ctx(a, device: int = 0) -> _lib.Context:
    """A context holding only the matrix (plain CG / host preconditioners)."""
    hit = _solver_cache.get(device)
    if hit is not None and _same_matrix(hit[0], a):
        return hit[1]
    ctx = _lib.Context(device)
    ctx.set_matrix(a)
    _solver_cache[device] = (private_copy(a), ctx)
    return ctx


def _as_csr(a):
    a = sp.csr_matrix(a)
    if not a.has_sorted_indices:
        a = a.copy()
        a.sort_indices()
    return a


def pcg(a, b, precond, tol: float, max_iter: int, u0=None, flexible: bool = False):
    """Preconditioned conjugate gradient on the GPU; returns (u, SolveReport).

    ``flexible=True``: flexible CG (beta = <r', z' - z>/rho) for nonlinear
    preconditioners such as the GNN operator; an addition to the reference API
    (its default, False, is the reference's recurrence, sparse.py:122-126)."""
    from .hybrid import DdmGnnPreconditioner

    if tol <= 0:
        raise ValueError("tol must be positive")
    b = np.asarray(b, dtype=float)
    n = b.shape[0]
    if u0 is not None:
        u0 = np.asarray(u0, dtype=float)
        if u0.shape != (n,):
            raise ValueError("u0 dimension mismatch")
    a = _as_csr(a)
    if a.shape != (n, n):  # the reference fails in `b - a @ u` (sparse.py:96)
        raise ValueError("dimension mismatch")
    from .asm import AsmPreconditioner

    if isinstance(precond, (DdmGnnPreconditioner, AsmPreconditioner, Ic0Preconditioner)) and \
            _same_matrix(precond.a, a):
        ctx, level = precond.context, precond._level_code
        u, it, hist, conv = ctx.pcg(b, u0, tol, max_iter, level, flexible=flexible)
    elif precond is None:
        u, it, hist, conv = _solver_ctx(a).pcg(b, u0, tol, max_iter, _lib.PRECOND_NONE,
                                               flexible=flexible)
    else:
        fn = precond if callable(precond) else precond.__call__
        u, it, hist, conv = _solver_ctx(a).pcg_host_precond(b, u0, tol, max_iter, fn,
                                                            flexible=flexible)
    return u, SolveReport(it, hist, conv, hist[-1], tol)


def fcg(a, b, precond, tol: float, max_iter: int, u0=None):
    """Flexible CG (opt-in; ``pcg(..., flexible=True)``)."""
    return pcg(a, b, precond, tol, max_iter, u0=u0, flexible=True)


def cg(a, b, tol: float, max_iter: int, u0=None):
    """Unpreconditioned conjugate gradient (sparse.py:130-132)."""
    return pcg(a, b, None, tol, max_iter, u0=u0)


class Ic0Preconditioner:
    """Zero-fill incomplete Cholesky x -> L^-T (L^-1 x) (sparse.py:170-179), on the GPU:
    factorised once on the host (the reference's algorithm, sparse.py:184-227), applied
    with two sync-free triangular-solve kernels (csrc/ic0.cu)."""

    def __init__(self, ctx, a):
        self._ctx = ctx
        self.a = a
        self._level_code = _lib.IC0

    @property
    def context(self):
        return self._ctx

    @property
    def l(self) -> sp.csr_matrix:  # noqa: E743 — the reference's attribute name
        ip, ix, dv = self._ctx.export_ic0()
        n = ip.size - 1
        return sp.csr_matrix((dv, ix, ip), shape=(n, n))

    def __call__(self, x):
        x = np.asarray(x, dtype=float)
        n = self.a.shape[0]
        if x.shape != (n,):  # the reference's spsolve_triangular raises (sparse.py:177-179)
            raise ValueError(f"expected vector of length {n}, got shape {x.shape}")
        return self._ctx.apply_host(x, self._level_code)


def ic0(a: sp.csr_matrix, device: int = 0) -> Ic0Preconditioner:
    """Incomplete Cholesky with zero fill on the lower-triangular pattern of A
    (sparse.py:184-227): RuntimeError("IC(0) breakdown ...") on a missing diagonal or
    a nonpositive pivot, no diagonal shift."""
    a = sp.csr_matrix(a)
    if not a.has_sorted_indices:
        a = a.copy()
        a.sort_indices()
    ctx = _lib.Context(device)
    ctx.set_matrix(a)
    ctx.set_ic0()
    return Ic0Preconditioner(ctx, private_copy(a))

