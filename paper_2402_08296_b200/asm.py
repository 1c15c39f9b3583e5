"""Setup-time coarse-space helpers (mirrors pkg/src/ddmgnn/asm.py:28-41).

The coarse matrix R0 A R0^T is assembled and factorised once per
preconditioner (as in the reference), then handed to the device as a dense
fp64 inverse that the per-apply coarse kernel multiplies (csrc/krylov.cu).
For K >= 512 the O(K^3) parts (rank check, LU) run on the GPU (cuSOLVER via
torch.linalg) — setup, not the per-apply path.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg
import scipy.sparse as sp

from .decomp import Decomposition
from .sparse import private_copy

__all__ = ["extract_local_matrix", "coarse_matrix", "coarse_inverse", "AsmPreconditioner",
           "build_asm", "apply_asm"]


def extract_local_matrix(a: sp.csr_matrix, idx: np.ndarray) -> sp.csr_matrix:
    """Principal submatrix R_i A R_i^T for an ascending index set (asm.py:28-32)."""
    sub = a[idx, :][:, idx].tocsr()
    sub.sort_indices()
    return sub


_GPU_SETUP_MIN_K = 512  # below this the host LAPACK path is as fast


def _setup_device():
    """CUDA device for the O(K^3) coarse setup, or None (small K / no GPU)."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        return None
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None


def _rank(gram: np.ndarray) -> int:
    """numpy.linalg.matrix_rank's rule (largest singular value x max(M, N) x eps) on the
    symmetric PSD Gram matrix, whose singular values are its eigenvalues — computed
    with the GPU's symmetric eigensolver for large K (the host SVD takes ~40 s at
    K = 1e4, BASELINE config D)."""
    k = gram.shape[0]
    dev = _setup_device() if k >= _GPU_SETUP_MIN_K else None
    if dev is None:
        return int(np.linalg.matrix_rank(gram))
    import torch

    ev = torch.linalg.eigvalsh(torch.as_tensor(gram, device=dev)).abs()
    tol = ev.max() * k * np.finfo(np.float64).eps
    return int((ev > tol).sum().item())


def coarse_matrix(a: sp.csr_matrix, dec: Decomposition) -> np.ndarray:
    """Dense K x K Galerkin coarse matrix after the R0 rank check (asm.py:35-41)."""
    r0 = dec.r0
    gram = (r0 @ r0.T).toarray()
    if _rank(gram) < dec.n_subdomains:
        raise RuntimeError("coarse rows are rank deficient")
    return (r0 @ a @ r0.T).toarray()


def coarse_inverse(cm: np.ndarray) -> np.ndarray:
    """Dense inverse through the reference's LU path (sparse.py:144-150).

    Raises the reference's "singular coarse matrix: matrix is exactly
    singular" (hybrid.py:93-96 wrapping sparse.py:147-148).
    """
    k = cm.shape[0]
    dev = _setup_device() if k >= _GPU_SETUP_MIN_K else None
    if dev is not None:  # same partial-pivoting LU (getrf/getrs) through cuSOLVER
        import torch

        m = torch.as_tensor(np.ascontiguousarray(cm), device=dev)
        lu, piv, info = torch.linalg.lu_factor_ex(m)
        if int(info.item()) > 0:
            raise RuntimeError("singular coarse matrix: matrix is exactly singular")
        eye = torch.eye(k, dtype=m.dtype, device=dev)
        return torch.linalg.lu_solve(lu, piv, eye).cpu().numpy()
    lu, piv = scipy.linalg.lu_factor(cm, check_finite=False)
    if np.any(np.diag(lu) == 0.0):
        raise RuntimeError("singular coarse matrix: matrix is exactly singular")
    return scipy.linalg.lu_solve((lu, piv), np.eye(k), check_finite=False)


# ---------------------------------------------------------------------------- DDM-LU


class AsmPreconditioner:
    """Additive Schwarz with exact local solves — the reference's DDM-LU comparator
    (asm.py:44-55; cli.py methods "ddm-lu-1" / "ddm-lu-2"), on the GPU: the local
    matrices are factorised once (cuSOLVER, dense inverses resident in HBM, 8 sum k_i^2
    bytes) and every apply is one kernel of per-subdomain GEMVs plus the gluing /
    coarse kernels shared with the GNN preconditioner."""

    def __init__(self, ctx, a, dec: Decomposition, level: str, coarse):
        from . import _lib

        self._ctx = ctx
        self.a = a
        self.dec = dec
        self.level = level
        self.coarse_matrix = coarse
        self._level_code = _lib.ASM_TWO if level == "two" else _lib.ASM_ONE

    @property
    def context(self):
        return self._ctx

    @property
    def n(self) -> int:
        return self.dec.n_dofs

    def __call__(self, r):
        return apply_asm(self, r)


class _DeviceView:
    """A library-owned device buffer as a torch tensor (no copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def build_asm(a: sp.csr_matrix, dec: Decomposition, level: str, device: int = 0,
              chunk_bytes: int = 1 << 30) -> AsmPreconditioner:
    """Extract and factorise all local (and, for level="two", coarse) matrices
    (asm.py:58-77) — batched dense inverses on the GPU (identity-padded to the
    batch's largest subdomain)."""
    import torch

    from . import _lib

    if level not in ("one", "two"):
        raise ValueError(f"level must be 'one' or 'two', got {level!r}")
    a = sp.csr_matrix(a)
    if not a.has_sorted_indices:
        a = a.copy()
        a.sort_indices()
    ctx = _lib.Context(device)
    ctx.set_matrix(a)
    ctx.set_geometry(np.zeros((dec.n_dofs, 2)))  # the exact solves need no geometry
    ctx.set_decomposition(dec.subdomains)
    ctx.build()
    sizes = np.array([s.size for s in dec.subdomains], dtype=np.int64)
    off = np.concatenate(([0], np.cumsum(sizes * sizes))).astype(np.int64)
    base = ctx.alloc_local_inverses(off)
    dev = torch.device("cuda", ctx.device)
    i, k_sub = 0, len(dec.subdomains)
    while i < k_sub:
        j, kmax = i + 1, int(sizes[i])
        while j < k_sub and (j - i + 1) * max(kmax, int(sizes[j])) ** 2 * 8 <= chunk_bytes:
            kmax = max(kmax, int(sizes[j]))
            j += 1
        batch = np.zeros((j - i, kmax, kmax))
        for t in range(i, j):
            k = int(sizes[t])
            batch[t - i, :k, :k] = extract_local_matrix(a, dec.subdomains[t]).toarray()
            batch[t - i, range(k, kmax), range(k, kmax)] = 1.0
        inv, info = torch.linalg.inv_ex(torch.as_tensor(batch, device=dev))
        bad = torch.nonzero(info).flatten()
        if bad.numel():  # asm.py:64-67
            raise RuntimeError(f"singular local matrix in subdomain {i + int(bad[0].item())}: "
                               "matrix is exactly singular")
        for t in range(i, j):
            k = int(sizes[t])
            if k:
                dst = torch.as_tensor(_DeviceView(base + 8 * int(off[t]), k * k), device=dev)
                dst.copy_(inv[t - i, :k, :k].reshape(-1))
        i = j
    torch.cuda.synchronize(dev)
    cm = None
    if level == "two":
        try:
            cm = coarse_matrix(a, dec)
            cinv = coarse_inverse(cm)
        except RuntimeError as exc:
            msg = str(exc)
            raise RuntimeError(msg if msg.startswith("singular coarse matrix")
                               else f"singular coarse matrix: {msg}") from exc
        ctx.set_coarse_inverse(cinv)
    return AsmPreconditioner(ctx, private_copy(a), dec, level, cm)


def apply_asm(p: AsmPreconditioner, r):
    """z = sum_i R_i^T A_i^-1 R_i r (+ coarse correction) (asm.py:98-113)."""
    from . import _lib

    n = p.n
    if type(r).__module__.startswith("torch") and getattr(r, "is_cuda", False):
        import torch

        if r.shape != (n,):
            raise ValueError(f"expected vector of length {n}, got shape {tuple(r.shape)}")
        r = r.to(dtype=torch.float64).contiguous()
        z = torch.empty_like(r)
        stream = torch.cuda.current_stream(r.device).cuda_stream or _lib.LEGACY_STREAM
        p.context.apply_device(r.data_ptr(), z.data_ptr(), p._level_code, stream, True)
        return z
    r = np.asarray(r, dtype=float)
    if r.shape != (n,):
        raise ValueError(f"expected vector of length {n}, got shape {r.shape}")
    return p.context.apply_host(r, p._level_code)

