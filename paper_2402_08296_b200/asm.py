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

__all__ = ["extract_local_matrix", "coarse_matrix", "coarse_inverse"]


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
