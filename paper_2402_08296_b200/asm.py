"""Setup-time coarse-space helpers (mirrors pkg/src/ddmgnn/asm.py:28-41).

The coarse matrix R0 A R0^T is assembled and factorised once per
preconditioner (as in the reference), then handed to the device as a dense
fp64 inverse that the per-apply coarse kernel multiplies (csrc/krylov.cu).
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


def coarse_matrix(a: sp.csr_matrix, dec: Decomposition) -> np.ndarray:
    """Dense K x K Galerkin coarse matrix after the R0 rank check (asm.py:35-41)."""
    r0 = dec.r0
    gram = (r0 @ r0.T).toarray()
    if np.linalg.matrix_rank(gram) < dec.n_subdomains:
        raise RuntimeError("coarse rows are rank deficient")
    return (r0 @ a @ r0.T).toarray()


def coarse_inverse(cm: np.ndarray) -> np.ndarray:
    """Dense inverse through the reference's LU path (sparse.py:144-150).

    Raises the reference's "singular coarse matrix: matrix is exactly
    singular" (hybrid.py:93-96 wrapping sparse.py:147-148).
    """
    lu, piv = scipy.linalg.lu_factor(cm, check_finite=False)
    if np.any(np.diag(lu) == 0.0):
        raise RuntimeError("singular coarse matrix: matrix is exactly singular")
    return scipy.linalg.lu_solve((lu, piv), np.eye(cm.shape[0]), check_finite=False)
