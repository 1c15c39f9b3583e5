"""Decomposition data contract (input format of the GPU path).

Mirrors pkg/src/ddmgnn/decomp.py:29-68 (Decomposition + JSON I/O),
:180-193 (_finish_decomposition: multiplicity partition of unity) and
:219-246 (restrict / extend / nicolaides).  The partitioner itself
(decomp.py:71-216) is an input producer and out of scope for this round.
These are setup-time host helpers; the per-apply restriction/prolongation
runs in the CUDA kernels.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

__all__ = ["Decomposition", "finish_decomposition", "restrict", "extend", "nicolaides"]


@dataclass(frozen=True)
class Decomposition:
    subdomains: list
    base_owner: np.ndarray
    overlap: int
    pou_weights: list
    r0: sp.csr_matrix

    @property
    def n_subdomains(self) -> int:
        return len(self.subdomains)

    @property
    def n_dofs(self) -> int:
        return self.base_owner.shape[0]

    def to_json(self) -> str:
        return json.dumps({"overlap": self.overlap, "owner": self.base_owner.tolist(),
                           "subdomains": [s.tolist() for s in self.subdomains]})

    @staticmethod
    def from_json(text: str) -> "Decomposition":
        obj = json.loads(text)
        subs = [np.asarray(s, dtype=np.int64) for s in obj["subdomains"]]
        owner = np.asarray(obj["owner"], dtype=np.int64)
        return finish_decomposition(subs, owner, int(obj["overlap"]))


def finish_decomposition(subdomains, owner, overlap: int) -> Decomposition:
    """PoU weights D_i = 1/multiplicity and R0 (decomp.py:180-193)."""
    owner = np.asarray(owner, dtype=np.int64)
    subdomains = [np.asarray(s, dtype=np.int64) for s in subdomains]
    n = owner.shape[0]
    multiplicity = np.zeros(n)
    for sub in subdomains:
        multiplicity[sub] += 1.0
    if np.any(multiplicity == 0):
        raise ValueError("subdomains do not cover all DOFs")
    weights = [1.0 / multiplicity[sub] for sub in subdomains]
    dec = Decomposition(subdomains, owner, overlap, weights, r0=None)
    object.__setattr__(dec, "r0", nicolaides(dec))
    return dec


def restrict(dec: Decomposition, i: int, x: np.ndarray) -> np.ndarray:
    x = np.asarray(x)
    if x.shape != (dec.n_dofs,):
        raise ValueError(f"expected global vector of length {dec.n_dofs}")
    return x[dec.subdomains[i]]


def extend(dec: Decomposition, i: int, v: np.ndarray) -> np.ndarray:
    v = np.asarray(v)
    sub = dec.subdomains[i]
    if v.shape != (sub.shape[0],):
        raise ValueError(f"expected local vector of length {sub.shape[0]}")
    out = np.zeros(dec.n_dofs)
    out[sub] = v
    return out


def nicolaides(dec: Decomposition) -> sp.csr_matrix:
    """K x N coarse matrix of PoU-weighted subdomain indicators (decomp.py:238-246)."""
    k, n = dec.n_subdomains, dec.n_dofs
    rows = np.concatenate([np.full(s.size, r) for r, s in enumerate(dec.subdomains)])
    cols = np.concatenate(dec.subdomains)
    vals = np.concatenate(dec.pou_weights)
    r0 = sp.csr_matrix((vals, (rows, cols)), shape=(k, n))
    r0.sort_indices()
    return r0
