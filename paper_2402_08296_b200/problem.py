"""Problem setup (input producers) with the reference's exact semantics.

Ports of the reference's O(N)/O(K*N) Python set-up loops to native code
(csrc/problem.cpp, host-only) so that the 100k / 1M / 10M-node BASELINE
configurations can be built on the GPU host in seconds:

    generate_blob_mesh(seed, target_nodes, perturbation)   mesh.py:153-207
    assemble(mesh, coeffs)                                  fem.py:91-173
    partition(a, target_size, seed)                         decomp.py:92-159
    add_overlap(owner, a, overlap)                          decomp.py:196-216
    sample_coeffs(rng), build_problem(seed, config)         dataset.py:79-92

All floating-point expressions the reference evaluates with numpy (ring
coordinates, element matrices, load vector, Dirichlet data) are evaluated
here with the *same* numpy expressions, and the native code reproduces the
reference's loop and accumulation order, so outputs are bit-identical to the
reference on the same machine (tests/test_problem_builder.py).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .decomp import Decomposition, finish_decomposition

__all__ = ["Mesh", "PolyCoeffs", "LinearSystem", "ProblemConfig", "Problem", "generate_blob_mesh",
           "assemble", "partition", "add_overlap", "sample_coeffs", "build_problem"]

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libddmgnn_problem.so")
_plib = None

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p


def _lib():
    global _plib
    if _plib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} not built (make -C paper_2402_08296_b200/csrc)")
        L = ctypes.CDLL(_LIB_PATH)
        L.ddmp_last_error.restype = ctypes.c_char_p
        L.ddmp_blob_triangles.restype = _i64
        L.ddmp_blob_triangles.argtypes = [_i64, _vp, _vp]
        L.ddmp_boundary_flags.argtypes = [_i64, _i64, _vp, _vp]
        L.ddmp_assemble.restype = _vp
        L.ddmp_assemble.argtypes = [_i64, _i64, _vp, _vp, _vp, _vp, _vp]
        L.ddmp_assemble_sizes.argtypes = [_vp, _vp, _vp]
        L.ddmp_assemble_copy.argtypes = [_vp, _vp, _vp, _vp, _vp]
        L.ddmp_assemble_free.argtypes = [_vp]
        L.ddmp_partition.argtypes = [_i64, _vp, _vp, _i64, _i64, _vp]
        L.ddmp_add_overlap.restype = _vp
        L.ddmp_add_overlap.argtypes = [_i64, _vp, _vp, _vp, _i64]
        L.ddmp_overlap_sizes.argtypes = [_vp, _vp, _vp]
        L.ddmp_overlap_copy.argtypes = [_vp, _vp, _vp]
        L.ddmp_overlap_free.argtypes = [_vp]
        _plib = L
    return _plib


def _p(a: np.ndarray):
    return _vp(a.ctypes.data)


@dataclass(frozen=True)
class Mesh:
    coords: np.ndarray
    triangles: np.ndarray
    boundary: np.ndarray

    @property
    def n_nodes(self) -> int:
        return self.coords.shape[0]


@dataclass(frozen=True)
class PolyCoeffs:
    f_coeffs: tuple
    g_coeffs: tuple


@dataclass(frozen=True)
class LinearSystem:
    a: sp.csr_matrix
    b: np.ndarray
    interior_of_node: np.ndarray
    node_of_interior: np.ndarray
    boundary_nodes: np.ndarray
    g_values: np.ndarray

    @property
    def n(self) -> int:
        return self.b.shape[0]


@dataclass(frozen=True)
class ProblemConfig:
    target_nodes: int = 900
    perturbation: float = 0.2
    subdomain_size: int = 150
    overlap: int = 2


@dataclass
class Problem:
    mesh: Mesh
    coeffs: PolyCoeffs
    system: LinearSystem
    dec: Decomposition
    coords: np.ndarray


def boundary_flags(n_nodes: int, triangles: np.ndarray) -> np.ndarray:
    tris = np.ascontiguousarray(triangles, dtype=np.int64)
    flags = np.zeros(n_nodes, dtype=np.uint8)
    _lib().ddmp_boundary_flags(n_nodes, tris.shape[0], _p(tris), _p(flags))
    return flags.astype(bool)


def generate_blob_mesh(seed: int, target_nodes: int, perturbation: float) -> Mesh:
    """mesh.py:153-207 (coordinates in numpy exactly as the reference; rings in C++)."""
    if target_nodes < 16:
        raise ValueError(f"target_nodes must be >= 16, got {target_nodes}")
    if not 0.0 <= perturbation <= 0.3:
        raise ValueError(f"perturbation must be in [0, 0.3], got {perturbation}")
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, 4)
    b = rng.uniform(-1.0, 1.0, 4)
    amp = float(np.sum(np.hypot(a, b)))

    def radius(theta):
        if amp == 0.0 or perturbation == 0.0:
            return np.ones_like(theta)
        modes = np.arange(1, 5)[:, None] * theta[None, :]
        g = (a[:, None] * np.cos(modes) + b[:, None] * np.sin(modes)).sum(axis=0)
        return 1.0 + perturbation * g / amp

    n_rings = max(2, round(np.sqrt(target_nodes / 3.0)))
    gamma = 2.0 * (target_nodes - 1) / (n_rings * (n_rings + 1))
    ring_sizes = [max(3, round(gamma * j)) for j in range(1, n_rings + 1)]
    ring_sizes[-1] += target_nodes - (1 + sum(ring_sizes))
    ring_sizes[-1] = max(3, ring_sizes[-1])
    coords = [np.zeros((1, 2))]
    for j, nj in enumerate(ring_sizes, start=1):
        theta = 2.0 * np.pi * np.arange(nj) / nj
        rho = (j / n_rings) * radius(theta)
        coords.append(np.column_stack((rho * np.cos(theta), rho * np.sin(theta))))
    rs = np.asarray(ring_sizes, dtype=np.int64)
    L = _lib()
    t_count = L.ddmp_blob_triangles(n_rings, _p(rs), None)
    tris = np.empty((t_count, 3), dtype=np.int64)
    L.ddmp_blob_triangles(n_rings, _p(rs), _p(tris))
    all_coords = np.vstack(coords)
    mesh = Mesh(all_coords, tris, boundary_flags(len(all_coords), tris))
    for arr in (mesh.coords, mesh.triangles, mesh.boundary):
        arr.setflags(write=False)
    return mesh


def sample_coeffs(rng: np.random.Generator) -> PolyCoeffs:
    """dataset.py:79-81."""
    vals = rng.uniform(-10.0, 10.0, 9)
    return PolyCoeffs(tuple(vals[:3]), tuple(vals[3:]))


def _eval(p: PolyCoeffs, which: str, x, y):
    """fem.py:42-52."""
    if which == "source":
        r1, r2, r3 = p.f_coeffs
        return r1 * (x - 1.0) ** 2 + r2 * y**2 + r3
    r4, r5, r6, r7, r8, r9 = p.g_coeffs
    return r4 * x**2 + r5 * y**2 + r6 * x * y + r7 * x + r8 * y + r9


def assemble(mesh: Mesh, problem) -> LinearSystem:
    """fem.py:91-173."""
    if isinstance(problem, PolyCoeffs):
        f = lambda x, y: _eval(problem, "source", x, y)  # noqa: E731
        g = lambda x, y: _eval(problem, "boundary", x, y)  # noqa: E731
    else:
        f, g = problem
    interior = ~mesh.boundary
    n_int = int(interior.sum())
    if n_int == 0:
        raise ValueError("mesh has no interior nodes")
    interior_of_node = -np.ones(mesh.n_nodes, dtype=np.int64)
    interior_of_node[interior] = np.arange(n_int)
    node_of_interior = np.flatnonzero(interior)
    boundary_nodes = np.flatnonzero(mesh.boundary)
    x, y = mesh.coords[:, 0], mesh.coords[:, 1]
    f_vals = np.asarray(f(x, y), dtype=float)
    g_full = np.zeros(mesh.n_nodes)
    g_full[boundary_nodes] = np.asarray(g(x[boundary_nodes], y[boundary_nodes]), dtype=float)
    tris = np.ascontiguousarray(mesh.triangles, dtype=np.int64)
    p0, p1, p2 = mesh.coords[tris[:, 0]], mesh.coords[tris[:, 1]], mesh.coords[tris[:, 2]]
    areas = 0.5 * ((p1[:, 0] - p0[:, 0]) * (p2[:, 1] - p0[:, 1])
                   - (p2[:, 0] - p0[:, 0]) * (p1[:, 1] - p0[:, 1]))
    xt = mesh.coords[tris, 0]
    yt = mesh.coords[tris, 1]
    bt = np.stack((yt[:, 1] - yt[:, 2], yt[:, 2] - yt[:, 0], yt[:, 0] - yt[:, 1]), axis=1)
    ct = np.stack((xt[:, 2] - xt[:, 1], xt[:, 0] - xt[:, 2], xt[:, 1] - xt[:, 0]), axis=1)
    k_el = (bt[:, :, None] * bt[:, None, :] + ct[:, :, None] * ct[:, None, :]) / (
        4.0 * areas)[:, None, None]
    k_el = np.ascontiguousarray(k_el)
    load = np.bincount(tris.ravel(), weights=np.repeat(areas / 3.0, 3) * f_vals[tris].ravel(),
                       minlength=mesh.n_nodes)
    bflags = np.ascontiguousarray(mesh.boundary, dtype=np.uint8)
    L = _lib()
    h = L.ddmp_assemble(mesh.n_nodes, tris.shape[0], _p(tris), _p(k_el), _p(bflags), _p(load),
                        _p(g_full))
    try:
        ni, nnz = ctypes.c_int64(0), ctypes.c_int64(0)
        L.ddmp_assemble_sizes(h, ctypes.byref(ni), ctypes.byref(nnz))
        indptr = np.empty(ni.value + 1, dtype=np.int64)
        indices = np.empty(nnz.value, dtype=np.int32)
        data = np.empty(nnz.value, dtype=np.float64)
        b_red = np.empty(ni.value, dtype=np.float64)
        L.ddmp_assemble_copy(h, _p(indptr), _p(indices), _p(data), _p(b_red))
    finally:
        L.ddmp_assemble_free(h)
    a = sp.csr_matrix((data, indices, indptr), shape=(n_int, n_int))
    return LinearSystem(a, b_red, interior_of_node, node_of_interior, boundary_nodes,
                        g_full[boundary_nodes])


def _csr_arrays(a):
    a = sp.csr_matrix(a)
    return (np.ascontiguousarray(a.indptr, dtype=np.int64),
            np.ascontiguousarray(a.indices, dtype=np.int32))


def partition(adjacency, target_size: int, seed: int) -> np.ndarray:
    """decomp.py:92-159 (start node drawn with numpy exactly like the reference)."""
    indptr, indices = _csr_arrays(adjacency)
    n = adjacency.shape[0]
    if not 1 <= target_size <= n:
        raise ValueError(f"target_size must be in [1, {n}], got {target_size}")
    start = int(np.random.default_rng(seed).integers(n))
    owner = np.empty(n, dtype=np.int64)
    L = _lib()
    if L.ddmp_partition(n, _p(indptr), _p(indices), int(target_size), start, _p(owner)) != 0:
        raise ValueError(L.ddmp_last_error().decode())
    return owner


def add_overlap(base_owner: np.ndarray, adjacency, overlap: int) -> Decomposition:
    """decomp.py:196-216."""
    if overlap < 0:
        raise ValueError("overlap must be >= 0")
    indptr, indices = _csr_arrays(adjacency)
    owner = np.ascontiguousarray(base_owner, dtype=np.int64)
    L = _lib()
    h = L.ddmp_add_overlap(owner.shape[0], _p(indptr), _p(indices), _p(owner), int(overlap))
    try:
        k, tot = ctypes.c_int64(0), ctypes.c_int64(0)
        L.ddmp_overlap_sizes(h, ctypes.byref(k), ctypes.byref(tot))
        ptr = np.empty(k.value + 1, dtype=np.int64)
        idx = np.empty(tot.value, dtype=np.int64)
        L.ddmp_overlap_copy(h, _p(ptr), _p(idx))
    finally:
        L.ddmp_overlap_free(h)
    subs = [idx[ptr[i]:ptr[i + 1]] for i in range(k.value)]
    return finish_decomposition(subs, owner, overlap)


def build_problem(seed: int, config: ProblemConfig = ProblemConfig()) -> Problem:
    """dataset.py:84-92."""
    mesh = generate_blob_mesh(seed, config.target_nodes, config.perturbation)
    coeffs = sample_coeffs(np.random.default_rng((seed, 1)))
    system = assemble(mesh, coeffs)
    owner = partition(system.a, config.subdomain_size, seed)
    dec = add_overlap(owner, system.a, config.overlap)
    coords = mesh.coords[system.node_of_interior]
    return Problem(mesh, coeffs, system, dec, coords)
