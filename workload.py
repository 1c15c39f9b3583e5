"""Benchmark workloads shared by both arms of bench.py (and build()).

The BASELINE configurations are built once by the native problem builder
(paper_2402_08296_b200/problem.py — bit-identical to the reference's
``dataset.build_problem``, tests/test_problem_builder.py) and cached as a plain
.npz under data/problems/ (git-ignored; it travels to the GPU box with the
snapshot).  Both arms load the same file, so they time the same A, b,
coordinates and subdomains, and the reference arm's process never maps any of
this repository's native libraries: reading the cache needs numpy only.
``__graft_entry__.build()`` creates the config-C cache; when it is missing the
reference arm builds it in a child process (recorded as ``problem_source``).
"""

from __future__ import annotations

import os
import subprocess
import sys
import time
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
CACHE = os.path.join(ROOT, "data", "problems")


@dataclass
class Workload:
    a: object            # scipy CSR
    b: np.ndarray
    coords: np.ndarray
    subdomains: list
    owner: np.ndarray
    overlap: int
    target: int
    subdomain_size: int
    source: str
    seconds: float

    @property
    def n(self) -> int:
        return self.b.shape[0]

    @property
    def k(self) -> int:
        return len(self.subdomains)

    @property
    def v(self) -> int:
        return int(sum(s.size for s in self.subdomains))


def cache_path(target: int, subdomain_size: int, overlap: int) -> str:
    return os.path.join(CACHE, f"blob0_{target}_{subdomain_size}_{overlap}.npz")


def write_cache(target: int, subdomain_size: int = 1000, overlap: int = 2) -> str:
    """Build with the native builder (setup only) and store the arrays."""
    sys.path.insert(0, ROOT)
    from paper_2402_08296_b200.problem import ProblemConfig, build_problem

    prob = build_problem(0, ProblemConfig(target, 0.2, subdomain_size, overlap))
    a, subs = prob.system.a, prob.dec.subdomains
    path = cache_path(target, subdomain_size, overlap)
    os.makedirs(CACHE, exist_ok=True)
    tmp = f"{path}.{os.getpid()}.tmp.npz"  # ranks may build concurrently
    np.savez_compressed(
        tmp, indptr=a.indptr.astype(np.int32), indices=a.indices.astype(np.int32), data=a.data,
        b=prob.system.b, coords=prob.coords,
        sub_ptr=np.concatenate(([0], np.cumsum([s.size for s in subs]))).astype(np.int64),
        sub_idx=np.concatenate(subs).astype(np.int32),
        owner=prob.dec.base_owner.astype(np.int32), overlap=np.int64(overlap))
    os.replace(tmp, path)
    return path


def load(target: int, subdomain_size: int = 1000, overlap: int = 2,
         build_in_child: bool = True) -> Workload:
    """The cached workload; if absent, built (in a child process when
    ``build_in_child``, so the calling process loads no native library)."""
    import scipy.sparse as sp

    t0 = time.perf_counter()
    path = cache_path(target, subdomain_size, overlap)
    source = f"cache {os.path.relpath(path, ROOT)}"
    if not os.path.exists(path):
        if build_in_child:
            subprocess.run([sys.executable, os.path.abspath(__file__), str(target),
                            str(subdomain_size), str(overlap)], check=True)
            source = "built by the native builder in a child process, then loaded from .npz"
        else:
            write_cache(target, subdomain_size, overlap)
            source = "built by the native builder in-process"
    g = np.load(path)
    n = g["b"].shape[0]
    a = sp.csr_matrix((g["data"], g["indices"], g["indptr"]), shape=(n, n))
    ptr, idx = g["sub_ptr"], g["sub_idx"].astype(np.int64)
    subs = [idx[ptr[i]:ptr[i + 1]] for i in range(len(ptr) - 1)]
    return Workload(a, g["b"], g["coords"], subs, g["owner"].astype(np.int64),
                    int(g["overlap"]), target, subdomain_size, source,
                    time.perf_counter() - t0)


if __name__ == "__main__":
    args = [int(x) for x in sys.argv[1:]] or [1_000_000]
    print(write_cache(*args))
