"""Digest goldens of the REFERENCE problem builder at BASELINE configs B and C.

Runs the reference's own ``dataset.build_problem`` (mesh.py:153-207,
fem.py:91-173, decomp.py:92-216) read-only from /root/reference/pkg/src and
records SHA-256 digests of every array the hot path consumes (A's CSR arrays,
b, interior coordinates, base owner, overlapping subdomains).  The arrays
themselves are 100-1000 MB, so only the digests and a few scalars are
committed; ``tests/test_problem_builder.py`` rebuilds the same problem with the
native builder and compares digests bit for bit.

The reference partitioner is O(K*N) pure Python (SURVEY.md finding 8): about
3 minutes at B and hours at C, so C runs in the background:

    python tests/golden/make_golden_builder.py B
    nohup python tests/golden/make_golden_builder.py C &
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

HERE = os.path.dirname(os.path.abspath(__file__))
CONFIGS = {"B": 100_000, "C": 1_000_000}


def digests(a, b, coords, owner, subdomains):
    """Digest of each array in a canonical dtype/byte order (little endian)."""

    def h(x, dt):
        return hashlib.sha256(np.ascontiguousarray(x, dtype=dt).tobytes()).hexdigest()

    sizes = np.array([s.size for s in subdomains], dtype=np.int64)
    return {
        "indptr": h(a.indptr, "<i8"),
        "indices": h(a.indices, "<i8"),
        "data": h(a.data, "<f8"),
        "b": h(b, "<f8"),
        "coords": h(coords, "<f8"),
        "owner": h(owner, "<i8"),
        "sub_sizes": h(sizes, "<i8"),
        "sub_idx": h(np.concatenate(subdomains), "<i8"),
    }


def main(which):
    from ddmgnn.dataset import ProblemConfig, build_problem

    target = CONFIGS[which]
    t0 = time.perf_counter()
    p = build_problem(0, ProblemConfig(target, 0.2, 1000, 2))
    secs = time.perf_counter() - t0
    out = {
        "config": which,
        "call": f"ddmgnn.dataset.build_problem(0, ProblemConfig({target}, 0.2, 1000, 2))",
        "n": int(p.system.n),
        "nnz": int(p.system.a.nnz),
        "k": int(p.dec.n_subdomains),
        "v": int(sum(s.size for s in p.dec.subdomains)),
        "reference_seconds": round(secs, 1),
        "sha256": digests(p.system.a, p.system.b, p.coords, p.dec.base_owner, p.dec.subdomains),
    }
    path = os.path.join(HERE, f"builder_{which}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    for w in sys.argv[1:] or ["B"]:
        main(w)
