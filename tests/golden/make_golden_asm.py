"""Golden fixtures for the DDM-LU comparator (the reference's build_asm / apply_asm,
asm.py:58-113, and pcg with it, cli.py:67-70), produced by running the REFERENCE
read-only from /root/reference/pkg/src on the problem of A.npz.

    python tests/golden/make_golden_asm.py   ->  tests/golden/asm.npz
"""

import os
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, "/root/reference/pkg/src")
from ddmgnn.asm import apply_asm, build_asm  # noqa: E402
from ddmgnn.decomp import Decomposition  # noqa: E402
from ddmgnn.sparse import pcg  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    g = dict(np.load(os.path.join(HERE, "A.npz")))
    n = g["b"].shape[0]
    a = sp.csr_matrix((g["data"], g["indices"], g["indptr"]), shape=(n, n))
    ptr, idx = g["sub_ptr"], g["sub_idx"]
    subs = [idx[ptr[i]:ptr[i + 1]].astype(np.int64) for i in range(len(ptr) - 1)]
    import json

    dec = Decomposition.from_json(json.dumps({"overlap": int(g["overlap"]),
                                              "owner": g["owner"].tolist(),
                                              "subdomains": [s.tolist() for s in subs]}))
    out = {}
    for level in ("one", "two"):
        p = build_asm(a, dec, level)
        out[f"z_{level}"] = apply_asm(p, g["r"])
        _u, rep = pcg(a, g["b"], p, 1e-6, 500)
        out[f"hist_{level}"] = np.asarray(rep.residual_history)
    np.savez_compressed(os.path.join(HERE, "asm.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()


def ic0_fixture():
    """ic0 factor and PCG-IC(0) history on the A.npz problem (sparse.py:184-227)."""
    from ddmgnn.sparse import ic0

    g = dict(np.load(os.path.join(HERE, "A.npz")))
    n = g["b"].shape[0]
    a = sp.csr_matrix((g["data"], g["indices"], g["indptr"]), shape=(n, n))
    m = ic0(a)
    _u, rep = pcg(a, g["b"], m, 1e-6, 5000)
    l = m.l.tocsr()
    np.savez_compressed(os.path.join(HERE, "ic0.npz"), l_indptr=l.indptr, l_indices=l.indices,
                        l_data=l.data, z=m(g["r"]), hist=np.asarray(rep.residual_history))
    print("ic0", l.nnz, rep.iterations)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "ic0":
    ic0_fixture()
