import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} missing")
    return dict(np.load(path))


def problem_from(g, prefix=""):
    """(A csr, b, coords, subdomain list) from a golden fixture."""
    import scipy.sparse as sp

    n = g[f"{prefix}b"].shape[0]
    a = sp.csr_matrix((g[f"{prefix}data"], g[f"{prefix}indices"], g[f"{prefix}indptr"]), shape=(n, n))
    ptr, idx = g[f"{prefix}sub_ptr"], g[f"{prefix}sub_idx"]
    subs = [idx[ptr[i]:ptr[i + 1]] for i in range(len(ptr) - 1)]
    return a, g[f"{prefix}b"], g[f"{prefix}coords"], subs


def rel_l2(x, y):
    return float(np.linalg.norm(np.asarray(x) - np.asarray(y)) / max(np.linalg.norm(y), 1e-300))
