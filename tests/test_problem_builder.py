"""The native problem builder reproduces the reference's problem setup bit for
bit (mesh.py:153-207, fem.py:91-173, decomp.py:92-216, dataset.py:84-92),
checked against the golden fixtures that the reference itself produced."""
import numpy as np
import pytest

from conftest import load_golden


def _check(prob, g, prefix=""):
    a = prob.system.a
    assert np.array_equal(a.indptr, g[f"{prefix}indptr"])
    assert np.array_equal(a.indices, g[f"{prefix}indices"])
    assert np.array_equal(a.data, g[f"{prefix}data"])
    assert np.array_equal(prob.system.b, g[f"{prefix}b"])
    assert np.array_equal(prob.coords, g[f"{prefix}coords"])
    assert np.array_equal(prob.dec.base_owner, g[f"{prefix}owner"])
    ptr, idx = g[f"{prefix}sub_ptr"], g[f"{prefix}sub_idx"]
    assert len(prob.dec.subdomains) == len(ptr) - 1
    for i, s in enumerate(prob.dec.subdomains):
        assert np.array_equal(s, idx[ptr[i]:ptr[i + 1]])


def test_small_problem_bitwise():
    from paper_2402_08296_b200.problem import ProblemConfig, build_problem

    g = load_golden("small.npz")
    _check(build_problem(21, ProblemConfig(500, 0.15, 100, 2)), g)


def test_config_a_bitwise():
    from paper_2402_08296_b200.problem import ProblemConfig, build_problem

    g = load_golden("A.npz")
    _check(build_problem(0, ProblemConfig(5000, 0.2, 1000, 2)), g)


@pytest.mark.parametrize("j", range(5))
def test_heldout_bitwise(j):
    from paper_2402_08296_b200.problem import ProblemConfig, build_problem

    g = load_golden("heldout.npz")
    _check(build_problem(500 + j, ProblemConfig(600, 0.2, 110, 2)), g, f"p{j}_")


def test_partition_errors():
    import scipy.sparse as sp

    from paper_2402_08296_b200.problem import partition

    a = sp.identity(4, format="csr")
    with pytest.raises(ValueError, match="not connected"):
        partition(a, 2, 0)
    with pytest.raises(ValueError, match="target_size"):
        partition(a, 0, 0)
