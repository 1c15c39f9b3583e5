"""IC(0) comparator on the GPU against the reference's own tests
(pkg/tests/test_sparse.py:119-151) and fixtures it produced
(tests/golden/make_golden_asm.py ic0): factor pattern/values, apply, and PCG
iteration counts within +-1."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import load_golden, problem_from, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ddm():
    import paper_2402_08296_b200 as m

    return m


def test_ic0_diagonal_exact(ddm):
    a = sp.csr_matrix(np.diag([4.0, 9.0, 16.0]))
    _, rep = ddm.pcg(a, np.ones(3), ddm.ic0(a), 1e-12, 10)
    assert rep.iterations == 1


def test_ic0_tridiagonal_equals_cholesky(ddm):
    n = 60
    a = sp.diags([[-1.0] * (n - 1), [2.0] * n, [-1.0] * (n - 1)], [-1, 0, 1]).tocsr()
    m = ddm.ic0(a)
    assert np.allclose(m.l.toarray(), np.linalg.cholesky(a.toarray()), atol=1e-13)
    _, rep = ddm.pcg(a, np.ones(n), m, 1e-12, 10)
    assert rep.iterations == 1


def test_ic0_breakdown_raises(ddm):
    a = sp.csr_matrix(np.array([[1.0, 2.0], [2.0, 1.0]]))
    with pytest.raises(RuntimeError, match="IC\\(0\\) breakdown"):
        ddm.ic0(a)


def test_ic0_matches_reference_config_a(ddm):
    gold = load_golden("ic0.npz")
    g = load_golden("A.npz")
    a, b, _coords, _subs = problem_from(g)
    m = ddm.ic0(a)
    l = m.l
    assert np.array_equal(l.indptr, gold["l_indptr"]) and np.array_equal(l.indices, gold["l_indices"])
    np.testing.assert_allclose(l.data, gold["l_data"], rtol=1e-12, atol=1e-14)
    assert rel_l2(m(g["r"]), gold["z"]) < 1e-12
    _u, rep = ddm.pcg(a, b, m, 1e-6, 5000)
    assert rep.converged and abs(rep.iterations - (len(gold["hist"]) - 1)) <= 1
