"""GPU trainer (paper_2402_08296_b200/train.py) against the reference's own
training (dss.py:392-469) on a dataset it harvested (tests/golden/make_golden_train.py):
same losses per epoch and the same parameters after 3 epochs (fp64; the summation
order of the gradients differs, so agreement is to rounding)."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _unpack(g, prefix):
    from paper_2402_08296_b200.train import LocalProblem

    out, e0, n0, z0, p0 = [], 0, 0, 0, 0
    for k, ne, nnz in zip(g[f"{prefix}_counts"], g[f"{prefix}_ecounts"], g[f"{prefix}_nnz"]):
        ip = g[f"{prefix}_indptr"][p0:p0 + k + 1]
        a = sp.csr_matrix((g[f"{prefix}_data"][z0:z0 + nnz], g[f"{prefix}_indices"][z0:z0 + nnz],
                           ip), shape=(k, k))
        out.append(LocalProblem(g[f"{prefix}_edges"][e0:e0 + ne], g[f"{prefix}_vec"][e0:e0 + ne],
                                g[f"{prefix}_len"][e0:e0 + ne], a, g[f"{prefix}_c"][n0:n0 + k]))
        e0, n0, z0, p0 = e0 + ne, n0 + k, z0 + nnz, p0 + k + 1
    return out


def test_trainer_matches_reference_three_epochs():
    import paper_2402_08296_b200 as ddm
    from paper_2402_08296_b200.train import Trainer

    g = load_golden("train.npz")
    model = ddm.init_model(3, 4, alpha=1e-3, seed=1)
    assert np.array_equal(ddm.flat_params(model), g["flat0"])
    tr, va = _unpack(g, "tr"), _unpack(g, "va")
    trained, log = Trainer(model).fit(tr, va, epochs=3, batch_size=20, seed=0)
    np.testing.assert_allclose(np.array(log)[:, 1:3], g["log"][:, 1:3], rtol=1e-9)
    np.testing.assert_allclose(ddm.flat_params(trained), g["flat3"], rtol=1e-7, atol=1e-10)
