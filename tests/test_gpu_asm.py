"""DDM-LU comparator on the GPU (the reference's build_asm / apply_asm,
asm.py:58-113; cli.py "ddm-lu-1"/"ddm-lu-2") against fixtures produced by the
reference itself (tests/golden/make_golden_asm.py): fp64 apply within 1e-10
(dense inverses vs SuperLU differ only in rounding) and PCG iteration counts
within +-1."""
import numpy as np
import pytest

from conftest import load_golden, problem_from, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ddm():
    import paper_2402_08296_b200 as m

    return m


def _problem(ddm):
    g = load_golden("A.npz")
    a, b, _coords, subs = problem_from(g)
    dec = ddm.finish_decomposition(subs, g["owner"], int(g["overlap"]))
    return g, a, b, dec


@pytest.mark.parametrize("level", ["one", "two"])
def test_asm_apply_and_pcg_match_reference(ddm, level):
    gold = load_golden("asm.npz")
    g, a, b, dec = _problem(ddm)
    p = ddm.build_asm(a, dec, level)
    z = p(g["r"])
    assert rel_l2(z, gold[f"z_{level}"]) < 1e-10
    _u, rep = ddm.pcg(a, b, p, 1e-6, 500)
    ref = gold[f"hist_{level}"]
    assert rep.converged and abs(rep.iterations - (len(ref) - 1)) <= 1
    np.testing.assert_allclose(rep.residual_history[:5], ref[:5], rtol=1e-8)


def test_asm_torch_path_and_repeat(ddm):
    import torch

    g, a, _b, dec = _problem(ddm)
    p = ddm.build_asm(a, dec, "two")
    r = torch.tensor(g["r"], device="cuda")
    z = p(r)
    assert z.is_cuda and np.array_equal(z.cpu().numpy(), p(g["r"]))


def test_asm_rejects_bad_level(ddm):
    g, a, _b, dec = _problem(ddm)
    with pytest.raises(ValueError):
        ddm.build_asm(a, dec, "three")
