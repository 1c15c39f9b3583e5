"""GPU checks at BASELINE sizes: config B (~100k DOFs) apply
against the CPU oracle (the oracle finishes one forward in seconds there), and
size-independent properties at config C (~1M DOFs): exact positive
homogeneity z(2r) = 2 z(r) (the reference normalises r_i, hybrid.py:103-108, so
scaling by a power of two is exact end to end), bitwise repeatability, zero in
-> zero out, and the SpMV against scipy bit for bit (sequential row sums,
sparse.py:107)."""
import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def ddm():
    import paper_2402_08296_b200 as m

    return m


def _build(target, ns=1000, overlap=2):
    from paper_2402_08296_b200.problem import ProblemConfig, build_problem

    return build_problem(0, ProblemConfig(target, 0.2, ns, overlap))


@pytest.fixture(scope="module")
def config_b():
    return _build(100_000)


@pytest.fixture(scope="module")
def config_c():
    return _build(1_000_000)


@pytest.mark.parametrize("level", ["one", "two"])
def test_config_b_apply_matches_oracle(ddm, config_b, level):
    from oracle import ddm_oracle as orc

    prob = config_b
    model = ddm.init_model(10, 10, seed=1)
    p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec, model, level=level)
    om = orc.model_from_flat(10, 10, model.alpha, 1, ddm.flat_params(model))
    ref = orc.OraclePreconditioner(prob.system.a, prob.coords, prob.dec.subdomains, om, level=level)
    r = np.random.default_rng(0).standard_normal(prob.system.n)
    assert rel_l2(p(r), ref(r)) < TOL


def test_config_c_properties(ddm, config_c):
    import torch

    prob = config_c
    p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec, ddm.init_model(10, 10, seed=1))
    r = torch.tensor(np.random.default_rng(0).standard_normal(prob.system.n), device="cuda")
    z1 = p(r)
    z2 = p(r)
    assert torch.equal(z1, z2)                       # deterministic
    assert torch.equal(p(2.0 * r), 2.0 * z1)         # exact positive homogeneity
    assert torch.count_nonzero(p(torch.zeros_like(r))) == 0
    assert bool(torch.isfinite(z1).all())


def test_config_c_spmv_bitwise(ddm, config_c):
    import torch

    prob = config_c
    a = prob.system.a
    p = ddm.build_ddm_gnn(a, prob.coords, prob.dec, ddm.init_model(2, 10, seed=1), level="one")
    x = np.random.default_rng(3).standard_normal(a.shape[0])
    xd = torch.tensor(x, device="cuda")
    yd = torch.empty_like(xd)
    st = torch.cuda.current_stream().cuda_stream or 1
    p.context.spmv_device(xd.data_ptr(), yd.data_ptr(), st)
    torch.cuda.synchronize()
    assert np.array_equal(yd.cpu().numpy(), a @ x)


@pytest.mark.parametrize("ns,cs", [(2000, 2), (5000, 4), (10000, 8)])
def test_config_e_cluster_matches_flat(ddm, monkeypatch, ns, cs):
    """Config E subdomain sizes beyond one CTA's shared memory: the 2/4/8-CTA
    cluster path against the flat path (same per-node arithmetic; only the
    restriction norm's summation order differs) and its own repeatability."""
    import torch

    prob = _build(50 * ns, ns=ns, overlap=2)
    model = ddm.init_model(10, 10, seed=1)
    r = torch.tensor(np.random.default_rng(0).standard_normal(prob.system.n), device="cuda")
    out = {}
    for path in ("1", "0"):
        monkeypatch.setenv("DDMGNN_CLUSTER", path)
        p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec, model)
        info = p.info()
        assert info["n_big"] == info["K"]
        if path == "1":
            assert info["n_cluster"] == info["K"] and info["cluster_launches"] >= 1
            assert info["k_max"] > (cs // 2) * 1400  # sized to need a cluster of cs CTAs
        else:
            assert info["n_cluster"] == 0
        out[path] = p(r)
        if path == "1":
            assert torch.equal(out[path], p(r))
    z1, z0 = out["1"].cpu().numpy(), out["0"].cpu().numpy()
    assert rel_l2(z1, z0) < 1e-6


def test_two_ctas_per_sm_matches_oracle(ddm, monkeypatch):
    """Subdomains small enough for two CTAs per SM (448 threads, several slice
    rounds per warp) against the oracle and against one CTA per SM."""
    from oracle import ddm_oracle as orc

    prob = _build(30_000, ns=500, overlap=1)
    model = ddm.init_model(10, 10, seed=1)
    r = np.random.default_rng(0).standard_normal(prob.system.n)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("DDMGNN_TWO_CTA", mode)
        p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec, model)
        assert 448 < p.info()["k_max"] <= 900 and p.info()["n_big"] == 0
        out[mode] = p(r)
    om = orc.model_from_flat(10, 10, model.alpha, 2, ddm.flat_params(model))
    ref = orc.OraclePreconditioner(prob.system.a, prob.coords, prob.dec.subdomains, om, "two")(r)
    assert rel_l2(out["1"], ref) < TOL
    assert rel_l2(out["1"], out["0"]) < 1e-6
