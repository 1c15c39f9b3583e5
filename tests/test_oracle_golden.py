"""Pin the CPU oracle against golden vectors produced by the reference itself.

The fixtures come from tests/golden/make_golden.py (which imports
/root/reference); the oracle restatement must reproduce them to fp64
round-off, which makes it a trustworthy checker for the CUDA path.
"""
import os

import numpy as np
import pytest

from conftest import load_golden, problem_from, rel_l2
from oracle import ddm_oracle as orc


def _model(g, tag):
    kb, d, seed = (int(x) for x in g[f"{tag}_meta"])
    return orc.model_from_flat(kb, d, float(g[f"{tag}_alpha"]), seed, g[f"{tag}_flat"])


def test_init_model_matches_reference_draws():
    g = load_golden("small.npz")
    for tag in ("m340", "m234"):
        kb, d, seed = (int(x) for x in g[f"{tag}_meta"])
        assert np.array_equal(orc.init_model_flat(kb, d, seed), g[f"{tag}_flat"])


def test_local_graphs_bitwise():
    g = load_golden("small.npz")
    a, _b, coords, subs = problem_from(g)
    counts = g["tpl_counts"]
    offs = np.concatenate(([0], np.cumsum(counts)))
    for i, s in enumerate(subs):
        t = orc.local_graph(a, s, coords)
        sl = slice(offs[i], offs[i + 1])
        assert np.array_equal(t.edges, g["tpl_edges"][sl])
        assert np.array_equal(t.edge_vec, g["tpl_edge_vec"][sl])
        assert np.array_equal(t.edge_len, g["tpl_edge_len"][sl])


def test_pou_and_coarse_bitwise():
    g = load_golden("small.npz")
    a, _b, _coords, subs = problem_from(g)
    w, r0 = orc.finish_decomposition(subs, a.shape[0])
    assert np.array_equal(np.concatenate(w), g["pou"])
    assert np.array_equal(orc.coarse_matrix(a, r0), g["coarse"])


@pytest.mark.parametrize("tag", ["m340", "m234"])
def test_apply_matches_reference(tag):
    g = load_golden("small.npz")
    a, _b, coords, subs = problem_from(g)
    model = _model(g, tag)
    p2 = orc.OraclePreconditioner(a, coords, subs, model, "two")
    p1 = orc.OraclePreconditioner(a, coords, subs, model, "one")
    for k, r in enumerate(g["r"]):
        assert rel_l2(p2(r), g[f"{tag}_z_two"][k]) < 1e-13
        assert rel_l2(p1(r), g[f"{tag}_z_loc"][k]) < 1e-13


def test_apply_config_a_matches_reference():
    g = load_golden("A.npz")
    a, _b, coords, subs = problem_from(g)
    model = orc.model_from_flat(10, 10, float(g["m1010_alpha"]), 1, g["m1010_flat"])
    assert np.array_equal(model_flat := np.concatenate([np.concatenate([np.ravel(x) for x in l[n]])
                                                         for l in model.layers
                                                         for n in ("phi_out", "phi_in", "psi", "dec")]),
                          g["m1010_flat"])
    p2 = orc.OraclePreconditioner(a, coords, subs, model, "two")
    assert rel_l2(p2(g["r"]), g["m1010_z_two"]) < 1e-13
    p1 = orc.OraclePreconditioner(a, coords, subs, model, "one")
    assert rel_l2(p1(g["r"]), g["m1010_z_loc"]) < 1e-13


def test_cg_history_matches_reference():
    g = load_golden("small.npz")
    a, b, _c, _s = problem_from(g)
    _u, it, hist, conv = orc.pcg(a, b, None, 1e-8, 500)
    assert conv and it == int(g["cg_iters"])
    assert np.allclose(hist, g["cg_hist"], rtol=1e-10, atol=0)


def test_desk_pcg_matches_reference():
    g = load_golden("A.npz")
    if "desk_pcg_hist" not in g:
        pytest.skip("desk weights not in fixture")
    a, b, coords, subs = problem_from(g)
    model = orc.load_model(__import__("os").path.join(__import__("conftest").GOLDEN, "desk_k10_d10.dss"))
    p = orc.OraclePreconditioner(a, coords, subs, model, "two")
    _u, it, hist, conv = orc.pcg(a, b, p, 1e-6, 500)
    ref = g["desk_pcg_hist"]
    assert abs(it - (len(ref) - 1)) <= 1
    assert np.allclose(hist[:20], ref[:20], rtol=1e-8)


def test_parallel_oracle_equals_serial_oracle():
    """oracle/parallel.py (the multi-process oracle used at configs B/C/D and by
    the bench's CPU legs) gives the serial oracle's z: same forward per subdomain,
    same gluing order (hybrid.py:133-135)."""
    from oracle.parallel import ParallelOracle

    g = load_golden("A.npz")
    a, _b, coords, subs = problem_from(g)
    m = orc.model_from_flat(10, 10, float(g["m1010_alpha"]), 1, g["m1010_flat"])
    ser = orc.OraclePreconditioner(a, coords, subs, m, "two")
    with ParallelOracle(a, coords, subs, m, level="two", workers=3) as par:
        assert par.workers == 3
        for r in (g["r"], 2.0 * g["r"]):
            assert rel_l2(par(r), ser(r)) < 1e-15
            assert rel_l2(par.apply(r, "one"), g["m1010_z_loc"] * (1 if r is g["r"] else 2)) < 1e-12
        desk = orc.load_model(os.path.join(os.path.dirname(__file__), "golden", "desk_k10_d10.dss"))
        par.set_model(desk)
        assert rel_l2(par(g["r"]), g["desk_z_two"]) < 1e-13


def test_oracle_flexible_cg():
    """Flexible CG (opt-in; Polak-Ribiere beta): with z = r it is CG in exact
    arithmetic (r_k+1 . r_k = 0), so it needs the reference CG's iteration count
    to +-1; its default (flexible=False) is the reference recurrence."""
    g = load_golden("small.npz")
    a, b, _c, _s = problem_from(g)
    _u, it, hist, conv = orc.pcg(a, b, None, 1e-8, 500, flexible=True)
    assert conv and abs(it - int(g["cg_iters"])) <= 1
    _u, it0, hist0, _ = orc.pcg(a, b, None, 1e-8, 500)
    assert np.allclose(hist0, g["cg_hist"], rtol=1e-10)
    assert np.allclose(hist[:10], hist0[:10], rtol=1e-9)
