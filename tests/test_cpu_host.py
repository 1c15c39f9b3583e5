"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
the product fails loudly without a GPU (no CPU fallback), and the host-side
mirrors of the reference's data formats behave like the reference
(pkg/tests/test_hybrid.py:47-52, test_dss.py:26-40,262-290, test_decomp.py:85-130)."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ddmgnn_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ddmgnn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2402_08296_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = _declared()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
    assert {s[0] for s in _lib.SIGNATURES} == set(names)


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2402_08296_b200 as ddm
    import scipy.sparse as sp

    from paper_2402_08296_b200 import _lib

    with pytest.raises(RuntimeError):
        _lib.Context(0)
    with pytest.raises(RuntimeError):
        ddm.cg(sp.identity(4, format="csr"), np.ones(4), 1e-8, 10)


def test_plan_batches_matches_reference():
    from paper_2402_08296_b200 import plan_batches

    plan = plan_batches([1000] * 234, 59000)
    assert len(plan) == 4
    assert sorted(sum(plan, [])) == list(range(234))
    assert plan_batches([10, 500, 10], 100) == [[0], [1], [2]]
    with pytest.raises(ValueError):
        plan_batches([1], 0)


def test_param_counts_and_init_draws():
    import paper_2402_08296_b200 as ddm
    from conftest import load_golden

    table = {(5, 5): 1755, (5, 10): 6255, (10, 10): 12510, (10, 20): 47010, (30, 10): 37530}
    for (kb, d), expected in table.items():
        assert ddm.param_count(kb, d) == expected == ddm.init_model(kb, d).n_params()
    g = load_golden("small.npz")
    assert np.array_equal(ddm.flat_params(ddm.init_model(3, 4, seed=0)), g["m340_flat"])
    assert np.array_equal(ddm.flat_params(ddm.init_model(2, 3, seed=4)), g["m234_flat"])


def test_save_load_bit_exact(tmp_path):
    import paper_2402_08296_b200 as ddm

    m = ddm.init_model(3, 4, seed=5)
    p1, p2 = tmp_path / "m1.dss", tmp_path / "m2.dss"
    ddm.save_model(m, p1)
    ddm.save_model(ddm.load_model(p1), p2)
    assert p1.read_bytes() == p2.read_bytes()
    p2.write_bytes(p1.read_bytes()[:-8])
    with pytest.raises(ValueError, match="weight block size mismatch"):
        ddm.load_model(p2)
    p2.write_bytes(b'{"format": "dss-v0"}\n')
    with pytest.raises(ValueError, match="unsupported model format"):
        ddm.load_model(p2)


def test_desk_weights_readable_by_both():
    import paper_2402_08296_b200 as ddm
    from conftest import GOLDEN
    from oracle import ddm_oracle as orc

    path = os.path.join(GOLDEN, "desk_k10_d10.dss")
    if not os.path.exists(path):
        pytest.skip("desk weights missing")
    m = ddm.load_model(path)
    o = orc.load_model(path)
    assert (m.k_bar, m.d) == (o.k_bar, o.d) == (10, 10)


def test_partition_of_unity_and_nicolaides_hand_case():
    import paper_2402_08296_b200 as ddm

    subs = [np.array([0, 1, 2, 3]), np.array([2, 3, 4, 5])]
    dec = ddm.finish_decomposition(subs, np.array([0, 0, 0, 1, 1, 1]), 1)
    r0 = dec.r0.toarray()
    assert np.array_equal(r0, [[1, 1, .5, .5, 0, 0], [0, 0, .5, .5, 1, 1]])
    x = np.random.default_rng(0).standard_normal(6)
    acc = sum(ddm.extend(dec, i, dec.pou_weights[i] * ddm.restrict(dec, i, x)) for i in range(2))
    assert np.abs(acc - x).max() <= 1e-15 * np.abs(x).max()
    with pytest.raises(ValueError, match="do not cover"):
        ddm.finish_decomposition([np.array([0, 1])], np.zeros(3, dtype=np.int64), 0)
    j = ddm.Decomposition.from_json(dec.to_json())
    assert all(np.array_equal(a, b) for a, b in zip(j.subdomains, dec.subdomains))


def test_validate_csr():
    import scipy.sparse as sp

    from paper_2402_08296_b200 import validate_csr

    a = sp.random(20, 20, density=0.2, format="csr", random_state=0)
    a.sort_indices()
    validate_csr(a)
    bad = a.copy()
    bad.indices[bad.indptr[3]:bad.indptr[4]] = bad.indices[bad.indptr[3]:bad.indptr[4]][::-1]
    if bad.indptr[4] - bad.indptr[3] > 1:
        with pytest.raises(ValueError, match="row 3"):
            validate_csr(bad)


def test_gnn_launch_count():
    """Launches per GNN forward as bench.py reports them (gpu_launches): per chunk
    the CTA kernel (if any subdomain fits one CTA), one per cluster size in use,
    and for flat-path subdomains a restriction prologue (first chunk) + 2 per layer."""
    from paper_2402_08296_b200._lib import Context

    ctx = Context.__new__(Context)

    def count(**kw):
        base = dict(K=997, n_big=0, n_cluster=0, cluster_launches=0, k_bar=10, lmax=10,
                    n_chunks=1)
        base.update(kw)
        ctx.info = lambda: base
        return ctx.gnn_launches()

    assert count() == 1
    assert count(n_big=7, n_cluster=7, cluster_launches=1) == 2          # config C
    assert count(K=50, n_big=50, n_cluster=50, cluster_launches=2) == 2  # clusters only
    assert count(n_big=3, n_cluster=0) == 1 + 1 + 20                     # flat path
    assert count(k_bar=30, n_chunks=3, n_big=2, n_cluster=1, cluster_launches=1) == 3 * 2 + 1 + 60


def test_validate_csr_reports_first_bad_row():
    """The reference scans rows in order (sparse.py:64-67): an out-of-range column
    in row 4 is reported as row 4, before a later unsorted row."""
    import scipy.sparse as sp

    from paper_2402_08296_b200 import validate_csr

    a = sp.csr_matrix(np.eye(8))
    bad = sp.csr_matrix((a.data.copy(), a.indices.copy(), a.indptr.copy()), shape=(8, 8))
    bad.indices[4] = 9
    with pytest.raises(ValueError, match="row 4:"):
        validate_csr(bad)
    m = sp.csr_matrix(np.ones((6, 6)))
    m.indices[m.indptr[5]:m.indptr[6]] = m.indices[m.indptr[5]:m.indptr[6]][::-1].copy()
    m.indices[m.indptr[2] + 1] = -1
    with pytest.raises(ValueError, match="row 2:"):
        validate_csr(m)
