"""The CTA path's dataflow layer schedule (gnn_impl.cuh cta_layer_df) against the
barrier schedule it replaced (DDMGNN_DATAFLOW=0, read at every enqueue).  The
schedule only reorders whole slice items; every node's arithmetic is the same, so
the two must agree BIT FOR BIT — and any missed dependency (a B item reading a Q
row before its phase A wrote it, or an A item overwriting Q rows still being read)
would show up as a mismatch or as run-to-run differences.  compute-sanitizer is not
available on the GPU pool, so this repetition test is the race check; parity with
the oracle at B and C is covered in test_gpu_fullsize.py / test_gpu_north_star.py."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _problem(target, ns=1000, overlap=2):
    from paper_2402_08296_b200.problem import ProblemConfig, build_problem

    return build_problem(0, ProblemConfig(target, 0.2, ns, overlap))


def _applies(p, r, n, dataflow):
    old = os.environ.get("DDMGNN_DATAFLOW")
    os.environ["DDMGNN_DATAFLOW"] = "1" if dataflow else "0"
    try:
        return [p(r).clone() for _ in range(n)]
    finally:
        if old is None:
            del os.environ["DDMGNN_DATAFLOW"]
        else:
            os.environ["DDMGNN_DATAFLOW"] = old


@pytest.mark.parametrize("target,ns,level", [(100_000, 1000, "two"), (100_000, 500, "one"),
                                             (1_000_000, 1000, "two"),
                                             # cluster path (keeps cluster barriers: the
                                             # switch must not change it)
                                             (200_000, 2000, "two"), (250_000, 5000, "one")])
def test_dataflow_schedule_bitwise_equals_barriers(target, ns, level):
    import torch

    import paper_2402_08296_b200 as ddm

    prob = _problem(target, ns)
    p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec, ddm.init_model(10, 10, seed=1),
                          level=level)
    r = torch.tensor(np.random.default_rng(3).standard_normal(prob.system.n), device="cuda")
    ref = _applies(p, r, 1, dataflow=False)[0]
    outs = _applies(p, r, 25, dataflow=True)
    for z in outs:
        assert torch.equal(z, ref)


def test_dataflow_multi_chunk_model():
    """k_bar = 30: three launches of 10 layers each (the flags restart per launch)."""
    import torch

    import paper_2402_08296_b200 as ddm

    prob = _problem(100_000)
    p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec, ddm.init_model(30, 10, seed=2))
    r = torch.tensor(np.random.default_rng(4).standard_normal(prob.system.n), device="cuda")
    ref = _applies(p, r, 1, dataflow=False)[0]
    for z in _applies(p, r, 5, dataflow=True):
        assert torch.equal(z, ref)
