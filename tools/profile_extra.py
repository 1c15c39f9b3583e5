"""Profiling target for the comparator kernels at config C: DDM-LU apply
(asm_local_kernel + coarse GEMV + gluing) and IC(0) apply (sync-free triangular
solves).  Run under ncu (tools/profile_round.sh style)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08296_b200 as ddm  # noqa: E402
from paper_2402_08296_b200 import _lib  # noqa: E402
from paper_2402_08296_b200.problem import ProblemConfig, build_problem  # noqa: E402

prob = build_problem(0, ProblemConfig(int(os.environ.get("TARGET_NODES", "1000000")), 0.2, 1000, 2))
r = torch.tensor(np.random.default_rng(0).standard_normal(prob.system.n), device="cuda")
p = ddm.build_asm(prob.system.a, prob.dec, "two")
for _ in range(2):
    p(r)
del p
torch.cuda.empty_cache()
m = ddm.ic0(prob.system.a)
z = torch.empty_like(r)
for _ in range(2):
    m.context.apply_device(r.data_ptr(), z.data_ptr(), _lib.IC0, 0, True)
torch.cuda.synchronize()
print("ok")
