"""Host-overhead probe of the sharded path: apply_owned and one distributed PCG
iteration at world size 1 (no collectives) vs the single-context apply."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08296_b200 as ddm  # noqa: E402
from paper_2402_08296_b200.problem import ProblemConfig, build_problem  # noqa: E402
from paper_2402_08296_b200.sharded import ShardedDdmGnn  # noqa: E402

prob = build_problem(0, ProblemConfig(int(os.environ.get("TARGET_NODES", "1000000")), 0.2, 1000, 2))
model = ddm.load_model(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "tests", "golden", "desk_k10_d10.dss"))
sh = ShardedDdmGnn(prob.system.a, prob.coords, prob.dec, model)
r = sh.owned_part(np.random.default_rng(0).standard_normal(prob.system.n))
z = torch.empty_like(r)
for _ in range(3):
    sh.apply_owned(r, z)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    sh.apply_owned(r, z)
torch.cuda.synchronize()
t_apply = (time.perf_counter() - t0) / 20
t0 = time.perf_counter()
u, rep = sh.pcg(prob.system.b, 1e-6, 1000)
t_pcg = time.perf_counter() - t0
print(json.dumps({"sharded_apply_ms_world1": 1e3 * t_apply, "pcg_s": t_pcg,
                  "iterations": rep.iterations, "ms_per_iteration": 1e3 * t_pcg / rep.iterations,
                  "converged": rep.converged}))
# host issue cost of one apply_owned (no synchronisation inside the loop)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    sh.apply_owned(r, z)
t_issue = (time.perf_counter() - t0) / 50
torch.cuda.synchronize()
t_total = (time.perf_counter() - t0) / 50
print(json.dumps({"apply_host_issue_ms": 1e3 * t_issue, "apply_wall_ms": 1e3 * t_total}))
