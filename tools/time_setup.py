"""Setup-cost probe at a given mesh size: native problem build, preconditioner
build (layout + coarse matrix + inverse), and one timed apply."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08296_b200 as ddm  # noqa: E402
from paper_2402_08296_b200.asm import coarse_inverse, coarse_matrix  # noqa: E402
from paper_2402_08296_b200.problem import ProblemConfig, build_problem  # noqa: E402

target = int(os.environ.get("TARGET_NODES", "10000000"))
t0 = time.perf_counter()
prob = build_problem(0, ProblemConfig(target, 0.2, 1000, 2))
t_prob = time.perf_counter() - t0
t0 = time.perf_counter()
cm = coarse_matrix(prob.system.a, prob.dec)
t_cm = time.perf_counter() - t0
t0 = time.perf_counter()
inv = coarse_inverse(cm)
t_inv = time.perf_counter() - t0
t0 = time.perf_counter()
p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec, ddm.init_model(10, 10, seed=1))
t_build = time.perf_counter() - t0
r = torch.tensor(np.random.default_rng(0).standard_normal(prob.system.n), device="cuda")
for _ in range(3):
    z = p(r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    z = p(r)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"target": target, "N": prob.system.n, "K": prob.dec.n_subdomains,
                  "info": p.info(), "problem_build_s": t_prob, "coarse_matrix_s": t_cm,
                  "coarse_inverse_s": t_inv, "preconditioner_build_s": t_build,
                  "apply_ms": e0.elapsed_time(e1) / 5}))
