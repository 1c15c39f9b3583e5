"""The paper's method comparison on the GPU (the reference CLI's METHODS,
cli.py:28,60-75): CG, DDM-LU one/two-level (exact local solves) and DDM-GNN
(pinned desk weights) — iterations and device time to 1e-6 on a BASELINE config.

    TARGET_NODES=1000000 python tools/compare_methods.py
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2402_08296_b200 as ddm  # noqa: E402
from paper_2402_08296_b200.problem import ProblemConfig, build_problem  # noqa: E402

target = int(os.environ.get("TARGET_NODES", "100000"))
prob = build_problem(0, ProblemConfig(target, 0.2, 1000, 2))
a, b = prob.system.a, prob.system.b
desk = ddm.load_model(os.path.join(ROOT, "tests", "golden", "desk_k10_d10.dss"))
methods = {
    "cg": lambda: None,
    "ic0": lambda: ddm.ic0(a),
    "ddm-lu-1": lambda: ddm.build_asm(a, prob.dec, "one"),
    "ddm-lu-2": lambda: ddm.build_asm(a, prob.dec, "two"),
    "ddm-gnn": lambda: ddm.build_ddm_gnn(a, prob.coords, prob.dec, desk),
}
for name, make in methods.items():
    t0 = time.perf_counter()
    p = make()
    t_setup = time.perf_counter() - t0
    ddm.pcg(a, b, p, 1e-6, 3000) if p is not None else ddm.cg(a, b, 1e-6, 3000)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    u, rep = ddm.pcg(a, b, p, 1e-6, 3000) if p is not None else ddm.cg(a, b, 1e-6, 3000)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    print(json.dumps({"method": name, "N": prob.system.n, "K": prob.dec.n_subdomains,
                      "iterations": rep.iterations, "converged": rep.converged,
                      "final_relres": rep.final_relres, "solve_s": t, "setup_s": t_setup,
                      "ms_per_iteration": 1e3 * t / max(1, rep.iterations)}), flush=True)
    del p
    torch.cuda.empty_cache()
