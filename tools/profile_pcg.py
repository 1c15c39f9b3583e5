"""A short PCG-DDM-GNN solve at a BASELINE config (ncu target for the per-iteration
kernels: spmv_kernel, update_kernel, coarse_gemv_kernel, prolong_kernel,
pupdate_kernel, gnn_kernel)."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2402_08296_b200 as ddm  # noqa: E402
import workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--target-nodes", type=int, default=1_000_000)
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--flexible", action="store_true")
args = ap.parse_args()
w = workload.load(args.target_nodes, 1000, 2, build_in_child=False)
dec = ddm.finish_decomposition(w.subdomains, w.owner, w.overlap)
p = ddm.build_ddm_gnn(w.a, w.coords, dec,
                      ddm.load_model(os.path.join(ROOT, "tests", "golden", "desk_k10_d10.dss")))
u, rep = ddm.pcg(w.a, w.b, p, 1e-6, args.iters, flexible=args.flexible)
print(rep.iterations, rep.residual_history[-1])
