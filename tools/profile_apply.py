"""Build a BASELINE config on the GPU box and run a few preconditioner applies
(target for ncu: `-k regex:gnn_kernel`)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08296_b200 as ddm  # noqa: E402
from paper_2402_08296_b200.problem import ProblemConfig, build_problem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--target-nodes", type=int, default=1_000_000)
ap.add_argument("--subdomain-size", type=int, default=1000)
ap.add_argument("--overlap", type=int, default=2)
ap.add_argument("--applies", type=int, default=3)
ap.add_argument("--kbar", type=int, default=10)
ap.add_argument("--level", default="two")
args = ap.parse_args()
prob = build_problem(0, ProblemConfig(args.target_nodes, 0.2, args.subdomain_size, args.overlap))
p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec, ddm.init_model(args.kbar, 10, seed=1),
                      level=args.level)
print(p.info())
r = torch.tensor(np.random.default_rng(0).standard_normal(prob.system.n), device="cuda")
for _ in range(args.applies):
    z = p(r)
x = torch.ones_like(r)
y = torch.empty_like(r)
st = torch.cuda.Stream()
for _ in range(args.applies):
    p.context.spmv_device(x.data_ptr(), y.data_ptr(), st.cuda_stream)
torch.cuda.synchronize()
print("ok", float(z.norm()))
