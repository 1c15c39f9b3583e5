"""Quick device timing of apply / GNN-only / SpMV on a golden fixture (dev aid)."""
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08296_b200 as ddm  # noqa: E402

g = dict(np.load(sys.argv[1] if len(sys.argv) > 1 else "tests/golden/A.npz"))
n = g["b"].shape[0]
a = sp.csr_matrix((g["data"], g["indices"], g["indptr"]), shape=(n, n))
ptr, idx = g["sub_ptr"], g["sub_idx"]
subs = [idx[ptr[i]:ptr[i + 1]] for i in range(len(ptr) - 1)]
dec = ddm.finish_decomposition(subs, g["owner"], int(g["overlap"]))
model = ddm.init_model(10, 10, seed=1)
p = ddm.build_ddm_gnn(a, g["coords"], dec, model)
ctx = p.context
r = torch.tensor(g["r"] if "r" in g else np.random.default_rng(0).standard_normal(n), device="cuda")
if r.dim() > 1:
    r = r[0].contiguous()
z = torch.empty_like(r)
s = torch.cuda.current_stream().cuda_stream
out = {"info": p.info()}
for name, fn in [("apply2", lambda: ctx.apply_device(r.data_ptr(), z.data_ptr(), 2, s, False)),
                 ("gnn", lambda: ctx.launch_gnn_only(r.data_ptr(), s)),
                 ("spmv", lambda: ctx.spmv_device(r.data_ptr(), z.data_ptr(), s))]:
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        fn()
    e1.record()
    torch.cuda.synchronize()
    out[name + "_ms"] = e0.elapsed_time(e1) / 50
t0 = time.perf_counter()
u, rep = ddm.cg(a, g["b"], 1e-6, 5000)
out["cg_iters"], out["cg_s"] = rep.iterations, time.perf_counter() - t0
print(json.dumps(out))
