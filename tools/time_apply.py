"""Quick apply timing of one library build (kernel variant experiments):
DDMGNN_B200_LIB=<path> python tools/time_apply.py  -> one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08296_b200 as ddm  # noqa: E402
from paper_2402_08296_b200 import _lib  # noqa: E402
from paper_2402_08296_b200.problem import ProblemConfig, build_problem  # noqa: E402

target = int(os.environ.get("TARGET_NODES", "1000000"))
ns = int(os.environ.get("SUBDOMAIN_SIZE", "1000"))
prob = build_problem(0, ProblemConfig(target, 0.2, ns, int(os.environ.get("OVERLAP", "2"))))
p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec, ddm.init_model(int(os.environ.get("KBAR", "10")), 10, seed=1))
ctx = p.context
dev = torch.device("cuda:0")
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
r = torch.tensor(np.random.default_rng(0).standard_normal(prob.system.n), device=dev)
z = torch.empty_like(r)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
for _ in range(3):
    ctx.apply_device(r.data_ptr(), z.data_ptr(), 2, st.cuda_stream, True)
ref = z.clone()
ts, tg = [], []
for i in range(20):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.apply_device(r.data_ptr(), z.data_ptr(), 2, st.cuda_stream, False)
    e1.record(st)
    flush.zero_()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(st)
    ctx.launch_gnn_only(r.data_ptr(), st.cuda_stream)
    g1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    tg.append(g0.elapsed_time(g1))
print(json.dumps({"lib": os.path.basename(_lib.LIB_PATH), "N_s": ns, "apply_ms": float(np.median(ts)),
                  "gnn_ms": float(np.median(tg)), "repeat_bitwise": bool(torch.equal(z, ref))}))
