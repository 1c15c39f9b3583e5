"""Device time-to-solution of PCG-DDM-GNN at a BASELINE config (desk weights):
one JSON line with iterations, seconds and ms per iteration (kernel-variant A/B:
DDMGNN_FUSED_TAIL=0/1, DDMGNN_B200_LIB=<variant>)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2402_08296_b200 as ddm  # noqa: E402
import workload  # noqa: E402

target = int(os.environ.get("TARGET_NODES", "1000000"))
w = workload.load(target, 1000, 2, build_in_child=False)
dec = ddm.finish_decomposition(w.subdomains, w.owner, w.overlap)
p = ddm.build_ddm_gnn(w.a, w.coords, dec,
                      ddm.load_model(os.path.join(ROOT, "tests", "golden", "desk_k10_d10.dss")))
ctx = p.context
dev = torch.device("cuda:0")
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
b = torch.tensor(w.b, device=dev)
u = torch.empty_like(b)
out = {"lib": os.path.basename(ddm._lib.LIB_PATH), "fused_tail": os.environ.get("DDMGNN_FUSED_TAIL", "1")}
for flex in (False, True):
    ctx.pcg(b.data_ptr(), None, 1e-6, 1000, 2, True, u.data_ptr(), st.cuda_stream, flexible=flex)
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _u, it, hist, conv = ctx.pcg(b.data_ptr(), None, 1e-6, 1000, 2, True, u.data_ptr(),
                                     st.cuda_stream, flexible=flex)
        e1.record(st)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    uh = u.cpu().numpy()
    true_rel = float(np.linalg.norm(w.b - w.a @ uh) / np.linalg.norm(w.b))
    key = "fcg" if flex else "pcg"
    out[key] = {"iterations": it, "converged": conv, "seconds": min(times),
                "ms_per_iteration": 1e3 * min(times) / it, "final_relres": hist[-1],
                "true_relres": true_rel}
print(json.dumps(out))
