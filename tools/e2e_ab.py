"""End-to-end apply throughput through ddmgnn_apply_host at config C (pinned host
r in, pinned host z out, host clock over 200 steps) — A/B of the staged input copy
(DDMGNN_STAGED_INPUT=0 disables); prints one JSON line with a z checksum."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2402_08296_b200 as ddm  # noqa: E402
import workload  # noqa: E402

w = workload.load(1_000_000, 1000, 2, build_in_child=False)
dec = ddm.finish_decomposition(w.subdomains, w.owner, w.overlap)
p = ddm.build_ddm_gnn(w.a, w.coords, dec, ddm.init_model(10, 10, seed=1))
ctx = p.context
r_pin = torch.from_numpy(np.random.default_rng(0).standard_normal(w.n)).pin_memory()
z_pin = torch.empty(w.n, dtype=torch.float64).pin_memory()
rh, zh = r_pin.numpy(), z_pin.numpy()
for _ in range(20):
    ctx.apply_host(rh, 2, out=zh)
z0 = zh.copy()
res = []
for rep in range(3):
    t0 = time.perf_counter()
    for _ in range(200):
        ctx.apply_host(rh, 2, out=zh)
    res.append((time.perf_counter() - t0) / 200)
zd = torch.empty(w.n, dtype=torch.float64, device="cuda")
ctx.apply_device(torch.tensor(rh, device="cuda").data_ptr(), zd.data_ptr(), 2,
                 torch.cuda.current_stream().cuda_stream or 1, True)
torch.cuda.synchronize()
print(json.dumps({"staged": os.environ.get("DDMGNN_STAGED_INPUT", "1"),
                  "e2e_ms": [1e3 * x for x in res], "e2e_per_s": 1.0 / min(res),
                  "repeat_bitwise": bool(np.array_equal(z0, zh)),
                  "equals_device_apply": bool(np.array_equal(zh, zd.cpu().numpy())),
                  "z_sum": float(zh.sum())}))
