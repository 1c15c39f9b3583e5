"""Breakdown of the end-to-end apply at config C: pinned H2D / D2H copy times
(CUDA events), device apply, and ddmgnn_apply_host wall time."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08296_b200 as ddm  # noqa: E402
from paper_2402_08296_b200.problem import ProblemConfig, build_problem  # noqa: E402

prob = build_problem(0, ProblemConfig(1_000_000, 0.2, 1000, 2))
p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec, ddm.init_model(10, 10, seed=1))
ctx, n = p.context, prob.system.n
r_pin = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).pin_memory()
z_pin = torch.empty(n, dtype=torch.float64).pin_memory()
rd = r_pin.to("cuda")
zd = torch.empty_like(rd)
st = torch.cuda.current_stream()
out = {}


def ev_time(fn, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out["h2d_ms"] = ev_time(lambda: rd.copy_(r_pin, non_blocking=True))
out["d2h_ms"] = ev_time(lambda: z_pin.copy_(zd, non_blocking=True))
out["h2d_GBps"] = 8 * n / out["h2d_ms"] / 1e6
out["d2h_GBps"] = 8 * n / out["d2h_ms"] / 1e6
out["apply_device_ms"] = ev_time(lambda: ctx.apply_device(rd.data_ptr(), zd.data_ptr(), 2,
                                                          st.cuda_stream, False))
rh, zh = r_pin.numpy(), z_pin.numpy()
for _ in range(3):
    ctx.apply_host(rh, 2, out=zh)
t0 = time.perf_counter()
for _ in range(20):
    ctx.apply_host(rh, 2, out=zh)
out["apply_host_wall_ms"] = (time.perf_counter() - t0) / 20 * 1e3
t0 = time.perf_counter()
for _ in range(20):
    ctx.apply_device(rd.data_ptr(), zd.data_ptr(), 2, st.cuda_stream, True)
out["apply_device_sync_wall_ms"] = (time.perf_counter() - t0) / 20 * 1e3
print(json.dumps(out))


def wall(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


cs = ctx  # noqa
ctx_stream = torch.cuda.Stream()


def manual():
    with torch.cuda.stream(ctx_stream):
        rd.copy_(r_pin, non_blocking=True)
        ctx.apply_device(rd.data_ptr(), zd.data_ptr(), 2, ctx_stream.cuda_stream, False)
        z_pin.copy_(zd, non_blocking=True)
    ctx_stream.synchronize()


rp, zp = np.array(rh), np.empty_like(zh)
res = {"apply_host_pinned": wall(lambda: ctx.apply_host(rh, 2, out=zh)),
       "apply_host_pageable": wall(lambda: ctx.apply_host(rp, 2, out=zp)),
       "manual_torch_copies": wall(manual),
       "apply_device_sync": wall(lambda: ctx.apply_device(rd.data_ptr(), zd.data_ptr(), 2,
                                                          ctx_stream.cuda_stream, True))}
print(json.dumps(res))
