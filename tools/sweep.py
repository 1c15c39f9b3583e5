"""BASELINE config E: GNN-apply microbench sweep — subdomain size x overlap x
message-passing depth on synthetic blob meshes (target >= 50 N_s nodes so K >= 50),
random-init weights, d = 10 (or --dims).  One JSON line per configuration:
applies timed with CUDA events (L2 flushed), executed FP32 TFLOP/s of the GNN
launch against the measured FP32 peak (bench.py's roofline definitions: executed flops
and SURVEY §8(d)'s F_gnn).

    python tools/sweep.py [--sizes 500,1000,2000,5000] [--overlaps 1,2,3] [--kbars 5,10,20,30]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2402_08296_b200 as ddm  # noqa: E402
from bench import fp32_peak_tflops, gnn_flops, gnn_flops_exec  # noqa: E402
from paper_2402_08296_b200.problem import ProblemConfig, build_problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="500,1000,2000,5000")
    ap.add_argument("--overlaps", default="1,2,3")
    ap.add_argument("--kbars", default="5,10,20,30")
    ap.add_argument("--dims", default="10", help="latent widths d (config E: 10, optionally 5, 20)")
    ap.add_argument("--min-nodes", type=int, default=100_000)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    peak, peak_src = fp32_peak_tflops(1965.0)
    h0 = os.environ.get("DDMGNN_H0_SKIP", "1") != "0"
    for ns in [int(x) for x in args.sizes.split(",")]:
        for ov in [int(x) for x in args.overlaps.split(",")]:
            t0 = time.perf_counter()
            prob = build_problem(0, ProblemConfig(max(args.min_nodes, 50 * ns), 0.2, ns, ov))
            t_build = time.perf_counter() - t0
            r = torch.tensor(np.random.default_rng(0).standard_normal(prob.system.n), device=dev)
            z = torch.empty_like(r)
            for kb, dd in [(int(x), int(y)) for x in args.kbars.split(",")
                           for y in args.dims.split(",")]:
                p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec,
                                      ddm.init_model(kb, dd, seed=1))
                ctx, info = p.context, p.info()
                for _ in range(2):
                    ctx.apply_device(r.data_ptr(), z.data_ptr(), 2, st.cuda_stream, True)

                def apply_once():
                    ctx.apply_device(r.data_ptr(), z.data_ptr(), 2, st.cuda_stream, False)

                def gnn_once():
                    ctx.launch_gnn_only(r.data_ptr(), st.cuda_stream)

                ta, tg = [], []
                for _ in range(args.reps):
                    for dst, fn in ((ta, apply_once), (tg, gnn_once)):
                        flush.zero_()
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(st)
                        fn()
                        e1.record(st)
                        torch.cuda.synchronize()
                        dst.append(e0.elapsed_time(e1))
                gms = float(np.median(tg))
                fl = gnn_flops_exec(kb, dd, info["V"], info["E"], h0)
                fs = gnn_flops(kb, dd, info["V"], info["E"])
                print(json.dumps({
                    "N_s": ns, "overlap": ov, "k_bar": kb, "d": dd, "N": prob.system.n, "K": info["K"],
                    "V": info["V"], "E": info["E"], "k_max": info["k_max"], "n_big": info["n_big"],
                    "apply_ms": float(np.median(ta)), "gnn_ms": gms,
                    "gnn_tflops": fl / (gms * 1e-3) / 1e12,
                    "frac_fp32": fl / (gms * 1e-3) / 1e12 / peak,
                    "F_gnn_tflops": fs / (gms * 1e-3) / 1e12,
                    "frac_fp32_F_gnn": fs / (gms * 1e-3) / 1e12 / peak, "peak": peak,
                    "subdomain_node_layers_per_s": info["V"] * kb / (gms * 1e-3),
                    "problem_build_s": t_build}), flush=True)
                del p


if __name__ == "__main__":
    main()
