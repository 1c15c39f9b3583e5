"""Benchmark of the DDM-GNN hot path on B200.

Workload (BASELINE.json configs[2], "C"): 2D Poisson P1 blob mesh with
~1M nodes (generate_blob_mesh(0, 1_000_000, 0.2), coefficients seed (0,1)),
partition(A, 1000, 0), overlap 2 -> N=996,546 DOFs, K=997 subdomains,
two-level DDM-GNN (k_bar=10, d=10, random-init weights init_model(10,10,seed=1)),
built on the box by the native problem builder (bit-identical to the reference).

A "step" is one preconditioner application z = M r over the whole problem
(restriction + batched GNN over all 997 subdomains + coarse solve + gluing).
  value  = precond applies/sec, device-timed with CUDA events per step, inputs
           resident in HBM, L2 flushed (256 MB write) before every step.
  e2e    = same metric through the C ABI with HOST buffers (ddmgnn_apply_host:
           pinned H2D of r, apply, D2H of z inside the timed region).
Also reported: the fused GNN kernel's roofline (FP32 CUDA-core bound), the
SpMV's HBM roofline, a full PCG solve (time per iteration / time-to-solution),
and the CPU baseline (the oracle restatement of the reference, numpy/OpenBLAS
on the host cores, on a bounded sample of subdomains).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import signal
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-solution to 1e-6 (s) and precond applies/sec, 1/2/4/8 B200 vs host CPU"
UNIT = "precond applies/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--target-nodes", type=int, default=1_000_000)
    ap.add_argument("--subdomain-size", type=int, default=1000)
    ap.add_argument("--overlap", type=int, default=2)
    ap.add_argument("--kbar", type=int, default=10)
    ap.add_argument("--d", type=int, default=10)
    ap.add_argument("--level", default="two", choices=["one", "two"])
    ap.add_argument("--weights", default="random", help="'random' or a dss-v1 file")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-pcg", action="store_true")
    ap.add_argument("--pcg-weights", default=os.path.join(ROOT, "tests", "golden", "desk_k10_d10.dss"),
                    help="weights of the time-to-solution leg (trained; random weights do not "
                         "converge, SURVEY.md finding 4)")
    ap.add_argument("--pcg-max-iter", type=int, default=1000)
    ap.add_argument("--exchange", default="p2p", choices=["collective", "p2p"],
                    help="multi-GPU exchanges: device-flag-ordered peer-memory puts and "
                         "all-reduces, graph-replayed (p2p), or torch.distributed NCCL "
                         "collectives issued from the host (collective)")
    return ap.parse_args()


def gnn_flops(k_bar, d, v, e):
    """SURVEY.md §8d's F_gnn: minimal factorised FP32 flops of one GNN apply."""
    per_node = (8 * d * d + 2 * d) + (4 * d * d + 4 * d) + (2 * (3 * d + 1) * d + 2 * d * d + 2 * d) + 2 * d
    return float(k_bar * (per_node * v + 16 * d * e) + (2 * d * d + 2 * d) * v)


def gnn_flops_exec(k_bar, d, v, e, h0_skip=False):
    """FP32 flops the fused kernel executes (FMA = 2, relu not counted):
    per node and layer Q and P ((d+2) -> 2d each), psi first layer ((3d+2) -> d with the
    messages' second layer folded in), psi second layer (d -> d), h update (d), and the
    shift-form edge loop's width * P FMA (2d); per edge and layer y = Q + |d| WL (FMA)
    and the sum add over 2d hidden units (the max is not counted); decoder once.
    With h0_skip the first layer skips the h rows of P, Q and psi (h = 0)."""
    dh = (d + 1) // 2 * 2
    per_node = (2 * (2 * (d + 2) * 2 * d) + 2 * (3 * d + 2) * dh + 2 * d * dh + 2 * dh
                + 2 * 2 * d)
    per_edge = 2 * d * (2 + 1)
    skipped = (2 * (2 * d * 2 * d) + 2 * d * dh) * v if h0_skip else 0
    return float(k_bar * (per_node * v + per_edge * e) + (2 * d * dh + 2 * d) * v - skipped)


def fp32_peak_tflops(sm_mhz):
    """FP32 CUDA-core peak: the FFMA2 microbenchmark measured on this pool's B200s
    (profiles/r02_fp32_peak.json, tools/ubench/fp32_peak.cu, with its clock record),
    else the nominal 148 SM x 128 lanes x 2 flop x sm_max_mhz."""
    nominal = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "r02_fp32_peak.json")))
        return float(rec["fp32_ffma2_tflops"]), (
            f"measured FFMA2 peak {rec['fp32_ffma2_tflops']:.1f} TFLOP/s at "
            f"{rec.get('sm_mhz_median', '?')} MHz (profiles/r02_fp32_peak.json, "
            f"tools/ubench/fp32_peak.cu); nominal {nominal:.1f} at {sm_mhz:.0f} MHz")
    except (OSError, ValueError, KeyError):
        return nominal, ("nominal 148 SM x 128 FP32 lanes x 2 flop x sm_max_mhz (no measured "
                         "FP32 figure committed)")


def profiled_traffic(kernel):
    """DRAM bytes per launch from this round's committed ncu capture (profiles/)."""
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), reverse=True):
        try:
            t = json.load(open(path))[kernel]
            return t["traffic_bytes"], os.path.relpath(path, ROOT)
        except (OSError, ValueError, KeyError):
            continue
    return None, None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self._proc = None
        return self

    def pause(self):
        """Stop polling (SIGSTOP) while host-timed work runs: an nvidia-smi query
        holds the driver for milliseconds and would land inside host-clocked steps."""
        if self._proc:
            self._proc.send_signal(signal.SIGSTOP)

    def resume(self):
        if self._proc:
            self._proc.send_signal(signal.SIGCONT)

    def _read(self):
        for line in self._proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self._proc:
            time.sleep(0.25)
            self._proc.terminate()
            self._proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def load_workload(args, build_in_child):
    """The cached config (workload.py): both arms time the same A, b, coords and
    subdomains; the reference process reads it with numpy only."""
    import workload

    return workload.load(args.target_nodes, args.subdomain_size, args.overlap,
                         build_in_child=build_in_child)


def weights_desc(args):
    return ("random init_model(%d,%d,seed=1)" % (args.kbar, args.d) if args.weights == "random"
            else os.path.relpath(args.weights, ROOT))


def config_obj(args, w, world):
    """The `config` object both arms print (identical for the same launch)."""
    return {
        "workload": f"C: blob mesh target {args.target_nodes} nodes (N={w.n}), "
                    f"N_s={args.subdomain_size}, overlap {args.overlap}, K={w.k}, V={w.v}, "
                    f"{args.level}-level DDM-GNN k_bar={args.kbar} d={args.d}, weights "
                    f"{weights_desc(args)}",
        "step": "one full preconditioner apply z = M r (hybrid.py:112-136: restriction, "
                "K local GNN solves, coarse solve, gluing) on r = default_rng(0).standard_normal(N)",
        "l2": "GPU arm: L2 flushed (256 MB write) before every timed step",
        "parallelism": f"{world} GPU rank(s)" + (" (subdomain shards)" if world > 1 else "")
                       + "; reference arm: rank 0 on all host cores",
    }


def load_model(args):
    import paper_2402_08296_b200 as ddm

    if args.weights == "random":
        return ddm.init_model(args.kbar, args.d, seed=1)
    return ddm.load_model(args.weights)


def oracle_model(args):
    from oracle import ddm_oracle as orc

    if args.weights == "random":
        return orc.model_from_flat(args.kbar, args.d, 1e-3, 1,
                                   orc.init_model_flat(args.kbar, args.d, 1))
    return orc.load_model(args.weights)


# ----------------------------------------------------------------------------- CPU legs


def host_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(),
            "blas_threads_per_process": 1,
            "numpy": np.__version__}


def cpu_full_applies(w, args, steps, warmup, workers=None):
    """The reference's full apply (hybrid.py:112-136 restated in oracle/ddm_oracle.py
    and spread over host cores by oracle/parallel.py: all K subdomains' forwards,
    the coarse lu_solve and the gluing) timed per step on the host clock."""
    from oracle.parallel import ParallelOracle

    r = np.random.default_rng(0).standard_normal(w.n)
    t0 = time.perf_counter()
    with ParallelOracle(w.a, w.coords, w.subdomains, oracle_model(args), level=args.level,
                        workers=workers) as par:
        t_setup = time.perf_counter() - t0
        for _ in range(warmup):
            par(r)
        times = []
        for _ in range(steps):
            t1 = time.perf_counter()
            z = par(r)
            times.append(time.perf_counter() - t1)
        # where the time goes on the host: the parent's coarse solve + gluing
        t1 = time.perf_counter()
        if args.level == "two":
            par.coarse_term(r)
        t_coarse = time.perf_counter() - t1
        nw = par.workers
    return {"times_s": times, "setup_s": t_setup, "workers": nw, "coarse_s": t_coarse,
            "z_norm": float(np.linalg.norm(z))}


def cpu_single_core(w, args, frac=0.03, seed=0):
    """One core (one process, one BLAS thread): the oracle forward over a random
    sample of subdomains, extrapolated linearly in subdomain nodes."""
    from threadpoolctl import threadpool_limits

    from oracle import ddm_oracle as orc

    rng = np.random.default_rng(seed)
    k = w.k
    sample = np.sort(rng.choice(k, max(1, int(round(frac * k))), replace=False))
    om = oracle_model(args)
    r = np.random.default_rng(0).standard_normal(w.n)
    graphs = [orc.local_graph(w.a, w.subdomains[i], w.coords) for i in sample]
    cs = [r[w.subdomains[i]] / np.linalg.norm(r[w.subdomains[i]]) for i in sample]
    v_s = sum(g.node_count for g in graphs)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        orc.forward(om, graphs, cs)
        t = time.perf_counter() - t0
    return {"seconds_per_apply_extrapolated": t * w.v / v_s,
            "sample": f"{sample.size}/{k} random subdomains ({v_s}/{w.v} subdomain nodes), "
                      f"forward only, 1 process x 1 BLAS thread, extrapolated linearly in V"}


def cpu_pcg_config_a():
    """The reference's end-to-end PCG-DDM-GNN (sparse.py:76-127 + hybrid.py:112-136,
    restated) at BASELINE config A with the pinned desk weights, one worker
    process per subdomain (oracle/parallel.py)."""
    import scipy.sparse as sp

    from oracle import ddm_oracle as orc

    g = np.load(os.path.join(ROOT, "tests", "golden", "A.npz"))
    n = g["b"].shape[0]
    a = sp.csr_matrix((g["data"], g["indices"], g["indptr"]), shape=(n, n))
    ptr, idx = g["sub_ptr"], g["sub_idx"]
    subs = [idx[ptr[i]:ptr[i + 1]] for i in range(len(ptr) - 1)]
    from oracle.parallel import ParallelOracle

    m = orc.load_model(os.path.join(ROOT, "tests", "golden", "desk_k10_d10.dss"))
    t0 = time.perf_counter()
    with ParallelOracle(a, g["coords"], subs, m, level="two") as pre:
        t_setup = time.perf_counter() - t0
        t0 = time.perf_counter()
        _u, it, hist, conv = orc.pcg(a, g["b"], pre, 1e-6, 500)
        secs = time.perf_counter() - t0
        nw = pre.workers
    return {"config": "A (N=%d, K=%d)" % (n, len(subs)), "seconds": secs,
            "iterations": it, "converged": conv, "final_relres": hist[-1],
            "setup_s": t_setup, "weights": "tests/golden/desk_k10_d10.dss",
            "processes": nw, "blas_threads_per_process": 1}


def cpu_pcg_record(cfg):
    """Recorded CPU PCG of a config too long for every bench run (tools/cpu_pcg.py)."""
    import glob

    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_cpu_pcg_{cfg}.json")),
                       reverse=True):
        try:
            rec = json.load(open(path))
            rec["record"] = os.path.relpath(path, ROOT)
            return rec
        except (OSError, ValueError):
            continue
    return None


def cpu_baseline(w, args, steps=2):
    """cpu_baseline of the GPU arm (rank 0, N=1): full oracle applies on all host
    cores (a bounded sample of the workload: `steps` applies), the one-core figure,
    and the CPU time-to-solution at config A (and B from its record)."""
    full = cpu_full_applies(w, args, steps=steps, warmup=1)
    sec = float(np.median(full["times_s"]))
    single = cpu_single_core(w, args)
    return {
        "value": 1.0 / sec, "unit": UNIT, "cores": full["workers"], "kind": "port",
        "sample": f"{steps} full applies (all {w.k} subdomains + coarse lu_solve + gluing, "
                  f"hybrid.py:112-136) of oracle/ddm_oracle.py over {full['workers']} "
                  f"processes x 1 BLAS thread (oracle/parallel.py), after 1 warm-up apply",
        "seconds_per_apply": sec, "seconds_per_apply_all": full["times_s"],
        "coarse_solve_s": full["coarse_s"], "setup_s": full["setup_s"],
        "single_core": single, "host": host_info(),
        "pcg_config_a": cpu_pcg_config_a(), "pcg_config_b": cpu_pcg_record("B"),
    }


def mapped_repo_libs():
    """Shared objects of this repository mapped into this process (/proc/self/maps)."""
    found = set()
    try:
        for line in open("/proc/self/maps"):
            path = line.split()[-1] if line.strip() else ""
            if path.startswith(ROOT) and ".so" in os.path.basename(path):
                found.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(found)


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path (the oracle
    port of hybrid.py:112-136, pinned to the reference's own outputs) on all host
    cores, one FULL apply of the config per step.  Rank 0 only; reads the workload
    from the .npz cache (no native library of this repository in this process)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    w = load_workload(args, build_in_child=True)
    res = cpu_full_applies(w, args, steps=args.steps, warmup=args.warmup)
    times = res["times_s"]
    ms = 1e3 * float(np.mean(times))
    v = 1e3 / ms
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_obj(args, w, world),
        "cpu_baseline": {
            "value": v, "unit": UNIT, "cores": res["workers"], "kind": "port",
            "sample": f"every step one full apply over all {w.k} subdomains (forwards + coarse "
                      f"lu_solve + gluing, hybrid.py:112-136), oracle/ddm_oracle.py over "
                      f"{res['workers']} processes x 1 BLAS thread (oracle/parallel.py)",
            "seconds_per_step": times, "setup_s": res["setup_s"], "host": host_info(),
        },
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "problem_source": w.source,
        "native_libs_mapped": mapped_repo_libs(),
        "pcg_config_a": cpu_pcg_config_a(),
        "pcg_config_b": cpu_pcg_record("B"),
    }
    print(json.dumps(out))


# ----------------------------------------------------------------------------- GPU arm


def time_to_solution(ddm, p, a, b_host, args, lvl, dev, stream, weights=None, flexible=False,
                     restore=True):
    """Device-timed PCG (sparse.py:76-127) to 1e-6 with trained weights: warm-up
    solve (captures the CUDA graphs), then one solve between CUDA events on the
    solve's stream; setup excluded (as cli.py:195-199 minus the build).
    ``flexible``: the opt-in flexible CG."""
    import torch

    ctx = p.context
    weights = weights or args.pcg_weights
    p.reload_model(ddm.load_model(weights))
    b = torch.tensor(b_host, device=dev)
    u = torch.empty_like(b)
    s = stream.cuda_stream
    ctx.pcg(b.data_ptr(), None, 1e-6, args.pcg_max_iter, lvl, True, u.data_ptr(), s,
            flexible=flexible)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _u, it, hist, conv = ctx.pcg(b.data_ptr(), None, 1e-6, args.pcg_max_iter, lvl, True,
                                 u.data_ptr(), s, flexible=flexible)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    sec = e0.elapsed_time(e1) / 1e3
    uh = u.cpu().numpy()
    true_rel = float(np.linalg.norm(b_host - a @ uh) / np.linalg.norm(b_host))
    if restore:
        p.reload_model(load_model(args))
    return {"seconds": sec, "iterations": it, "converged": conv, "final_relres": hist[-1],
            "true_relres": true_rel, "ms_per_iteration": 1e3 * sec / max(1, it),
            "max_iter": args.pcg_max_iter, "tol": 1e-6, "solver": "fcg" if flexible else "pcg",
            "weights": os.path.relpath(weights, ROOT),
            "timing": "CUDA events on the solve stream, device-resident b/u, graphs warm"}


def gpu_tts_small(ddm, args, dev, stream):
    """Device time-to-solution at BASELINE configs A and B (desk weights, two-level),
    beside the CPU's (cpu_baseline.pcg_config_a / pcg_config_b)."""
    import scipy.sparse as sp

    from paper_2402_08296_b200.problem import ProblemConfig, build_problem

    out = {}
    g = np.load(os.path.join(ROOT, "tests", "golden", "A.npz"))
    n = g["b"].shape[0]
    a = sp.csr_matrix((g["data"], g["indices"], g["indptr"]), shape=(n, n))
    ptr, idx = g["sub_ptr"], g["sub_idx"]
    subs = [idx[ptr[i]:ptr[i + 1]] for i in range(len(ptr) - 1)]
    dec = ddm.finish_decomposition(subs, g["owner"], int(g["overlap"]))
    problems = {"A": (a, g["b"], g["coords"], dec)}
    pb = build_problem(0, ProblemConfig(100_000, 0.2, 1000, 2))
    problems["B"] = (pb.system.a, pb.system.b, pb.coords, pb.dec)
    for name, (a, b, coords, dec) in problems.items():
        model = ddm.load_model(args.pcg_weights)
        p = ddm.build_ddm_gnn(a, coords, dec, model, level="two", device=dev.index or 0)
        out[name] = time_to_solution(ddm, p, a, b, args, 2, dev, stream, restore=False)
        out[name]["config"] = f"{name} (N={b.size}, K={dec.n_subdomains})"
        del p
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # DDMGNN_BENCH_BACKEND=gloo runs the sharded path with several ranks per GPU
        # (host-staged collectives) — a functional check on a one-GPU box
        backend = os.environ.get("DDMGNN_BENCH_BACKEND", "nccl")
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
        return run_sharded(args, world, rank, local)
    w = load_workload(args, build_in_child=False)
    # the CPU baseline first, before this process initialises CUDA (its worker
    # processes are forked)
    cpu = cpu_baseline(w, args) if (world == 1 and rank == 0 and not args.no_cpu) else None
    torch.cuda.set_device(local)

    import paper_2402_08296_b200 as ddm

    dec = ddm.finish_decomposition(w.subdomains, w.owner, w.overlap)
    model = load_model(args)
    t0 = time.perf_counter()
    p = ddm.build_ddm_gnn(w.a, w.coords, dec, model, level=args.level, device=local)
    t_build = time.perf_counter() - t0
    info = p.info()
    ctx = p.context
    n = w.n
    lvl = 2 if args.level == "two" else 1
    dev = torch.device(f"cuda:{local}")
    r = torch.tensor(np.random.default_rng(0).standard_normal(n), device=dev)
    z = torch.empty_like(r)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2
    stream = torch.cuda.Stream(dev)  # events and kernels on the same (non-default) stream
    torch.cuda.set_stream(stream)
    s = stream.cuda_stream

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # warmup (also checks the apply for non-finite states once)
    ctx.apply_device(r.data_ptr(), z.data_ptr(), lvl, s, True)
    for _ in range(max(0, args.warmup - 1)):
        ctx.apply_device(r.data_ptr(), z.data_ptr(), lvl, s, False)
    barrier()

    # ---- device-timed applies (per-step events, L2 flushed outside the events) ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    gnn_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        barrier()
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            ctx.apply_device(r.data_ptr(), z.data_ptr(), lvl, s, False)
            ev[i][1].record(stream)
        barrier()
        # the dominant kernel alone (restriction + fused GNN), same stream
        for i in range(args.steps):
            flush.zero_()
            gnn_ev[i][0].record(stream)
            ctx.launch_gnn_only(r.data_ptr(), s)
            gnn_ev[i][1].record(stream)
        barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    gnn_ms = sum(a.elapsed_time(b) for a, b in gnn_ev) / args.steps
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * 1e3 / ms_max

    # ---- SpMV roofline (HBM) ----
    a = w.a
    x = torch.tensor(np.ones(n), device=dev)
    y = torch.empty_like(x)
    for _ in range(3):
        ctx.spmv_device(x.data_ptr(), y.data_ptr(), s)
    sp_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for e0, e1 in sp_ev:
        flush.zero_()
        e0.record(stream)
        ctx.spmv_device(x.data_ptr(), y.data_ptr(), s)
        e1.record(stream)
    torch.cuda.synchronize(dev)
    spmv_ms = sum(e0.elapsed_time(e1) for e0, e1 in sp_ev) / len(sp_ev)
    spmv_bytes = 12 * a.nnz + 20 * n

    # ---- end to end through the C ABI with host buffers (pinned, per the contract) ----
    r_pin = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).pin_memory()
    z_pin = torch.empty(n, dtype=torch.float64).pin_memory()
    r_host, z_host = r_pin.numpy(), z_pin.numpy()
    # host-clocked, so more steps than the device-timed loop (short host-timed
    # loops are noisy: CPU clock ramp, scheduler)
    e2e_steps = max(args.steps, 100)
    for _ in range(max(args.warmup, 10)):
        ctx.apply_host(r_host, lvl, out=z_host)
    clk.pause()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ctx.apply_host(r_host, lvl, out=z_host)
    t_e2e = (time.perf_counter() - t0) / e2e_steps
    clk.resume()
    e2e_t = torch.tensor([t_e2e], device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = world / float(e2e_t.item())

    # ---- time-to-solution: device-resident PCG to 1e-6 (trained weights) ----
    pcg = pcg_trained = pcg_flex = fcg_trained = tts_small = None
    if not args.no_pcg:
        pcg = time_to_solution(ddm, p, w.a, w.b, args, lvl, dev, stream)
        pcg_flex = time_to_solution(ddm, p, w.a, w.b, args, lvl, dev, stream, flexible=True)
        # weights trained on the GPU for this subdomain size (tools/train_gpu.py), if present
        for cand in ("gpu_k10_ns1000_long.dss", "gpu_k10_ns1000.dss"):
            path = os.path.join(ROOT, "weights", cand)
            if os.path.exists(path) and args.subdomain_size == 1000 and args.kbar == 10:
                pcg_trained = time_to_solution(ddm, p, w.a, w.b, args, lvl, dev, stream, path)
                fcg_trained = time_to_solution(ddm, p, w.a, w.b, args, lvl, dev, stream, path,
                                               flexible=True)
                break
        if world == 1:
            tts_small = gpu_tts_small(ddm, args, dev, stream)

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "MEASURED_PEAKS.json (of measured)" if "hbm_gbs" in peaks else \
        "fallback 6.65 TB/s from B200_PROFILING.md (of fallback; MEASURED_PEAKS.json absent)"
    sm_mhz = peaks.get("sm_max_mhz") or clk.summary().get("sm_max_mhz") or 1965.0
    fp32_peak, fp32_src = fp32_peak_tflops(sm_mhz)
    h0 = os.environ.get("DDMGNN_H0_SKIP", "1") != "0"
    flops_exec = gnn_flops_exec(info["k_bar"], info["d"], info["V"], info["E"], h0)
    flops_survey = gnn_flops(info["k_bar"], info["d"], info["V"], info["E"])
    # the contract's algorithmic figure: SURVEY.md §8(d)'s F_gnn per launch
    achieved = flops_survey / (gnn_ms * 1e-3) / 1e12
    achieved_exec = flops_exec / (gnn_ms * 1e-3) / 1e12
    gnn_traffic, traffic_src = profiled_traffic("gnn_kernel")
    spmv_traffic, _ = profiled_traffic("spmv_kernel")
    # per chunk: gnn_kernel, one launch per cluster size, and for subdomains beyond an
    # 8-CTA cluster the flat path (prologue in the first chunk + 2 launches per layer)
    n_gnn_launches = ctx.gnn_launches()
    per_step_launches = n_gnn_launches + (1 if lvl == 2 else 0) + 1
    clocks = clk.summary()
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 GNN / f64 Krylov+gluing",
            "data": "synthetic (reference problem generator restated natively; random-init weights)",
            "config": config_obj(args, w, world),
            "layout": {"E": info["E"], "E_pad": info["E_pad"], "k_max": info["k_max"],
                       "n_cluster": info["n_cluster"], "problem_source": w.source},
            "roofline": {
                "kernel": "gnn_kernel + concurrent gnn_cluster_kernel (fused restriction + "
                          f"{info['k_bar']} message-passing layers + decoder)",
                "bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": achieved / fp32_peak, "traffic": gnn_traffic,
                "traffic_source": traffic_src,
                "algorithmic": f"SURVEY.md §8(d) F_gnn = k(2120 V + 160 E) + 220 V (d=10) = "
                               f"{flops_survey:.3e} per launch (V={info['V']}, E={info['E']})",
                "executed_flops": flops_exec,
                "executed_tflops": achieved_exec,
                "frac_executed": achieved_exec / fp32_peak,
                "executed_note": "FP32 flops the kernel actually issues: k(1860 V + 60 E) + 220 V"
                                 + (" - 1000 V (layer 1 on h = 0)" if h0 else "")
                                 + " at d=10 (FMA = 2, relu not counted; DESIGN.md §4)",
                "peak_source": fp32_src,
                "gnn_ms": gnn_ms, "share_of_step": gnn_ms / ms,
            },
            "roofline_spmv": {
                "bound": "hbm", "achieved": spmv_bytes / (spmv_ms * 1e-3) / 1e9, "peak": hbm_peak,
                "unit": "GB/s", "frac": spmv_bytes / (spmv_ms * 1e-3) / 1e9 / hbm_peak,
                "traffic": spmv_traffic, "ms": spmv_ms, "algorithmic_bytes": spmv_bytes,
                "peak_source": hbm_src,
            },
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "steps": e2e_steps, "h2d_bytes_per_step": 8 * n,
                    "d2h_bytes_per_step": 8 * n},
            "gpu_launches": per_step_launches * args.steps,
            "clocks": clocks,
            "pcg": pcg,
            "pcg_flexible": pcg_flex,
            "pcg_trained_weights": pcg_trained,
            "pcg_flexible_trained_weights": fcg_trained,
            "time_to_solution_small": tts_small,
            "setup_s": {"problem_load": w.seconds, "preconditioner_build": t_build},
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def run_sharded(args, world, rank, local):
    """N GPUs, one process each: the config's subdomains sharded across the ranks
    (paper_2402_08296_b200/sharded.py).  With --exchange p2p (default) the halo /
    term exchanges, the all-gather and the dot all-reduces are device-flag-ordered
    puts over CUDA-IPC peer memory (NVLink), so one apply and one PCG iteration are
    CUDA graphs replayed with no host barrier; --exchange collective issues NCCL
    collectives from the host instead.  Strong scaling: the whole problem is fixed,
    `value` = applies/s of the whole problem, device time = max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_2402_08296_b200 as ddm
    from paper_2402_08296_b200.sharded import ShardedDdmGnn

    dev = torch.device(f"cuda:{local}")
    w = load_workload(args, build_in_child=False)
    dec = ddm.finish_decomposition(w.subdomains, w.owner, w.overlap)
    model = load_model(args)
    t0 = time.perf_counter()
    exchange = args.exchange
    try:
        sh = ShardedDdmGnn(w.a, w.coords, dec, model, level=args.level, device=local,
                           exchange=exchange)
    except Exception as exc:  # no peer mappings on this box: host-issued collectives
        print(f"[bench] p2p exchange unavailable ({exc!r}); using collectives", file=sys.stderr)
        exchange = "collective"
        sh = ShardedDdmGnn(w.a, w.coords, dec, model, level=args.level, device=local,
                           exchange=exchange)
    t_build = time.perf_counter() - t0
    r_glob = np.random.default_rng(0).standard_normal(w.n)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    r = sh.owned_part(r_glob)
    z = torch.empty_like(r)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    graph = sh.capture_apply(r, z) if sh.device_ordered else None

    def step():
        if graph is not None:
            graph.replay()
        else:
            sh.apply_owned(r, z)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)
    dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    t = torch.tensor([ms], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    # end to end: host r (owned part) in, host z (owned part) out, every step
    r_host = torch.from_numpy(r_glob[sh.plan.owned].copy()).pin_memory()
    z_host = torch.empty_like(r_host).pin_memory()
    torch.cuda.synchronize(dev)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r.copy_(r_host, non_blocking=True)
        step()
        z_host.copy_(z, non_blocking=True)
        stream.synchronize()
    e2e = torch.tensor([(time.perf_counter() - t0) / args.steps], device=dev)
    dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    pcg = None
    if not args.no_pcg:
        sh.close()
        sh = ShardedDdmGnn(w.a, w.coords, dec, ddm.load_model(args.pcg_weights),
                           level=args.level, device=local, exchange=exchange)
        sh.pcg(w.b, 1e-6, 3)  # warm-up (graph capture, communicators)
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        u, rep = sh.pcg(w.b, 1e-6, args.pcg_max_iter)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        tt = torch.tensor([time.perf_counter() - t0, e0.elapsed_time(e1) / 1e3], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        true_rel = float(np.linalg.norm(w.b - w.a @ u) / np.linalg.norm(w.b))
        pcg = {"seconds": float(tt[1].item()), "host_seconds": float(tt[0].item()),
               "iterations": rep.iterations, "converged": rep.converged,
               "final_relres": rep.final_relres, "true_relres": true_rel,
               "weights": os.path.relpath(args.pcg_weights, ROOT),
               "timing": "CUDA events around the whole collective solve on each rank's "
                         "stream (incl. the host's status polls), max over ranks"}
    if rank == 0:
        out = {
            "metric": METRIC, "value": 1e3 / ms_max, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 GNN / f64 Krylov+gluing",
            "data": "synthetic (reference problem generator restated natively; random-init weights)",
            "config": config_obj(args, w, world),
            "sharding": {"exchange": exchange, "graph": graph is not None,
                         "ranks": world},
            "e2e": {"value": 1.0 / float(e2e.item()), "unit": UNIT,
                    "h2d_bytes_per_step": 8 * sh.plan.n_own, "d2h_bytes_per_step": 8 * sh.plan.n_own},
            "gpu_launches": sh.launches_per_apply() * args.steps, "clocks": clk.summary(),
            "pcg": pcg,
            "setup_s": {"problem_load": w.seconds, "preconditioner_build": t_build},
        }
        print(json.dumps(out))
    sh.close()
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
