"""Record the reference's CPU time-to-solution at a BASELINE config (run on the
GPU box's host): PCG-DDM-GNN to 1e-6 (sparse.py:76-127 + hybrid.py:112-136, as
restated by oracle/ddm_oracle.py and spread over all host cores by
oracle/parallel.py), desk weights, two-level.  bench.py reports the newest
profiles/r*_cpu_pcg_<cfg>.json beside the GPU time-to-solution.

    python tools/cpu_pcg.py B gpurun_out/r02_cpu_pcg_B.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import ddm_oracle as orc  # noqa: E402
from oracle.parallel import ParallelOracle  # noqa: E402
import workload  # noqa: E402

TARGETS = {"A": 5000, "B": 100_000, "C": 1_000_000}


def main(cfg, out_path):
    w = workload.load(TARGETS[cfg], 1000, 2, build_in_child=True)
    m = orc.load_model(os.path.join(ROOT, "tests", "golden", "desk_k10_d10.dss"))
    t0 = time.perf_counter()
    with ParallelOracle(w.a, w.coords, w.subdomains, m, level="two") as pre:
        t_setup = time.perf_counter() - t0
        t0 = time.perf_counter()
        _u, it, hist, conv = orc.pcg(w.a, w.b, pre, 1e-6, 1000)
        secs = time.perf_counter() - t0
        nw = pre.workers
    rec = {"config": f"{cfg} (N={w.n}, K={w.k})", "seconds": secs, "iterations": it,
           "converged": conv, "final_relres": hist[-1], "setup_s": t_setup,
           "weights": "tests/golden/desk_k10_d10.dss", "processes": nw,
           "blas_threads_per_process": 1, "host": bench.host_info(),
           "made_by": "tools/cpu_pcg.py"}
    with open(out_path, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
