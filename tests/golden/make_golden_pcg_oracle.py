"""PCG-DDM-GNN residual histories at BASELINE configs B and C (goldens).

The reference itself needs 4 s (B) to 45 s (C) per preconditioner apply on one
core (SURVEY.md finding 8), so its PCG at C is a 5-hour job.  These goldens are
produced instead by the CPU oracle — the float64 restatement of
``apply_ddm_gnn`` (hybrid.py:112-136) and ``pcg`` (sparse.py:76-127) that
tests/test_oracle_golden.py pins to the reference's own outputs (apply to
1e-13, PCG histories to 1e-10) — run over all host cores
(oracle/parallel.py).  The problem is the native builder's, which is
bit-identical to the reference builder (tests/golden/builder_B.json, and
builder_C.json once the reference's hours-long C build finishes).

    python tests/golden/make_golden_pcg_oracle.py B two desk
    python tests/golden/make_golden_pcg_oracle.py C two desk [workers]

Writes tests/golden/pcg_<cfg>_<level>_<weights>[_fcg].json with the full
relative-residual history, the iteration count and the convergence flag.
"""

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ddm_oracle as orc  # noqa: E402
from oracle.parallel import ParallelOracle  # noqa: E402

TARGETS = {"A": 5000, "B": 100_000, "C": 1_000_000}
WEIGHTS = {"desk": os.path.join(HERE, "desk_k10_d10.dss"),
           "gpu": os.path.join(ROOT, "weights", "gpu_k10_ns1000.dss")}


def main(cfg, level, weights, workers=None, flexible=False, max_iter=1000):
    from paper_2402_08296_b200.problem import ProblemConfig, build_problem

    prob = build_problem(0, ProblemConfig(TARGETS[cfg], 0.2, 1000, 2))
    a, b = prob.system.a, prob.system.b
    model = orc.load_model(WEIGHTS[weights])
    t0 = time.perf_counter()
    with ParallelOracle(a, prob.coords, prob.dec.subdomains, model, level=level,
                        workers=workers) as P:
        t_setup = time.perf_counter() - t0
        t0 = time.perf_counter()
        _u, it, hist, conv = orc.pcg(a, b, P, 1e-6, max_iter, flexible=flexible)
        secs = time.perf_counter() - t0
        nw = P.workers
    out = {"config": cfg, "level": level, "weights": os.path.relpath(WEIGHTS[weights], ROOT),
           "solver": "fcg" if flexible else "pcg", "tol": 1e-6, "max_iter": max_iter,
           "n": int(b.size), "iterations": int(it), "converged": bool(conv),
           "history": [float(x) for x in hist],
           "oracle_seconds": round(secs, 1), "oracle_setup_seconds": round(t_setup, 1),
           "workers": nw,
           "made_by": "tests/golden/make_golden_pcg_oracle.py (oracle/parallel.py + "
                      "oracle/ddm_oracle.py pcg)"}
    name = f"pcg_{cfg}_{level}_{weights}{'_fcg' if flexible else ''}.json"
    with open(os.path.join(HERE, name), "w") as fh:
        json.dump(out, fh)
    print(name, it, conv, hist[-1], f"{secs:.0f}s")


if __name__ == "__main__":
    args = [x for x in sys.argv[1:] if not x.startswith("--")]
    flex = "--fcg" in sys.argv
    cfg, level, weights = args[:3]
    workers = int(args[3]) if len(args) > 3 else None
    main(cfg, level, weights, workers, flex)
