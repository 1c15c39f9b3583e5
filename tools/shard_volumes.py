"""Communication volumes of the sharded solve per apply / PCG iteration (from the
shard plans, no GPU): halo DOFs, prolongation terms, collective sizes, and the load
balance of subdomain nodes over ranks, for a BASELINE config and G ranks.

    python tools/shard_volumes.py [--nodes 1000000] [--ranks 2,4,8]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_08296_b200.problem import ProblemConfig, build_problem  # noqa: E402
from paper_2402_08296_b200.sharded import plan_shards  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nodes", type=int, default=1_000_000)
ap.add_argument("--ranks", default="2,4,8")
args = ap.parse_args()
prob = build_problem(0, ProblemConfig(args.nodes, 0.2, 1000, 2))
for g in [int(x) for x in args.ranks.split(",")]:
    plans = plan_shards(prob.system.a, prob.coords, prob.dec, g)
    v = np.array([p.v_own for p in plans])
    halo = np.array([p.halo_recv_pos.size for p in plans])
    terms = np.array([sum(p.term_recv_counts) for p in plans])
    print(json.dumps({
        "N": prob.system.n, "K": prob.dec.n_subdomains, "ranks": g,
        "subdomain_nodes_per_rank_max": int(v.max()), "imbalance": float(v.max() / v.mean()),
        "halo_doubles_per_rank_max": int(halo.max()),
        "term_doubles_per_rank_max": int(terms.max()),
        "bytes_per_apply_per_rank_max": int(8 * (halo.max() + terms.max())),
        "allgather_bytes": int(16 * plans[0].k_slots * g),
    }), flush=True)
