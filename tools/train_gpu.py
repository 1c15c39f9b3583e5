"""Train DSS weights for larger subdomains on the GPU (paper_2402_08296_b200/train.py):
harvest local problems from DDM-LU-preconditioned solves of blob-mesh problems
(the reference's dataset recipe, dataset.py:95-121, at a chosen subdomain size),
train with the reference's recipe (Adam, clipping, plateau), save dss-v1, and
report the PCG-DDM-GNN iteration count on an evaluation problem.

    python tools/train_gpu.py OUT.dss [--kbar 10] [--ns 1000] [--problems 4]
        [--nodes 100000] [--epochs 30] [--samples 4000] [--eval-nodes 1000000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_08296_b200 as ddm  # noqa: E402
from paper_2402_08296_b200.problem import ProblemConfig, build_problem  # noqa: E402
from paper_2402_08296_b200.train import Trainer, harvest  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--kbar", type=int, default=10)
    ap.add_argument("--d", type=int, default=10)
    ap.add_argument("--ns", type=int, default=1000)
    ap.add_argument("--problems", type=int, default=4)
    ap.add_argument("--nodes", type=int, default=100_000)
    ap.add_argument("--epochs", type=int, default=30)
    ap.add_argument("--samples", type=int, default=4000)
    ap.add_argument("--batch", type=int, default=100)
    ap.add_argument("--eval-nodes", type=int, default=1_000_000)
    ap.add_argument("--init", default=None, help="dss-v1 file to start from")
    ap.add_argument("--select-every", type=int, default=0,
                    help="every N epochs run PCG with the current weights on a validation "
                         "problem and keep the checkpoint with the fewest iterations (the "
                         "training loss is not the solver's objective)")
    args = ap.parse_args()
    rng = np.random.default_rng(20261017)
    t0 = time.perf_counter()
    data = []
    for pid in range(args.problems):
        prob = build_problem(int(rng.integers(0, 2**62)),
                             ProblemConfig(args.nodes, 0.2, args.ns, 2))
        s = harvest(prob, 1e-6, 500, max_samples=args.samples, rng=rng)
        data.append(s)
        print(f"problem {pid}: {len(s)} samples", flush=True)
    n_val = max(1, args.problems // 4)
    train = [x for s in data[n_val:] for x in s]
    val = [x for s in data[:n_val] for x in s][: max(200, args.samples // 4)]
    t_data = time.perf_counter() - t0
    model = ddm.load_model(args.init) if args.init else ddm.init_model(args.kbar, args.d, alpha=1e-3, seed=1)
    best = {"it": None, "epoch": None}
    on_epoch = None
    if args.select_every:
        vprob = build_problem(int(rng.integers(0, 2**62)), ProblemConfig(args.nodes, 0.2, args.ns, 2))

        def on_epoch(epoch, get_model):
            if (epoch + 1) % args.select_every:
                return
            m = get_model()
            p = ddm.build_ddm_gnn(vprob.system.a, vprob.coords, vprob.dec, m)
            _u, rep = ddm.pcg(vprob.system.a, vprob.system.b, p, 1e-6, 2000)
            it = rep.iterations if rep.converged else 10**9
            print(f"  epoch {epoch}: validation PCG iterations {it}", flush=True)
            if best["it"] is None or it < best["it"]:
                best.update(it=it, epoch=epoch)
                ddm.save_model(m, args.out)
    t0 = time.perf_counter()
    trained, log = Trainer(model).fit(train, val, epochs=args.epochs, batch_size=args.batch,
                                      seed=0, log_every=1, on_epoch=on_epoch)
    t_train = time.perf_counter() - t0
    if best["it"] is None:
        ddm.save_model(trained, args.out)
    else:
        trained = ddm.load_model(args.out)
    with open(args.out + ".log.csv", "w") as fh:
        fh.write("epoch,train_loss,val_loss,lr\n")
        for e, tl, vl, lr in log:
            fh.write(f"{e},{tl!r},{vl!r},{lr!r}\n")
    res = {"out": args.out, "train_samples": len(train), "val_samples": len(val),
           "data_s": t_data, "train_s": t_train, "final": log[-1],
           "selected_epoch": best["epoch"], "selected_val_iterations": best["it"]}
    if args.eval_nodes:
        prob = build_problem(0, ProblemConfig(args.eval_nodes, 0.2, args.ns, 2))
        for name, m in (("trained", trained), ("desk", ddm.load_model(os.path.join(
                os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                "desk_k10_d10.dss")))):
            p = ddm.build_ddm_gnn(prob.system.a, prob.coords, prob.dec, m)
            _u, rep = ddm.pcg(prob.system.a, prob.system.b, p, 1e-6, 2000)
            res[f"eval_iterations_{name}"] = rep.iterations
            res[f"eval_converged_{name}"] = rep.converged
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
