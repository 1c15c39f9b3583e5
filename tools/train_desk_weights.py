"""Produce the pinned desk-trained weights file used by the convergence tests.

Runs the reference's own acceptance recipe verbatim
(/root/reference/pkg/tests/test_acceptance.py:36-37,60-69): dataset
`generate(TRAIN_DATASET)` then `train(init_model(10,10,1e-3,seed=1), ...,
TrainConfig(epochs=100, seed=0))`, and saves the result in the reference's
dss-v1 format (dss.py:530-544).  Needs /root/reference (this container only);
the output file is committed under tests/golden/ so the GPU box never needs
the reference.

    OPENBLAS_NUM_THREADS=2 python tools/train_desk_weights.py tests/golden/desk_k10_d10.dss
"""
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")
import ddmgnn as dg  # noqa: E402
from ddmgnn.dataset import DatasetConfig, ProblemConfig, generate, load_samples  # noqa: E402
from ddmgnn.dss import TrainConfig, init_model, save_model  # noqa: E402

TRAIN_PROBLEM = ProblemConfig(target_nodes=600, perturbation=0.2, subdomain_size=110, overlap=2)
TRAIN_DATASET = DatasetConfig(n_problems=20, problem=TRAIN_PROBLEM, seed=20260811)


def main(out_path: str) -> None:
    with tempfile.TemporaryDirectory() as tmp:
        generate(tmp, TRAIN_DATASET)
        train_graphs = [s.graph for s in load_samples(f"{tmp}/train.jsonl")]
        val_graphs = [s.graph for s in load_samples(f"{tmp}/val.jsonl")]
    model = init_model(10, 10, alpha=1e-3, seed=1)
    trained, log = dg.train(model, train_graphs, val_graphs, TrainConfig(epochs=100, seed=0))
    save_model(trained, out_path)
    with open(out_path + ".log.csv", "w") as fh:
        fh.write(dg.dss.training_log_csv(log))
    print("saved", out_path, "final train/val", log[-1][1], log[-1][2])


if __name__ == "__main__":
    main(sys.argv[1])
