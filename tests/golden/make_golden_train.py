"""Golden fixture for the GPU trainer (paper_2402_08296_b200/train.py), produced by
the REFERENCE (read-only /root/reference/pkg/src): a tiny harvested dataset
(dataset.generate, 2 problems) and the parameters after 3 epochs of the
reference's train() (dss.py:392-469) from init_model(3, 4, seed=1).

    python tests/golden/make_golden_train.py   ->  tests/golden/train.npz
"""

import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from ddmgnn.dataset import DatasetConfig, ProblemConfig, generate, load_samples  # noqa: E402
from ddmgnn.dss import TrainConfig, _param_arrays, init_model, train  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def pack(graphs, prefix, out):
    out[f"{prefix}_counts"] = np.array([g.node_count for g in graphs])
    out[f"{prefix}_ecounts"] = np.array([g.edges.shape[0] for g in graphs])
    out[f"{prefix}_edges"] = np.vstack([g.edges for g in graphs])
    out[f"{prefix}_vec"] = np.vstack([g.edge_vec for g in graphs])
    out[f"{prefix}_len"] = np.concatenate([g.edge_len for g in graphs])
    out[f"{prefix}_c"] = np.concatenate([g.c for g in graphs])
    mats = [g.a_local.tocsr() for g in graphs]
    out[f"{prefix}_nnz"] = np.array([m.nnz for m in mats])
    out[f"{prefix}_indptr"] = np.concatenate([m.indptr for m in mats])
    out[f"{prefix}_indices"] = np.concatenate([m.indices for m in mats])
    out[f"{prefix}_data"] = np.concatenate([m.data for m in mats])


def main():
    cfg = DatasetConfig(n_problems=2, problem=ProblemConfig(300, 0.2, 80, 2), seed=7,
                        ratios=(0.5, 0.5, 0.0))
    with tempfile.TemporaryDirectory() as tmp:
        generate(tmp, cfg)
        tr = [s.graph for s in load_samples(f"{tmp}/train.jsonl")][:60]
        va = [s.graph for s in load_samples(f"{tmp}/val.jsonl")][:30]
    model = init_model(3, 4, alpha=1e-3, seed=1)
    trained, log = train(model, tr, va, TrainConfig(epochs=3, batch_size=20, seed=0))
    out = {"flat0": np.concatenate([p.ravel() for p in _param_arrays(model)]),
           "flat3": np.concatenate([p.ravel() for p in _param_arrays(trained)]),
           "log": np.array([[e, t, v, lr] for e, t, v, lr in log])}
    pack(tr, "tr", out)
    pack(va, "va", out)
    np.savez_compressed(os.path.join(HERE, "train.npz"), **out)
    print(len(tr), len(va), log)


if __name__ == "__main__":
    main()
