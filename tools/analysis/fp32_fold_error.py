"""Analysis aid (not product, not a test): fp32 numpy emulation of the fused GNN
layer with the algebraic folds used by the CUDA kernel, against the fp64 oracle
forward, on the config-A golden problem.  Prints relative L2 errors of the
concatenated decoder outputs for: baseline fp32 (reference op order), +W2 fold,
+geometry fold (dx,dy folded into per-node projections with per-subdomain
centred fp32 coordinates)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import problem_from  # noqa: E402
from oracle import ddm_oracle as orc  # noqa: E402

f32 = np.float32


def emulate(model, graphs, cs, fold_w2, fold_geo):
    d = model.d
    outs = []
    for g, c in zip(graphs, cs):
        k = g.node_count
        src, dst = g.edges[:, 0], g.edges[:, 1]
        ev = g.edge_vec.astype(f32)
        el = g.edge_len.astype(f32)
        xy = (g.coords - g.coords.mean(axis=0)).astype(f32)
        h = np.zeros((k, d), f32)
        cc = c.astype(f32)
        deg = np.bincount(src, minlength=k).astype(f32)
        for layer in model.layers:
            w_out, b_out = layer["phi_out"][0], layer["phi_out"][1]
            w_in = layer["phi_in"][0].copy()
            w_in[2 * d: 2 * d + 2] *= -1.0
            w1 = np.hstack((w_out, w_in))
            b1 = np.concatenate((b_out, layer["phi_in"][1])).astype(f32)
            wsrc, wdst, wgeo = w1[:d].astype(f32), w1[d:2 * d].astype(f32), w1[2 * d:].astype(f32)
            P = h @ wsrc + b1
            Q = h @ wdst
            if fold_geo:
                P = P - xy @ wgeo[:2]
                Q = Q + xy @ wgeo[:2]
                x = P[src] + Q[dst] + el[:, None] * wgeo[2]
            else:
                x = P[src] + Q[dst] + ev @ wgeo[:2] + el[:, None] * wgeo[2]
            x = np.maximum(x, f32(0))
            S = np.zeros((k, 2 * d), f32)
            np.add.at(S, src, x)
            wp1, bp1, wp2, bp2 = layer["psi"]
            w2o, b2o, w2i, b2i = layer["phi_out"][2], layer["phi_out"][3], layer["phi_in"][2], layer["phi_in"][3]
            if fold_w2:
                mo = (w2o @ wp1[d + 1:2 * d + 1]).astype(f32)
                mi = (w2i @ wp1[2 * d + 1:]).astype(f32)
                bdeg = (b2o @ wp1[d + 1:2 * d + 1] + b2i @ wp1[2 * d + 1:]).astype(f32)
                u = (h @ wp1[:d].astype(f32) + cc[:, None] * wp1[d].astype(f32) + S[:, :d] @ mo
                     + S[:, d:] @ mi + deg[:, None] * bdeg + bp1.astype(f32))
            else:
                phio = S[:, :d] @ w2o.astype(f32) + deg[:, None] * b2o.astype(f32)
                phii = S[:, d:] @ w2i.astype(f32) + deg[:, None] * b2i.astype(f32)
                xn = np.hstack((h, cc[:, None], phio, phii))
                u = xn @ wp1.astype(f32) + bp1.astype(f32)
            u = np.maximum(u, f32(0))
            h = h + f32(model.alpha) * (u @ wp2.astype(f32) + bp2.astype(f32))
        dw1, db1, dw2, db2 = model.layers[-1]["dec"]
        o = np.maximum(h @ dw1.astype(f32) + db1.astype(f32), f32(0)) @ dw2.astype(f32) + db2.astype(f32)
        outs.append(o[:, 0].astype(np.float64))
    return np.concatenate(outs)


def main():
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", "A.npz")))
    a, _, coords, subs = problem_from(g)
    graphs = [orc.local_graph(a, s, coords) for s in subs]
    r = g["r"]
    cs = [r[s] / np.linalg.norm(r[s]) for s in subs]
    models = {"random k10": orc.model_from_flat(10, 10, float(g["m1010_alpha"]), 1, g["m1010_flat"]),
              "desk k10": orc.load_model(os.path.join(ROOT, "tests", "golden", "desk_k10_d10.dss"))}
    for name, m in models.items():
        ref = orc.forward(m, graphs, cs)
        for fw, fg in [(False, False), (True, False), (True, True)]:
            y = emulate(m, graphs, cs, fw, fg)
            print(f"{name:12s} fold_w2={fw!s:5s} fold_geo={fg!s:5s} rel-L2 {np.linalg.norm(y - ref) / np.linalg.norm(ref):.2e}")


if __name__ == "__main__":
    main()
