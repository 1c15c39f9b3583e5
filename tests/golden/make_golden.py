"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

This script imports the reference package read-only from
/root/reference/pkg/src (it exists only in the build container, never on the
GPU box) and records its inputs and outputs as compressed .npz files.  The
fixtures pin both the CPU oracle (oracle/ddm_oracle.py) and the CUDA path.

    python tests/golden/make_golden.py            # everything
    python tests/golden/make_golden.py small A    # selected fixtures

Fixtures
--------
small.npz   conftest `small_problem` (pkg/tests/conftest.py:64-70):
            build_problem(21, ProblemConfig(500, 0.15, 100, 2)); models
            init_model(3,4,seed=0) and init_model(2,3,seed=4); apply_ddm_gnn
            outputs (hybrid.py:112-136) for 5 residuals; templates
            (hybrid.py:36-46); CG history (sparse.py:130-132).
A.npz       BASELINE config A: generate_blob_mesh(0, 5000, 0.2), coeffs seed
            (0,1), partition(A, 1000, 0), overlap 2; model
            init_model(10,10,seed=1); apply outputs for r=default_rng(0);
            CG to 1e-6; with the pinned desk weights (desk_k10_d10.dss, if
            present) the PCG-DDM-GNN history to 1e-6.
heldout.npz held-out acceptance problems (test_acceptance.py:36,38,170-191),
            seeds 500-504 with the desk weights: PCG-DDM-GNN histories.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import ddmgnn as dg  # noqa: E402
from ddmgnn.dataset import ProblemConfig, build_problem, sample_coeffs  # noqa: E402
from ddmgnn.dss import _param_arrays, init_model, load_model  # noqa: E402
from ddmgnn.hybrid import apply_ddm_gnn, build_ddm_gnn  # noqa: E402
from ddmgnn.sparse import cg, pcg  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DESK = os.path.join(HERE, "desk_k10_d10.dss")


def flat(model):
    return np.concatenate([a.ravel() for a in _param_arrays(model)])


def problem_arrays(prefix, a, b, coords, dec):
    subs = dec.subdomains
    return {
        f"{prefix}indptr": a.indptr.astype(np.int64),
        f"{prefix}indices": a.indices.astype(np.int32),
        f"{prefix}data": a.data,
        f"{prefix}b": b,
        f"{prefix}coords": coords,
        f"{prefix}sub_ptr": np.concatenate(([0], np.cumsum([s.size for s in subs]))).astype(np.int64),
        f"{prefix}sub_idx": np.concatenate(subs).astype(np.int64),
        f"{prefix}owner": dec.base_owner.astype(np.int64),
        f"{prefix}overlap": np.int64(dec.overlap),
    }


def one_level(p, r):
    """hybrid.py:112-136 without the coarse term of :117 (SURVEY.md finding 2)."""
    return apply_ddm_gnn(p, r) - (p.dec.r0.T @ p.coarse_factorization.solve(p.dec.r0 @ r))


def local_only(p, r):
    """Exact one-level sum in the reference's gluing order, from a fresh zero vector."""
    from ddmgnn.dss import forward

    z = np.zeros(p.dec.n_dofs)
    for i, idx in enumerate(p.dec.subdomains):
        r_i = r[idx]
        s = float(np.linalg.norm(r_i))
        if s == 0.0:
            continue
        z[idx] += s * forward(p.model, p.templates[i].with_residual(r_i / s, s)).final_output
    return z


def make_small():
    prob = build_problem(21, ProblemConfig(target_nodes=500, perturbation=0.15,
                                           subdomain_size=100, overlap=2))
    a, b, coords, dec = prob.system.a, prob.system.b, prob.coords, prob.dec
    out = problem_arrays("", a, b, coords, dec)
    rng = np.random.default_rng(0)
    rs = rng.standard_normal((5, a.shape[0]))
    out["r"] = rs
    for tag, (kb, d, seed) in {"m340": (3, 4, 0), "m234": (2, 3, 4)}.items():
        model = init_model(kb, d, seed=seed)
        p = build_ddm_gnn(a, coords, dec, model)
        out[f"{tag}_flat"] = flat(model)
        out[f"{tag}_meta"] = np.array([kb, d, seed], dtype=np.int64)
        out[f"{tag}_alpha"] = np.float64(model.alpha)
        out[f"{tag}_z_two"] = np.stack([apply_ddm_gnn(p, r) for r in rs])
        out[f"{tag}_z_loc"] = np.stack([local_only(p, r) for r in rs])
        if tag == "m340":
            t = p.templates
            out["tpl_counts"] = np.array([g.edges.shape[0] for g in t], dtype=np.int64)
            out["tpl_edges"] = np.vstack([g.edges for g in t]).astype(np.int64)
            out["tpl_edge_vec"] = np.vstack([g.edge_vec for g in t])
            out["tpl_edge_len"] = np.concatenate([g.edge_len for g in t])
            out["coarse"] = dg.asm.coarse_matrix(a, dec)
            out["pou"] = np.concatenate(dec.pou_weights)
    _, rep = cg(a, b, 1e-8, 500)
    out["cg_hist"] = np.array(rep.residual_history)
    out["cg_iters"] = np.int64(rep.iterations)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print("small: n", a.shape[0], "K", dec.n_subdomains, "cg", rep.iterations)


def build_cfg(seed, target, pert, ns, overlap):
    mesh = dg.generate_blob_mesh(seed, target, pert)
    coeffs = sample_coeffs(np.random.default_rng((seed, 1)))
    system = dg.assemble(mesh, coeffs)
    owner = dg.partition(system.a, ns, seed)
    dec = dg.add_overlap(owner, system.a, overlap)
    return system.a, system.b, mesh.coords[system.node_of_interior], dec


def make_a():
    a, b, coords, dec = build_cfg(0, 5000, 0.2, 1000, 2)
    out = problem_arrays("", a, b, coords, dec)
    model = init_model(10, 10, seed=1)
    p = build_ddm_gnn(a, coords, dec, model)
    r = np.random.default_rng(0).standard_normal(a.shape[0])
    out["r"] = r
    out["m1010_flat"] = flat(model)
    out["m1010_alpha"] = np.float64(model.alpha)
    out["m1010_z_two"] = apply_ddm_gnn(p, r)
    out["m1010_z_loc"] = local_only(p, r)
    _, rep = cg(a, b, 1e-6, 5000)
    out["cg_hist"] = np.array(rep.residual_history)
    if os.path.exists(DESK):
        desk = load_model(DESK)
        pd = build_ddm_gnn(a, coords, dec, desk)
        out["desk_z_two"] = apply_ddm_gnn(pd, r)
        out["desk_z_loc"] = local_only(pd, r)
        _, rep2 = pcg(a, b, pd, 1e-6, 500)
        out["desk_pcg_hist"] = np.array(rep2.residual_history)
        out["desk_pcg_converged"] = np.int64(rep2.converged)
        print("A desk pcg", rep2.iterations, rep2.converged)
    np.savez_compressed(os.path.join(HERE, "A.npz"), **out)
    print("A: n", a.shape[0], "K", dec.n_subdomains, "cg", rep.iterations)


def make_heldout():
    if not os.path.exists(DESK):
        print("heldout: desk weights missing, skipped")
        return
    desk = load_model(DESK)
    out = {}
    for j, seed in enumerate(range(500, 505)):
        prob = build_problem(seed, ProblemConfig(600, 0.2, 110, 2))
        a, b, coords, dec = prob.system.a, prob.system.b, prob.coords, prob.dec
        out.update(problem_arrays(f"p{j}_", a, b, coords, dec))
        p = build_ddm_gnn(a, coords, dec, desk)
        _, rep = pcg(a, b, p, 1e-6, 500)
        out[f"p{j}_hist"] = np.array(rep.residual_history)
        r = np.random.default_rng(seed).standard_normal(a.shape[0])
        out[f"p{j}_r"] = r
        out[f"p{j}_z_two"] = apply_ddm_gnn(p, r)
        out[f"p{j}_z_loc"] = local_only(p, r)
        print("heldout seed", seed, "n", a.shape[0], "iters", rep.iterations)
    np.savez_compressed(os.path.join(HERE, "heldout.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "A", "heldout"]
    if "small" in which:
        make_small()
    if "A" in which:
        make_a()
    if "heldout" in which:
        make_heldout()
