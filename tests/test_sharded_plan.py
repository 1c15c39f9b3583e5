"""CPU tests of the sharded solve's host logic: subdomain
grouping, ownership, halo and prolongation-term routing — checked against the
single-process definitions of the reference's operator (hybrid.py:117,133-135:
z_j = sum over subdomains i containing j, ascending i), with real gloo
collectives between world_size-2 (and 3) process groups on 127.0.0.1."""
import os
import socket

import numpy as np
import pytest

from conftest import load_golden, problem_from


def _problem(name="A.npz"):
    import paper_2402_08296_b200 as ddm

    g = load_golden(name)
    a, b, coords, subs = problem_from(g)
    dec = ddm.finish_decomposition(subs, g["owner"], int(g["overlap"]))
    return a, b, coords, dec


def _transpose_lists(dec):
    """Per DOF: [(subdomain, index within subdomain)] ascending subdomain."""
    out = [[] for _ in range(dec.n_dofs)]
    for i, s in enumerate(dec.subdomains):
        for k, j in enumerate(s):
            out[j].append((i, k))
    return out


@pytest.mark.parametrize("n_ranks", [1, 2, 3, 5])
def test_plans_partition_dofs_and_cover_terms(n_ranks):
    from paper_2402_08296_b200.sharded import group_subdomains, plan_shards

    a, _b, coords, dec = _problem()
    groups = group_subdomains(dec, coords, n_ranks)
    assert sorted(set(groups.tolist())) == list(range(n_ranks))
    plans = plan_shards(a, coords, dec, n_ranks, groups)
    owned = np.concatenate([p.owned for p in plans])
    assert np.array_equal(np.sort(owned), np.arange(dec.n_dofs))
    tl = _transpose_lists(dec)
    for p in plans:
        assert np.all(np.diff(p.local) > 0)
        assert np.array_equal(p.local[p.own_pos], p.owned)
        # owned rows of A are complete in the local column set
        rows = a[p.owned]
        assert rows.nnz == p.a_loc[p.own_pos].nnz
        # entries of the transpose map: same count and subdomains as the global one
        for t, j in enumerate(p.owned):
            ent = p.tent[p.tptr[t]:p.tptr[t + 1]]
            assert [int(s) for s in ent[:, 1]] == [i for i, _ in tl[j]]
        # own subdomains in local numbering keep the ascending global order
        for i, sl in zip(p.own_subs, p.subs_loc):
            assert np.array_equal(p.local[sl], dec.subdomains[i])
        assert p.pou_own.shape == p.owned.shape


@pytest.mark.parametrize("n_ranks", [2, 3, 5])
def test_one_sided_put_layout_routes_every_value(n_ranks):
    """The peer-memory puts (PeerArena, sharded.put_layout) simulated on host
    arrays: every ghost of every rank receives its owner's value, every remote
    prolongation term lands where the owner's transpose map reads it, and the
    all-gather slots name each subdomain's (R0 r)_i / s_i."""
    from paper_2402_08296_b200.sharded import gather_slots, plan_shards, put_layout

    a, _b, coords, dec = _problem()
    plans = plan_shards(a, coords, dec, n_ranks)
    x = np.random.default_rng(0).standard_normal(dec.n_dofs)
    lays = [put_layout(plans, g) for g in range(n_ranks)]
    halo_recv = [np.full(max(1, p.halo_recv_pos.size), np.nan) for p in plans]
    zloc_ext = [np.full(p.v_own + sum(p.term_recv_counts) + 1, np.nan) for p in plans]
    # batched local values: subdomain i's entry k gets 1000 * i + k
    zloc = []
    for p in plans:
        zloc.append(np.concatenate([1000.0 * i + np.arange(dec.subdomains[i].size)
                                    for i in p.own_subs]) if p.own_subs.size else np.zeros(0))
    for me, p in enumerate(plans):
        lay = lays[me]
        x_own = x[p.owned]
        for h in range(n_ranks):
            b0, b1 = lay["halo_send_off"][h], lay["halo_send_off"][h + 1]
            d0 = lay["halo_dst_off"][h]
            halo_recv[h][d0:d0 + b1 - b0] = x_own[p.halo_send_idx[b0:b1]]
            t0, t1 = lay["term_send_off"][h], lay["term_send_off"][h + 1]
            e0 = lay["term_dst_off"][h]
            zloc_ext[h][e0:e0 + t1 - t0] = zloc[me][p.term_send_pos[t0:t1]]
    for g, p in enumerate(plans):
        ext = np.full(p.n_loc, np.nan)
        ext[p.own_pos] = x[p.owned]
        ext[p.halo_recv_pos] = halo_recv[g][:p.halo_recv_pos.size]
        assert np.array_equal(ext, x[p.local])
        zloc_ext[g][:p.v_own] = zloc[g]
        for t, j in enumerate(p.owned):
            for pos, i in p.tent[p.tptr[t]:p.tptr[t + 1]]:
                k = int(np.searchsorted(dec.subdomains[i], j))
                assert zloc_ext[g][pos] == 1000.0 * i + k
        i_r0r, i_sc = gather_slots(p)
        ks = p.k_slots
        for i in range(dec.n_subdomains):
            owner = int(i_r0r[i] // (2 * ks))
            assert i in plans[owner].own_subs
            row = int(np.flatnonzero(plans[owner].own_subs == i)[0])
            assert i_r0r[i] == owner * 2 * ks + row and i_sc[i] == i_r0r[i] + ks


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_08296_b200.sharded import Comm, plan_shards

        a, _b, coords, dec = _problem()
        plans = plan_shards(a, coords, dec, world)
        p = plans[rank]
        comm = Comm()
        rng = np.random.default_rng(7)
        x = rng.standard_normal(dec.n_dofs)
        # halo: owned values -> ghost copies must reproduce x on the local set
        own = torch.tensor(x[p.owned])
        send = own[torch.as_tensor(p.halo_send_idx, dtype=torch.long)]
        recv = torch.zeros(int(sum(p.halo_recv_counts)), dtype=torch.float64)
        comm.alltoallv(recv, send, p.halo_recv_counts, p.halo_send_counts)
        ext = np.full(p.n_loc, np.nan)
        ext[p.own_pos] = own.numpy()
        ext[p.halo_recv_pos] = recv.numpy()
        halo_ok = bool(np.array_equal(ext, x[p.local]))
        # prolongation terms: code every (subdomain, node) entry, route, and check the
        # owner sees exactly the global (subdomain, node) list of each owned DOF in order
        sizes = [s.size for s in dec.subdomains]
        zloc = np.concatenate([1000.0 * i + np.arange(sizes[i]) for i in p.own_subs]) \
            if p.own_subs.size else np.zeros(0)
        tsend = torch.tensor(zloc[p.term_send_pos] if zloc.size else np.zeros(0))
        trecv = torch.zeros(int(sum(p.term_recv_counts)), dtype=torch.float64)
        comm.alltoallv(trecv, tsend, p.term_recv_counts, p.term_send_counts)
        zext = np.concatenate([zloc, trecv.numpy()])
        tl = _transpose_lists(dec)
        terms_ok = True
        for t, j in enumerate(p.owned):
            ent = p.tent[p.tptr[t]:p.tptr[t + 1]]
            got = [zext[pos] for pos in ent[:, 0]]
            want = [1000.0 * i + k for i, k in tl[j]]
            terms_ok &= got == want
        # all-gather of per-subdomain values through the slot map
        ks = p.k_slots
        gin = torch.zeros(ks, dtype=torch.float64)
        gin[: p.own_subs.size] = torch.tensor(p.own_subs, dtype=torch.float64) * 3.0
        gout = torch.zeros(ks * world, dtype=torch.float64)
        comm.allgather(gout, gin)
        full = gout.numpy()[p.sub_slot]
        slots_ok = bool(np.array_equal(full, 3.0 * np.arange(dec.n_subdomains)))
        t = torch.tensor([float(rank + 1)])
        comm.allreduce_(t)
        red_ok = float(t.item()) == world * (world + 1) / 2
        q.put((rank, halo_ok, bool(terms_ok), slots_ok, red_ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchanges_route_every_value(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, *oks in sorted(res):
        assert all(oks), (rank, oks)
