"""Sharded DDM-GNN PCG: one process per GPU.

The reference solves on one CPU process (pkg/src/ddmgnn/sparse.py:76-127 with
the operator of hybrid.py:112-136).  Here the subdomains are split into G
spatially coherent groups (recursive coordinate bisection of the subdomain
centroids, weighted by subdomain size); rank g owns

* its group's subdomains (local GNN solves, CUDA kernels of csrc/gnn_impl.cuh),
* the DOFs whose base owner (decomp.py:29-44 ``base_owner``) lies in the group:
  the rows of A and the entries of every Krylov vector.

Its local context holds the group's subdomains over the rank's local DOF set
(owned DOFs + ghosts, numbered in ascending global order so each subdomain's
local graph, restriction and GNN arithmetic are exactly the single-GPU ones).
Per preconditioner apply (hybrid.py:112-136):

1. halo exchange of r (owned copies -> ghosts);
2. fused restriction + GNN over the own subdomains (one launch);
3. all-gather of the per-subdomain (R0 r)_i and s_i, coarse y = (R0 A R0^T)^-1 R0 r
   (replicated dense GEMV, hybrid.py:117);
4. reverse exchange of the individual prolongation terms s_i sol_i[j] for owned
   DOFs j of other ranks; the owner glues them in ascending subdomain order
   (hybrid.py:133-135), so z is bit-identical to the single-GPU apply.

The Krylov loop (sparse.py:76-127) all-reduces <p, Ap>, ||r||^2 and <r, z> and
exchanges the width-1 halo of p before the SpMV.  Collectives go through
torch.distributed: NCCL on device buffers, or gloo with host staging (used to
run two ranks on one GPU in the tests).  Everything per-iteration and
per-apply is a CUDA kernel of libddmgnn_b200.so; there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .asm import coarse_inverse, coarse_matrix
from .decomp import Decomposition
from .dss import DssModel, flat_params
from .sparse import SolveReport

__all__ = ["group_subdomains", "ShardPlan", "plan_shards", "Comm", "PeerExchange", "ShardedDdmGnn"]


# ---------------------------------------------------------------------------- planning


def group_subdomains(dec: Decomposition, coords: np.ndarray, n_groups: int) -> np.ndarray:
    """Group id of every subdomain: recursive coordinate bisection of the
    subdomain centroids, splitting the total subdomain size in proportion to the
    number of groups on each side (spatially coherent shards, small halos)."""
    k = dec.n_subdomains
    if n_groups < 1:
        raise ValueError("n_groups must be >= 1")
    if n_groups > k:
        raise ValueError(f"cannot split {k} subdomains into {n_groups} groups")
    sizes = np.array([s.size for s in dec.subdomains], dtype=np.float64)
    cen = np.array([coords[s].mean(axis=0) for s in dec.subdomains])
    out = np.zeros(k, dtype=np.int64)

    def split(ids, g0, ng):
        if ng == 1:
            out[ids] = g0
            return
        left = ng // 2
        ext = cen[ids].max(axis=0) - cen[ids].min(axis=0)
        axis = int(np.argmax(ext))
        order = ids[np.lexsort((ids, cen[ids, axis]))]
        cum = np.cumsum(sizes[order])
        cut = int(np.searchsorted(cum, cum[-1] * left / ng))
        cut = min(max(cut, left), order.size - (ng - left))  # every group non-empty
        split(order[:cut], g0, left)
        split(order[cut:], g0 + left, ng - left)

    split(np.arange(k), 0, n_groups)
    return out


@dataclass
class ShardPlan:
    """Everything rank ``rank`` needs (all index arrays int32 unless noted)."""

    rank: int
    n_ranks: int
    own_subs: np.ndarray      # int64, global subdomain ids, ascending
    owned: np.ndarray         # int64, global DOFs owned, ascending        (n_own)
    local: np.ndarray         # int64, global DOFs of the local set, ascending (n_loc)
    own_pos: np.ndarray       # positions of owned DOFs in the local set   (n_own)
    a_loc: sp.csr_matrix      # A[local][:, local]
    subs_loc: list            # own subdomains in local numbering (ascending)
    halo_send_idx: np.ndarray  # indices into the owned vector, grouped by destination
    halo_send_counts: list
    halo_recv_pos: np.ndarray  # positions in the local set, grouped by source
    halo_recv_counts: list
    term_send_pos: np.ndarray  # batched local positions of sent prolongation terms
    term_send_counts: list
    term_recv_counts: list
    tptr: np.ndarray          # (n_own + 1) transpose map over owned DOFs
    tent: np.ndarray          # (entries, 2): (position in zloc_ext, global subdomain)
    pou_own: np.ndarray       # float64 1/multiplicity of owned DOFs
    pou_loc: np.ndarray       # float64 1/multiplicity (global decomposition) of the local set
    sub_slot: np.ndarray      # (K,) slot of subdomain i in the all-gathered per-rank arrays
    k_slots: int              # per-rank slot count of the all-gather (max group size)
    v_own: int                # batched nodes of the own subdomains

    @property
    def n_own(self) -> int:
        return int(self.owned.size)

    @property
    def n_loc(self) -> int:
        return int(self.local.size)


def plan_shards(a: sp.csr_matrix, coords: np.ndarray, dec: Decomposition, n_ranks: int,
                groups: np.ndarray | None = None) -> list:
    """Deterministic plans for all ranks (every rank computes the same list)."""
    a = sp.csr_matrix(a)
    n, k = dec.n_dofs, dec.n_subdomains
    if groups is None:
        groups = group_subdomains(dec, coords, n_ranks)
    groups = np.asarray(groups, dtype=np.int64)
    subs = dec.subdomains
    sizes = np.array([s.size for s in subs], dtype=np.int64)
    owner_rank = groups[np.asarray(dec.base_owner, dtype=np.int64)]
    # batched local position of every (subdomain, node) entry on its group's rank
    lsub_ptr = np.zeros(k, dtype=np.int64)
    k_slot = np.zeros(k, dtype=np.int64)
    for g in range(n_ranks):
        ids = np.flatnonzero(groups == g)
        lsub_ptr[ids] = np.concatenate(([0], np.cumsum(sizes[ids])[:-1])) if ids.size else ids
        k_slot[ids] = np.arange(ids.size)
    k_slots = int(max(1, max(np.count_nonzero(groups == g) for g in range(n_ranks))))
    ent_sub = np.repeat(np.arange(k), sizes)
    ent_dof = np.concatenate(subs).astype(np.int64)
    ent_in = np.arange(ent_dof.size) - np.repeat(np.cumsum(sizes) - sizes, sizes)
    ent_lpos = lsub_ptr[ent_sub] + ent_in
    ent_rank = groups[ent_sub]
    order = np.argsort(ent_dof, kind="stable")  # by DOF, ascending subdomain within
    t_dof, t_sub, t_lpos, t_rank = ent_dof[order], ent_sub[order], ent_lpos[order], ent_rank[order]
    t_owner = owner_rank[t_dof]
    multiplicity = np.bincount(ent_dof, minlength=n).astype(np.float64)

    owned_all = [np.flatnonzero(owner_rank == g) for g in range(n_ranks)]
    plans = []
    locals_ = []
    for g in range(n_ranks):
        own_subs = np.flatnonzero(groups == g)
        owned = owned_all[g]
        rows = a[owned]
        parts = [owned, rows.indices.astype(np.int64)] + [subs[i] for i in own_subs]
        locals_.append(np.unique(np.concatenate(parts)))
    for g in range(n_ranks):
        own_subs = np.flatnonzero(groups == g)
        owned, local = owned_all[g], locals_[g]
        loc_of = np.full(n, -1, dtype=np.int64)
        loc_of[local] = np.arange(local.size)
        a_loc = a[local][:, local].tocsr()
        a_loc.sort_indices()
        subs_loc = [loc_of[subs[i]] for i in own_subs]
        # halo: ghosts of g grouped by owner rank (ascending global DOF within)
        ghosts = local[owner_rank[local] != g]
        g_owner = owner_rank[ghosts]
        recv_pos, recv_counts = [], []
        for h in range(n_ranks):
            gh = ghosts[g_owner == h]
            recv_pos.append(loc_of[gh])
            recv_counts.append(int(gh.size))
        send_idx, send_counts = [], []
        for h in range(n_ranks):
            lh = locals_[h]
            need = lh[owner_rank[lh] == g] if h != g else lh[:0]
            send_idx.append(np.searchsorted(owned, need))
            send_counts.append(int(need.size))
        # prolongation terms: entries whose DOF g owns, split local / remote by source
        sel = t_owner == g
        e_dof, e_sub, e_lpos, e_rank = t_dof[sel], t_sub[sel], t_lpos[sel], t_rank[sel]
        v_own = int(sizes[own_subs].sum())
        ext_pos = np.empty(e_dof.size, dtype=np.int64)
        is_loc = e_rank == g
        ext_pos[is_loc] = e_lpos[is_loc]
        term_recv_counts, off = [], v_own
        for h in range(n_ranks):
            m = e_rank == h
            cnt = int(np.count_nonzero(m)) if h != g else 0
            if h != g:
                ext_pos[m] = off + np.arange(cnt)
            term_recv_counts.append(cnt)
            off += cnt
        term_send_pos, term_send_counts = [], []
        for h in range(n_ranks):
            if h == g:
                term_send_pos.append(np.zeros(0, dtype=np.int64))
                term_send_counts.append(0)
                continue
            m = (t_owner == h) & (t_rank == g)
            term_send_pos.append(t_lpos[m])
            term_send_counts.append(int(np.count_nonzero(m)))
        tptr = np.zeros(owned.size + 1, dtype=np.int64)
        o_index = np.searchsorted(owned, e_dof)
        np.add.at(tptr, o_index + 1, 1)
        tptr = np.cumsum(tptr)
        tent = np.column_stack((ext_pos, e_sub))
        plans.append(ShardPlan(
            rank=g, n_ranks=n_ranks, own_subs=own_subs, owned=owned, local=local,
            own_pos=loc_of[owned].astype(np.int32), a_loc=a_loc, subs_loc=subs_loc,
            halo_send_idx=np.concatenate(send_idx).astype(np.int32),
            halo_send_counts=send_counts,
            halo_recv_pos=np.concatenate(recv_pos).astype(np.int32), halo_recv_counts=recv_counts,
            term_send_pos=np.concatenate(term_send_pos).astype(np.int32),
            term_send_counts=term_send_counts, term_recv_counts=term_recv_counts,
            tptr=tptr.astype(np.int32), tent=tent.astype(np.int32),
            pou_own=1.0 / multiplicity[owned], pou_loc=1.0 / multiplicity[local],
            sub_slot=(groups * k_slots + k_slot).astype(np.int32), k_slots=k_slots,
            v_own=v_own))
    return plans


# ---------------------------------------------------------------------------- collectives


class Comm:
    """torch.distributed collectives on CUDA tensors: NCCL directly, gloo through
    host staging (two ranks sharing one GPU in the tests).  World size 1 = no-ops."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self._dist = dist
        self.group = group
        self.active = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.active else 0
        self.size = dist.get_world_size(group) if self.active else 1
        self.nccl = self.active and dist.get_backend(group) == "nccl"

    def allreduce_(self, t):
        if self.size == 1:
            return t
        if self.nccl:
            self._dist.all_reduce(t, group=self.group)
        else:
            c = t.cpu()
            self._dist.all_reduce(c, group=self.group)
            t.copy_(c)
        return t

    def allgather(self, out, inp):
        """out (size * inp.numel()) = concatenation of every rank's inp."""
        if self.size == 1:
            out.copy_(inp)
            return out
        if self.nccl:
            self._dist.all_gather_into_tensor(out, inp, group=self.group)
        else:
            import torch

            parts = [torch.empty_like(inp, device="cpu") for _ in range(self.size)]
            self._dist.all_gather(parts, inp.cpu(), group=self.group)
            out.copy_(torch.cat(parts))
        return out

    def barrier(self):
        if self.size > 1:
            self._dist.barrier(group=self.group)

    def alltoallv(self, recv, send, recv_counts, send_counts):
        if self.size == 1:
            return recv
        if self.nccl:
            self._dist.all_to_all_single(recv, send, recv_counts, send_counts, group=self.group)
        else:
            rc = recv.cpu()
            self._dist.all_to_all_single(rc, send.cpu(), recv_counts, send_counts,
                                         group=self.group)
            recv.copy_(rc)
        return recv


class PeerExchange:
    """One-sided exchange over peer memory: every rank maps the other ranks'
    receive buffers (CUDA IPC handles, all-gathered once) and its gather kernel
    writes its segment straight into them — over NVLink between the GPUs of one box
    (P2P), or within one device when several ranks share a GPU (the tests).  The
    receive layout is the all-to-all one (segments ordered by source rank), so a
    plan serves both exchange modes.  Ordering: a barrier before the puts (the
    peers finished reading the previous contents) and after them (the data landed)."""

    def __init__(self, comm: "Comm", recv_buf, recv_counts, send_counts):
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor

        self.comm = comm
        self.send_counts = list(send_counts)
        me, size = comm.rank, comm.size
        everyone = [None] * size
        dist.all_gather_object(everyone, (list(recv_counts), reduce_tensor(recv_buf)),
                               group=comm.group)
        self.peers = {}
        for h, (counts, (fn, args)) in enumerate(everyone):
            if h == me or self.send_counts[h] == 0:
                continue
            buf = fn(*args)  # the peer's receive buffer, mapped into this process
            self.peers[h] = (buf, int(sum(counts[:me])))
        self._keep = recv_buf

    def put(self, lib, src_ptr: int, idx, stream: int):
        """Send segment h of the gather src[idx] into peer h's receive buffer."""
        self._sync()
        off = 0
        for h, cnt in enumerate(self.send_counts):
            if cnt and h in self.peers:
                buf, dst = self.peers[h]
                _lib.check(lib.ddmgnn_gather(src_ptr, idx.data_ptr() + 4 * off, cnt,
                                             buf.data_ptr() + 8 * dst, stream))
            off += cnt
        self._sync()

    def _sync(self):
        import torch

        torch.cuda.current_stream().synchronize()
        self.comm.barrier()


# ---------------------------------------------------------------------------- rank object


class ShardedDdmGnn:
    """Rank-local part of the sharded preconditioner + PCG."""

    def __init__(self, a: sp.csr_matrix, coords: np.ndarray, dec: Decomposition,
                 model: DssModel, level: str = "two", device: int | None = None, group=None,
                 plans: list | None = None, batch_nodes_cap: int = 100_000,
                 exchange: str = "collective"):
        import torch

        if level not in ("one", "two"):
            raise ValueError(f"level must be 'one' or 'two', got {level!r}")
        self.comm = Comm(group)
        a = sp.csr_matrix(a)
        if not a.has_sorted_indices:
            a = a.copy()
            a.sort_indices()
        coords = np.asarray(coords, dtype=float)
        if coords.shape != (dec.n_dofs, 2):
            raise ValueError(f"expected coords of shape ({dec.n_dofs}, 2)")
        if plans is None:
            plans = plan_shards(a, coords, dec, self.comm.size)
        if len(plans) != self.comm.size:
            raise ValueError("one shard plan per rank expected")
        self.plan = plan = plans[self.comm.rank]
        self.n = dec.n_dofs
        self.k = dec.n_subdomains
        self.level = level
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else int(device))
        dev = self.device
        ctx = _lib.Context(dev.index)
        ctx.set_matrix(plan.a_loc)
        ctx.set_geometry(coords[plan.local])
        ctx.set_decomposition(plan.subs_loc)
        ctx.set_batch_cap(batch_nodes_cap)
        ctx.build()
        ctx.set_pou(plan.pou_loc)  # R0 r uses the global multiplicities (decomp.py:184-190)
        ctx.set_model(model.k_bar, model.d, model.alpha, flat_params(model))
        self.ctx = ctx
        self.model = model
        self._lib = _lib.load()

        def it(x):
            return torch.as_tensor(np.ascontiguousarray(x, dtype=np.int32), device=dev)

        def ft(x):
            return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device=dev)

        f64 = dict(dtype=torch.float64, device=dev)
        self.own_pos = it(plan.own_pos)
        self.halo_send_idx, self.halo_recv_pos = it(plan.halo_send_idx), it(plan.halo_recv_pos)
        self.term_send_pos = it(plan.term_send_pos)
        self.tptr, self.tent = it(plan.tptr), it(plan.tent.reshape(-1))
        self.pou_own = ft(plan.pou_own)
        self.sub_slot = it(plan.sub_slot)
        self.kinv = None
        if level == "two":
            cm = coarse_matrix(a, dec)
            self.kinv = ft(coarse_inverse(cm))
        n_own, n_loc = plan.n_own, plan.n_loc
        self.r_ext = torch.zeros(n_loc, **f64)
        self.p_ext = torch.zeros(n_loc, **f64)
        self.q_ext = torch.zeros(n_loc, **f64)
        self.halo_send = torch.zeros(max(1, plan.halo_send_idx.size), **f64)
        self.halo_recv = torch.zeros(max(1, plan.halo_recv_pos.size), **f64)
        self.term_send = torch.zeros(max(1, plan.term_send_pos.size), **f64)
        self.zloc_ext = torch.zeros(plan.v_own + sum(plan.term_recv_counts) + 1, **f64)
        ks = plan.k_slots
        self.gath_in = torch.zeros(2 * ks, **f64)
        self.gath_out = torch.zeros(2 * ks * self.comm.size, **f64)
        self.own_slot = it(np.arange(plan.own_subs.size))
        self.r0r_full = torch.zeros(self.k, **f64)
        self.scale_full = torch.zeros(self.k, **f64)
        self.y = torch.zeros(self.k, **f64)
        self.work = torch.zeros(1184, **f64)
        self.scal = torch.zeros(4, **f64)
        self._all_owned = [pl.owned for pl in plans]
        if exchange not in ("collective", "p2p"):
            raise ValueError(f"exchange must be 'collective' or 'p2p', got {exchange!r}")
        self.exchange = exchange
        self._p2p_halo = self._p2p_terms = None
        if exchange == "p2p" and self.comm.size > 1:
            self._p2p_halo = PeerExchange(self.comm, self.halo_recv, plan.halo_recv_counts,
                                          plan.halo_send_counts)
            self._p2p_terms = PeerExchange(self.comm, self.zloc_ext[plan.v_own:],
                                           plan.term_recv_counts, plan.term_send_counts)

    def launches_per_apply(self) -> int:
        """Kernels of libddmgnn_b200 launched by one apply_owned."""
        multi = self.comm.size > 1
        gnn = self.ctx.gnn_launches()
        return (1 + 2 * multi) + gnn + 4 + (self.kinv is not None) + multi + 1

    # -- helpers --------------------------------------------------------------------------
    def _stream(self):
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream or _lib.LEGACY_STREAM

    def _c(self, status):
        _lib.check(status)

    def _halo(self, own_vec, ext_vec):
        """ext_vec = local-set copy of the distributed vector own_vec (owned + ghosts)."""
        lib, s, p = self._lib, self._stream(), self.plan
        self._c(lib.ddmgnn_scatter(own_vec.data_ptr(), self.own_pos.data_ptr(), p.n_own,
                                   ext_vec.data_ptr(), s))
        if self.comm.size == 1:
            return ext_vec
        ns, nr = p.halo_send_idx.size, p.halo_recv_pos.size
        if self._p2p_halo is not None:
            self._p2p_halo.put(lib, own_vec.data_ptr(), self.halo_send_idx, s)
        else:
            self._c(lib.ddmgnn_gather(own_vec.data_ptr(), self.halo_send_idx.data_ptr(), ns,
                                      self.halo_send.data_ptr(), s))
            self.comm.alltoallv(self.halo_recv[:nr], self.halo_send[:ns], p.halo_recv_counts,
                                p.halo_send_counts)
        self._c(lib.ddmgnn_scatter(self.halo_recv.data_ptr(), self.halo_recv_pos.data_ptr(), nr,
                                   ext_vec.data_ptr(), self._stream()))
        return ext_vec

    def _dot(self, x, y, slot):
        self._c(self._lib.ddmgnn_dot(x.numel(), x.data_ptr(), y.data_ptr(), self.work.data_ptr(),
                                     self.scal[slot:].data_ptr(), self._stream()))

    # -- operator ---------------------------------------------------------------------------
    def apply_owned(self, r_own, z_own=None):
        """z = M r on this rank's owned DOFs (hybrid.py:112-136); collective."""
        import torch

        lib, p = self._lib, self.plan
        if z_own is None:
            z_own = torch.empty_like(r_own)
        self._halo(r_own, self.r_ext)
        s = self._stream()
        self.ctx.launch_gnn_only(self.r_ext.data_ptr(), s)
        zloc, scale, r0r = self.ctx.local_outputs()
        ko, ks = p.own_subs.size, p.k_slots
        # all-gather (R0 r)_i and s_i of the own subdomains; slot map -> global order
        self._c(lib.ddmgnn_gather(r0r, self.own_slot.data_ptr(), ko, self.gath_in.data_ptr(), s))
        self._c(lib.ddmgnn_gather(scale, self.own_slot.data_ptr(), ko,
                                  self.gath_in[ks:].data_ptr(), s))
        self.comm.allgather(self.gath_out, self.gath_in)
        g2 = self.gath_out.view(self.comm.size, 2, ks)
        r0r_all = g2[:, 0, :].reshape(-1).contiguous()
        sc_all = g2[:, 1, :].reshape(-1).contiguous()
        s = self._stream()
        self._c(lib.ddmgnn_gather(r0r_all.data_ptr(), self.sub_slot.data_ptr(), self.k,
                                  self.r0r_full.data_ptr(), s))
        self._c(lib.ddmgnn_gather(sc_all.data_ptr(), self.sub_slot.data_ptr(), self.k,
                                  self.scale_full.data_ptr(), s))
        if self.kinv is not None:
            self._c(lib.ddmgnn_dense_gemv(self.k, self.kinv.data_ptr(), self.r0r_full.data_ptr(),
                                          self.y.data_ptr(), s))
        # own terms + remote terms (owner glues in ascending subdomain order)
        self.zloc_ext[:p.v_own].copy_(_view_f64(zloc, p.v_own, self.device))
        if self._p2p_terms is not None:
            self._p2p_terms.put(lib, zloc, self.term_send_pos, s)
        elif self.comm.size > 1:
            ns = p.term_send_pos.size
            self._c(lib.ddmgnn_gather(zloc, self.term_send_pos.data_ptr(), ns,
                                      self.term_send.data_ptr(), s))
            nr = sum(p.term_recv_counts)
            self.comm.alltoallv(self.zloc_ext[p.v_own:p.v_own + nr], self.term_send[:ns],
                                p.term_recv_counts, p.term_send_counts)
        self._c(lib.ddmgnn_prolong(p.n_own, int(self.kinv is not None), self.tptr.data_ptr(),
                                   self.tent.data_ptr(), self.pou_own.data_ptr(),
                                   self.y.data_ptr(), self.scale_full.data_ptr(),
                                   self.zloc_ext.data_ptr(), z_own.data_ptr(), self._stream()))
        return z_own

    def owned_part(self, x_global):
        import torch

        return torch.as_tensor(np.ascontiguousarray(np.asarray(x_global)[self.plan.owned],
                                                    dtype=np.float64), device=self.device)

    def gather_global(self, x_own) -> np.ndarray:
        """Full vector on every rank (all-gather of the owned parts)."""
        import torch

        p = self.plan
        m = max(1, max(o.size for o in self._all_owned))
        buf = torch.zeros(m, dtype=torch.float64, device=self.device)
        buf[:p.n_own] = x_own
        out = torch.zeros(m * self.comm.size, dtype=torch.float64, device=self.device)
        self.comm.allgather(out, buf)
        full = np.zeros(self.n)
        o = out.view(self.comm.size, m).cpu().numpy()
        for g, owned in enumerate(self._all_owned):
            full[owned] = o[g, :owned.size]
        return full

    # -- Krylov -----------------------------------------------------------------------------
    def pcg(self, b_global, tol: float, max_iter: int, check_every: int = 8,
            flexible: bool = False):
        """Distributed PCG (sparse.py:76-127) with this preconditioner; collective.
        Returns (u_global, SolveReport) on every rank.  ``flexible=True``: the opt-in
        flexible CG (beta = <r, z - z_old> / rho), as ``sparse.pcg``.

        The recurrence's scalars live on the device (``st``, see ddmgnn_pcg_scalars):
        <p, Ap>, ||r||^2 and <r, z> are reduced into it in place by the all-reduces,
        alpha / beta / the stopping test are computed there, and the updates turn into
        no-ops once the solve has stopped — so the host only polls the status every
        ``check_every`` iterations instead of synchronising on every dot product."""
        import torch

        if tol <= 0:
            raise ValueError("tol must be positive")
        b = np.asarray(b_global, dtype=np.float64)
        if b.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got shape {b.shape}")
        lib, p = self._lib, self.plan
        n_own = p.n_own
        bo = self.owned_part(b)
        u = torch.zeros_like(bo)
        r = bo.clone()
        q = torch.empty_like(bo)
        max_iter = max(0, int(max_iter))  # sparse.py:105: no iteration for max_iter < 0
        st = torch.zeros(12, dtype=torch.float64, device=self.device)
        hist = torch.zeros(max_iter + 1, dtype=torch.float64, device=self.device)
        stream = self._stream
        self._dot(bo, bo, 0)
        nb = float(np.sqrt(self._allreduce_scalar(0)))
        if nb == 0.0:  # sparse.py:93-94
            return np.zeros(self.n), SolveReport(0, [0.0], True, 0.0, tol)
        # r0 = b, so history[0] = ||b|| / ||b|| = 1 exactly (sparse.py:96-99)
        if 1.0 < tol:
            return np.zeros(self.n), SolveReport(0, [1.0], True, 1.0, tol)
        z = self.apply_owned(r)
        self.ctx.apply_status(self._stream())  # non-finite model output -> reference error
        pv = z.clone()
        z_old = torch.empty_like(z) if flexible else None
        self._c(lib.ddmgnn_dot(n_own, r.data_ptr(), z.data_ptr(), self.work.data_ptr(),
                               st[0:].data_ptr(), stream()))
        self.comm.allreduce_(st[0:1])  # rho = <r0, z0>
        st[4], st[5], st[10] = nb, float(tol), float(max_iter)
        hist[0] = 1.0  # r0 = b
        status = 0.0
        for it in range(max_iter):
            self._halo(pv, self.p_ext)
            s = stream()
            self.ctx.spmv_device(self.p_ext.data_ptr(), self.q_ext.data_ptr(), s)
            self._c(lib.ddmgnn_gather(self.q_ext.data_ptr(), self.own_pos.data_ptr(), n_own,
                                      q.data_ptr(), s))
            self._c(lib.ddmgnn_dot(n_own, pv.data_ptr(), q.data_ptr(), self.work.data_ptr(),
                                   st[1:].data_ptr(), s))
            self.comm.allreduce_(st[1:2])
            s = stream()
            self._c(lib.ddmgnn_pcg_scalars(0, st.data_ptr(), hist.data_ptr(), s))
            self._c(lib.ddmgnn_axpy2_dev(n_own, st.data_ptr(), pv.data_ptr(), q.data_ptr(),
                                         u.data_ptr(), r.data_ptr(), self.work.data_ptr(),
                                         st[3:].data_ptr(), s))
            self.comm.allreduce_(st[3:4])
            self._c(lib.ddmgnn_pcg_scalars(1, st.data_ptr(), hist.data_ptr(), stream()))
            if (it + 1) % check_every == 0 or it + 1 == max_iter:
                # the GNN status word of the applies since the last check, then the
                # solve's own status (both are device-side words: one poll each)
                self.ctx.apply_status(stream())
                status = float(st[9].item())
                if status != 0.0:
                    break
            if flexible:
                z_old.copy_(z)
            self.apply_owned(r, z)
            self._c(lib.ddmgnn_dot(n_own, r.data_ptr(), z.data_ptr(), self.work.data_ptr(),
                                   st[6:].data_ptr(), stream()))
            if flexible:
                self._c(lib.ddmgnn_dot_diff(n_own, r.data_ptr(), z.data_ptr(), z_old.data_ptr(),
                                            self.work.data_ptr(), st[11:].data_ptr(), stream()))
                self.comm.allreduce_(st[11:12])
            self.comm.allreduce_(st[6:7])
            s = stream()
            self._c(lib.ddmgnn_pcg_scalars(3 if flexible else 2, st.data_ptr(), hist.data_ptr(), s))
            self._c(lib.ddmgnn_xpby_dev(n_own, z.data_ptr(), st.data_ptr(), pv.data_ptr(), s))
        sh = st.cpu().numpy()
        status, iters = int(sh[9]), int(sh[8])
        if status == 3:
            raise RuntimeError("matrix not SPD: <p, Ap> <= 0")
        if status == 4:
            raise RuntimeError(f"non-finite residual at iteration {iters}")
        history = hist[: iters + 1].cpu().numpy().tolist()
        return self.gather_global(u), SolveReport(iters, history, status == 1, history[-1], tol)

    def _allreduce_scalar(self, slot: int) -> float:
        t = self.scal[slot:slot + 1]
        self.comm.allreduce_(t)
        return float(t.item())


def _view_f64(ptr: int, n: int, device):
    """A torch view of a device buffer owned by the C library (no copy)."""
    import torch

    if n == 0:
        return torch.zeros(0, dtype=torch.float64, device=device)

    class _Cai:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_Cai(), device=device)
