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

__all__ = ["group_subdomains", "ShardPlan", "plan_shards", "put_layout", "gather_slots", "Comm",
           "PeerArena", "ShardedDdmGnn"]


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


def put_layout(plans: list, me: int) -> dict:
    """Offsets of rank ``me``'s one-sided puts (PeerArena): per destination h the
    segment [send_off[h], send_off[h+1]) of its send list lands at dst_off[h] of
    h's receive buffer — the all-to-all layout, segments ordered by source rank —
    and its own receive buffer holds source h's segment at [recv_off[h],
    recv_off[h+1]).  Terms land behind the receiver's own v_own local entries."""
    g = len(plans)
    p = plans[me]

    def cum(c):
        return np.concatenate(([0], np.cumsum(c))).astype(np.int64)

    return {
        "halo_send_off": cum(p.halo_send_counts), "halo_recv_off": cum(p.halo_recv_counts),
        "halo_dst_off": np.array([sum(plans[h].halo_recv_counts[:me]) for h in range(g)],
                                 dtype=np.int64),
        "term_send_off": cum(p.term_send_counts), "term_recv_off": cum(p.term_recv_counts),
        "term_dst_off": np.array([plans[h].v_own + sum(plans[h].term_recv_counts[:me])
                                  for h in range(g)], dtype=np.int64),
    }


def gather_slots(plan: ShardPlan) -> tuple:
    """Positions of (R0 r)_i and s_i of every subdomain i in the all-gathered
    [rank][2 k_slots] buffer (rank g's row = its own subdomains' r0r, then scale)."""
    ks = plan.k_slots
    rank, slot = plan.sub_slot // ks, plan.sub_slot % ks
    return rank * 2 * ks + slot, rank * 2 * ks + ks + slot


# Channels of the device-resident exchanges (one per call site; csrc/shard.cu).
CH_HALO_P, CH_HALO_R, CH_TERMS, CH_GATHER, CH_PQ, CH_RR, CH_RZ, CH_RZO = range(8)
_FLAG_WORDS = 256   # DDMGNN_PEER_FLAG_WORDS
_ERR_WORD = _FLAG_WORDS - 1
_SLOT = 16          # doubles per rank in an all-reduce staging area
_N_CHANNELS = 8


class PeerArena:
    """Peer-visible device buffers of one rank plus the mappings of every other
    rank's (CUDA IPC, opened once; NVLink between the GPUs of one box, the same
    device when several ranks share a GPU in the tests).  The exchanges on it
    (csrc/shard.cu ``ddmgnn_peer_*``) are one-sided puts ordered by device-side
    epochs and acknowledgements in the ranks' flag blocks: no host barrier, so a
    whole sharded PCG iteration is stream-ordered and can be captured in a CUDA
    graph.  ``sizes``: buffer name -> number of doubles."""

    def __init__(self, comm: "Comm", device: int, sizes: dict):
        import ctypes

        import torch.distributed as dist

        self.lib = lib = _lib.load()
        self.comm, self.device = comm, int(device)
        g, me = comm.size, comm.rank
        if g > _FLAG_MAX_RANKS:
            raise ValueError(f"peer exchange supports at most {_FLAG_MAX_RANKS} ranks")
        sizes = {"_flags": _FLAG_WORDS, "_slots": _N_CHANNELS * g * _SLOT, **sizes}
        offsets, total = {}, 0
        for name, n in sizes.items():
            offsets[name] = total
            total += (max(1, int(n)) + 31) // 32 * 32  # 256-byte aligned
        base = ctypes.c_void_p()
        _lib.check(lib.ddmgnn_peer_alloc(self.device, 8 * total, ctypes.byref(base)))
        self._own = base.value
        handle = ctypes.create_string_buffer(64)
        _lib.check(lib.ddmgnn_ipc_get(base, handle))
        everyone = [None] * g
        dist.all_gather_object(everyone, (handle.raw, offsets), group=comm.group)
        self._opened = []
        bases = []
        err = None
        for h, (hnd, _offs) in enumerate(everyone):
            if h == me:
                bases.append(self._own)
                continue
            ptr = ctypes.c_void_p()
            try:
                _lib.check(lib.ddmgnn_ipc_open(self.device, hnd, ctypes.byref(ptr)))
            except RuntimeError as exc:  # e.g. no peer access between these two GPUs
                err = f"rank {me} cannot map rank {h}'s buffers: {exc}"
                break
            self._opened.append(ptr.value)
            bases.append(ptr.value)
        # every rank must agree, or the ranks would run different exchange modes
        verdicts = [None] * g
        dist.all_gather_object(verdicts, err, group=comm.group)
        bad = [v for v in verdicts if v]
        if bad:
            self.close()
            raise RuntimeError("peer exchange unavailable: " + bad[0])
        self.g, self.me = g, me
        self.offsets = offsets
        self._arr = {}
        for name in sizes:
            self._arr[name] = (ctypes.c_void_p * g)(
                *[bases[h] + 8 * everyone[h][1][name] for h in range(g)])
        self.flags = self._arr["_flags"]
        self._slots = {c: (ctypes.c_void_p * g)(
            *[self._arr["_slots"][h] + 8 * c * g * _SLOT for h in range(g)])
            for c in range(_N_CHANNELS)}

    def ptr(self, name: str) -> int:
        """This rank's own buffer `name` (device pointer)."""
        return self._arr[name][self.me]

    def view(self, name: str, n: int, device):
        return _view_f64(self.ptr(name), n, device)

    @staticmethod
    def _i64(x):
        import ctypes

        a = np.ascontiguousarray(x, dtype=np.int64)
        return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))

    def put(self, chan, src_ptr, idx_ptr, send_off, dst_name, dst_off, stream):
        _so, so = self._i64(send_off)
        _do, do = self._i64(dst_off)
        _lib.check(self.lib.ddmgnn_peer_put(self.g, self.me, chan, self.flags, src_ptr, idx_ptr,
                                            so, self._arr[dst_name], do, stream))

    def wait(self, chan, recv_off, recv_ptr, pos_ptr, ext_ptr, ack, stream):
        _ro, ro = self._i64(recv_off)
        _lib.check(self.lib.ddmgnn_peer_wait(self.g, self.me, chan, self.flags, ro, recv_ptr,
                                             pos_ptr, ext_ptr, int(ack), stream))

    def ack(self, chan, recv_off, stream):
        _ro, ro = self._i64(recv_off)
        _lib.check(self.lib.ddmgnn_peer_ack(self.g, self.me, chan, self.flags, ro, stream))

    def allreduce_(self, t, chan, stream):
        """t (contiguous fp64 device tensor, <= 16 values) = sum over ranks, in place."""
        _lib.check(self.lib.ddmgnn_peer_allreduce(self.g, self.me, chan, self.flags,
                                                  self._slots[chan], t.data_ptr(), t.numel(),
                                                  stream))

    def allgather(self, out_name, in_ptr, k, chan, stream):
        _lib.check(self.lib.ddmgnn_peer_allgather(self.g, self.me, chan, self.flags,
                                                  self._arr[out_name], in_ptr, k, stream))

    def timed_out(self) -> bool:
        """A device-side wait gave up (a peer never arrived); synchronising read."""
        import torch

        v = _view_i64(self._own + 8 * _ERR_WORD, 1, torch.device("cuda", self.device))
        return bool(v.item() != 0)

    def close(self):
        for p in self._opened:
            self.lib.ddmgnn_ipc_close(p)
        self._opened = []
        if self._own:
            self.lib.ddmgnn_peer_free(self._own)
            self._own = 0


_FLAG_MAX_RANKS = 8  # DDMGNN_PEER_MAX


# ---------------------------------------------------------------------------- rank object


class ShardedDdmGnn:
    """Rank-local part of the sharded preconditioner + PCG.

    ``exchange="collective"``: halo / term exchanges and the all-gather / all-reduces
    through torch.distributed (NCCL on device buffers, gloo host-staged).
    ``exchange="p2p"``: everything through :class:`PeerArena` — one-sided puts into
    the peers' receive buffers and flag-ordered all-reduces, all on the solve
    stream, so ``pcg`` and ``capture_apply`` run from CUDA graphs with the host
    polling the device status only every few iterations."""

    def __init__(self, a: sp.csr_matrix, coords: np.ndarray, dec: Decomposition,
                 model: DssModel, level: str = "two", device: int | None = None, group=None,
                 plans: list | None = None, batch_nodes_cap: int = 100_000,
                 exchange: str = "collective"):
        import torch

        if level not in ("one", "two"):
            raise ValueError(f"level must be 'one' or 'two', got {level!r}")
        if exchange not in ("collective", "p2p"):
            raise ValueError(f"exchange must be 'collective' or 'p2p', got {exchange!r}")
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
        g, me = self.comm.size, self.comm.rank
        self.own_pos = it(plan.own_pos)
        self.halo_send_idx, self.halo_recv_pos = it(plan.halo_send_idx), it(plan.halo_recv_pos)
        self.term_send_pos = it(plan.term_send_pos)
        self.tptr, self.tent = it(plan.tptr), it(plan.tent.reshape(-1))
        self.pou_own = ft(plan.pou_own)
        # (R0 r)_i and s_i of subdomain i in the all-gathered [rank][2 ks] layout
        ks = plan.k_slots
        i_r0r, i_scale = gather_slots(plan)
        self.idx_r0r, self.idx_scale = it(i_r0r), it(i_scale)
        self.kinv = None
        if level == "two":
            cm = coarse_matrix(a, dec)
            self.kinv = ft(coarse_inverse(cm))
        n_own, n_loc = plan.n_own, plan.n_loc
        self.r_ext = torch.zeros(n_loc, **f64)
        self.p_ext = torch.zeros(n_loc, **f64)
        self.q_ext = torch.zeros(n_loc, **f64)
        self.halo_send = torch.zeros(max(1, plan.halo_send_idx.size), **f64)
        self.term_send = torch.zeros(max(1, plan.term_send_pos.size), **f64)
        n_hrecv = int(plan.halo_recv_pos.size)
        n_zext = plan.v_own + sum(plan.term_recv_counts) + 1
        self.gath_in = torch.zeros(2 * ks, **f64)
        self.own_slot = it(np.arange(plan.own_subs.size))
        self.r0r_full = torch.zeros(self.k, **f64)
        self.scale_full = torch.zeros(self.k, **f64)
        self.y = torch.zeros(self.k, **f64)
        self.work = torch.zeros(1184, **f64)
        self.scal = torch.zeros(4, **f64)
        self._all_owned = [pl.owned for pl in plans]
        self.exchange = exchange
        self.arena = None
        lay = put_layout(plans, me)
        self._halo_send_off, self._halo_recv_off = lay["halo_send_off"], lay["halo_recv_off"]
        self._term_send_off, self._term_recv_off = lay["term_send_off"], lay["term_recv_off"]
        self._halo_dst_off, self._term_dst_off = lay["halo_dst_off"], lay["term_dst_off"]
        if exchange == "p2p" and g > 1:
            self.arena = PeerArena(self.comm, dev.index, {
                "halo_p": max(1, n_hrecv), "halo_r": max(1, n_hrecv), "zloc_ext": n_zext,
                "gath_out": 2 * ks * g})
            self.halo_recv = {CH_HALO_P: self.arena.view("halo_p", max(1, n_hrecv), dev),
                              CH_HALO_R: self.arena.view("halo_r", max(1, n_hrecv), dev)}
            self.zloc_ext = self.arena.view("zloc_ext", n_zext, dev)
            self.gath_out = self.arena.view("gath_out", 2 * ks * g, dev)
        else:
            hr = torch.zeros(max(1, n_hrecv), **f64)
            self.halo_recv = {CH_HALO_P: hr, CH_HALO_R: hr}
            self.zloc_ext = torch.zeros(n_zext, **f64)
            self.gath_out = torch.zeros(2 * ks * g, **f64)

    def close(self):
        """Release the peer mappings (collective: every rank calls it)."""
        if self.arena is not None:
            import torch

            torch.cuda.synchronize(self.device)
            self.comm.barrier()
            self.arena.close()
            self.arena = None

    @property
    def device_ordered(self) -> bool:
        """Every exchange of an iteration is stream-ordered on the device (peer
        arena or a single rank), so it can be captured in a CUDA graph."""
        return self.arena is not None or self.comm.size == 1

    def launches_per_apply(self) -> int:
        """Kernels of libddmgnn_b200 launched by one apply_owned."""
        multi = self.comm.size > 1
        gnn = self.ctx.gnn_launches()
        halo = 1 + (3 if self.arena is not None else 2) * multi
        gather = 2 + (1 if self.arena is not None else 0) * multi + 2
        terms = (3 if self.arena is not None else 1) * multi
        return halo + gnn + gather + (self.kinv is not None) + terms + 1

    # -- helpers --------------------------------------------------------------------------
    def _stream(self):
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream or _lib.LEGACY_STREAM

    def _c(self, status):
        _lib.check(status)

    def _allreduce(self, t, chan):
        if self.arena is not None:
            self.arena.allreduce_(t, chan, self._stream())
        else:
            self.comm.allreduce_(t)

    def _halo(self, own_vec, ext_vec, chan):
        """ext_vec = local-set copy of the distributed vector own_vec (owned + ghosts)."""
        lib, s, p = self._lib, self._stream(), self.plan
        self._c(lib.ddmgnn_scatter(own_vec.data_ptr(), self.own_pos.data_ptr(), p.n_own,
                                   ext_vec.data_ptr(), s))
        if self.comm.size == 1:
            return ext_vec
        ns, nr = p.halo_send_idx.size, p.halo_recv_pos.size
        recv = self.halo_recv[chan]
        if self.arena is not None:
            self.arena.put(chan, own_vec.data_ptr(), self.halo_send_idx.data_ptr(),
                           self._halo_send_off, "halo_p" if chan == CH_HALO_P else "halo_r",
                           self._halo_dst_off, s)
            self.arena.wait(chan, self._halo_recv_off, recv.data_ptr(),
                            self.halo_recv_pos.data_ptr(), ext_vec.data_ptr(), 1, s)
            return ext_vec
        self._c(lib.ddmgnn_gather(own_vec.data_ptr(), self.halo_send_idx.data_ptr(), ns,
                                  self.halo_send.data_ptr(), s))
        self.comm.alltoallv(recv[:nr], self.halo_send[:ns], p.halo_recv_counts,
                            p.halo_send_counts)
        self._c(lib.ddmgnn_scatter(recv.data_ptr(), self.halo_recv_pos.data_ptr(), nr,
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
        self._halo(r_own, self.r_ext, CH_HALO_R)
        s = self._stream()
        self.ctx.launch_gnn_only(self.r_ext.data_ptr(), s)
        zloc, scale, r0r = self.ctx.local_outputs()
        ko, ks = p.own_subs.size, p.k_slots
        # all-gather (R0 r)_i and s_i of the own subdomains; slot map -> global order
        self._c(lib.ddmgnn_gather(r0r, self.own_slot.data_ptr(), ko, self.gath_in.data_ptr(), s))
        self._c(lib.ddmgnn_gather(scale, self.own_slot.data_ptr(), ko,
                                  self.gath_in[ks:].data_ptr(), s))
        if self.arena is not None:
            self.arena.allgather("gath_out", self.gath_in.data_ptr(), 2 * ks, CH_GATHER, s)
        else:
            self.comm.allgather(self.gath_out, self.gath_in)
        s = self._stream()
        self._c(lib.ddmgnn_gather(self.gath_out.data_ptr(), self.idx_r0r.data_ptr(), self.k,
                                  self.r0r_full.data_ptr(), s))
        self._c(lib.ddmgnn_gather(self.gath_out.data_ptr(), self.idx_scale.data_ptr(), self.k,
                                  self.scale_full.data_ptr(), s))
        if self.kinv is not None:
            self._c(lib.ddmgnn_dense_gemv(self.k, self.kinv.data_ptr(), self.r0r_full.data_ptr(),
                                          self.y.data_ptr(), s))
        # own terms + remote terms (owner glues in ascending subdomain order)
        self.zloc_ext[:p.v_own].copy_(_view_f64(zloc, p.v_own, self.device))
        if self.arena is not None:
            self.arena.put(CH_TERMS, zloc, self.term_send_pos.data_ptr(), self._term_send_off,
                           "zloc_ext", self._term_dst_off, s)
            self.arena.wait(CH_TERMS, self._term_recv_off, 0, None, None, 0, s)
        elif self.comm.size > 1:
            ns = p.term_send_pos.size
            self._c(lib.ddmgnn_gather(zloc, self.term_send_pos.data_ptr(), ns,
                                      self.term_send.data_ptr(), s))
            nr = sum(p.term_recv_counts)
            self.comm.alltoallv(self.zloc_ext[p.v_own:p.v_own + nr], self.term_send[:ns],
                                p.term_recv_counts, p.term_send_counts)
        s = self._stream()
        self._c(lib.ddmgnn_prolong(p.n_own, int(self.kinv is not None), self.tptr.data_ptr(),
                                   self.tent.data_ptr(), self.pou_own.data_ptr(),
                                   self.y.data_ptr(), self.scale_full.data_ptr(),
                                   self.zloc_ext.data_ptr(), z_own.data_ptr(), s))
        if self.arena is not None:  # the received terms are consumed: let the senders reuse
            self.arena.ack(CH_TERMS, self._term_recv_off, s)
        return z_own

    def capture_apply(self, r_own, z_own):
        """A CUDA graph of ``apply_owned(r_own, z_own)`` (device-ordered exchanges only;
        replay on the current stream)."""
        import torch

        if not self.device_ordered:
            raise RuntimeError("graph capture needs exchange='p2p' (or a single rank)")
        self.apply_owned(r_own, z_own)  # warm-up outside the capture
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self.apply_owned(r_own, z_own)
        return graph

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
    def _iteration(self, u, r, pv, q, z, z_old, st, hist, flexible):
        """One PCG iteration (sparse.py:106-126) as stream work; the scalars live in
        st (see ddmgnn_pcg_scalars), the updates are no-ops once the solve stopped."""
        lib, p = self._lib, self.plan
        n_own = p.n_own
        stream = self._stream
        self._halo(pv, self.p_ext, CH_HALO_P)
        s = stream()
        self.ctx.spmv_device(self.p_ext.data_ptr(), self.q_ext.data_ptr(), s)
        self._c(lib.ddmgnn_gather(self.q_ext.data_ptr(), self.own_pos.data_ptr(), n_own,
                                  q.data_ptr(), s))
        self._c(lib.ddmgnn_dot(n_own, pv.data_ptr(), q.data_ptr(), self.work.data_ptr(),
                               st[1:].data_ptr(), s))
        self._allreduce(st[1:2], CH_PQ)
        s = stream()
        self._c(lib.ddmgnn_pcg_scalars(0, st.data_ptr(), hist.data_ptr(), s))
        self._c(lib.ddmgnn_axpy2_dev(n_own, st.data_ptr(), pv.data_ptr(), q.data_ptr(),
                                     u.data_ptr(), r.data_ptr(), self.work.data_ptr(),
                                     st[3:].data_ptr(), s))
        self._allreduce(st[3:4], CH_RR)
        self._c(lib.ddmgnn_pcg_scalars(1, st.data_ptr(), hist.data_ptr(), stream()))
        if flexible:
            z_old.copy_(z)
        self.apply_owned(r, z)
        self._c(lib.ddmgnn_dot(n_own, r.data_ptr(), z.data_ptr(), self.work.data_ptr(),
                               st[6:].data_ptr(), stream()))
        if flexible:
            self._c(lib.ddmgnn_dot_diff(n_own, r.data_ptr(), z.data_ptr(), z_old.data_ptr(),
                                        self.work.data_ptr(), st[11:].data_ptr(), stream()))
            self._allreduce(st[11:12], CH_RZO)
        self._allreduce(st[6:7], CH_RZ)
        s = stream()
        self._c(lib.ddmgnn_pcg_scalars(3 if flexible else 2, st.data_ptr(), hist.data_ptr(), s))
        self._c(lib.ddmgnn_xpby_dev(n_own, z.data_ptr(), st.data_ptr(), pv.data_ptr(), s))

    def _poll(self, st) -> float:
        """Status of the solve (synchronises): the GNN status word of the applies
        since the last poll, a timed-out peer wait, then the recurrence's own word."""
        self.ctx.apply_status(self._stream())  # non-finite model output -> reference error
        if self.arena is not None and self.arena.timed_out():
            raise RuntimeError("peer exchange timed out (a rank stopped responding)")
        return float(st[9].item())

    def pcg(self, b_global, tol: float, max_iter: int, check_every: int = 8,
            flexible: bool = False, graph: bool | None = None):
        """Distributed PCG (sparse.py:76-127) with this preconditioner; collective.
        Returns (u_global, SolveReport) on every rank.  ``flexible=True``: the opt-in
        flexible CG (beta = <r, z - z_old> / rho), as ``sparse.pcg``.

        The recurrence's scalars live on the device (``st``, see ddmgnn_pcg_scalars):
        <p, Ap>, ||r||^2 and <r, z> are reduced into it in place by the all-reduces,
        alpha / beta / the stopping test are computed there, and the updates turn into
        no-ops once the solve has stopped — so the host only polls the status every
        ``check_every`` iterations.  With device-ordered exchanges (``graph`` default)
        the iteration is captured once in a CUDA graph and replayed; the host issues
        nothing else between polls."""
        import torch

        if tol <= 0:
            raise ValueError("tol must be positive")
        b = np.asarray(b_global, dtype=np.float64)
        if b.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got shape {b.shape}")
        if graph is None:
            graph = self.device_ordered
        lib, p = self._lib, self.plan
        n_own = p.n_own
        max_iter = max(0, int(max_iter))  # sparse.py:105: no iteration for max_iter < 0
        # solve buffers persist across calls, so a captured iteration is reused
        sb = getattr(self, "_solve", None)
        if sb is None or sb["hist"].numel() < max_iter + 1:
            f64 = dict(dtype=torch.float64, device=self.device)
            sb = self._solve = {
                "u": torch.zeros(n_own, **f64), "r": torch.zeros(n_own, **f64),
                "q": torch.zeros(n_own, **f64), "z": torch.zeros(n_own, **f64),
                "pv": torch.zeros(n_own, **f64), "z_old": torch.zeros(n_own, **f64),
                "st": torch.zeros(12, **f64),
                "hist": torch.zeros(max(max_iter + 1, 1024), **f64), "graphs": {}}
        u, r, q, z, pv, st, hist = (sb[k] for k in ("u", "r", "q", "z", "pv", "st", "hist"))
        bo = self.owned_part(b)
        u.zero_()
        r.copy_(bo)
        st.zero_()
        hist.zero_()
        stream = self._stream
        self._dot(bo, bo, 0)
        nb = float(np.sqrt(self._allreduce_scalar(0)))
        if nb == 0.0:  # sparse.py:93-94
            return np.zeros(self.n), SolveReport(0, [0.0], True, 0.0, tol)
        # r0 = b, so history[0] = ||b|| / ||b|| = 1 exactly (sparse.py:96-99)
        if 1.0 < tol:
            return np.zeros(self.n), SolveReport(0, [1.0], True, 1.0, tol)
        self.apply_owned(r, z)
        self.ctx.apply_status(self._stream())  # non-finite model output -> reference error
        pv.copy_(z)
        z_old = sb["z_old"] if flexible else None
        self._c(lib.ddmgnn_dot(n_own, r.data_ptr(), z.data_ptr(), self.work.data_ptr(),
                               st[0:].data_ptr(), stream()))
        self._allreduce(st[0:1], CH_RZ)  # rho = <r0, z0>
        st[4], st[5], st[10] = nb, float(tol), float(max_iter)
        hist[0] = 1.0  # r0 = b
        args = (u, r, pv, q, z, z_old, st, hist, flexible)
        it = 0
        if max_iter > 0:
            # the first iteration runs eagerly (warms every kernel / communicator up)
            self._iteration(*args)
            it = 1
        gx = None
        if graph and it < max_iter and self._poll(st) == 0.0:
            gx = sb["graphs"].get(flexible)
            if gx is None:
                gx = sb["graphs"][flexible] = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gx):
                    self._iteration(*args)
        while it < max_iter:
            if gx is not None:
                gx.replay()
            else:
                self._iteration(*args)
            it += 1
            if it % check_every == 0 or it == max_iter:
                if self._poll(st) != 0.0:
                    break
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
        self._allreduce(t, CH_PQ)
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


def _view_i64(ptr: int, n: int, device):
    import torch

    class _Cai:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_Cai(), device=device)
