"""Multi-GPU factorization and solve: boxes sharded over ranks, top levels
computed by process groups (arXiv 2502.02395 §5; the reference only SIMULATES
this plan in comm_sim.py:1-186 — here the data really moves).

Ownership follows the reference's ProcAssignment (comm_sim.py:17-37): with
P = 2^L0 ranks, rank g owns box i of a level l >= L0 iff i >> (l - L0) == g
(contiguous leaf ranges); a box of a level l < L0 is computed by its subtree's
process group [i P/2^l, (i+1) P/2^l), so every rank computes one box per such
level and the root (replicated_work, comm_sim.py:151-167).

Exchanges (one process per GPU, torch.distributed; NCCL over NVLink on a
multi-GPU node, gloo through host memory in the tests):
  factorization
    halo_v(l)     after the diagonal phase of a level: V_j (n_j x r_j) of every
                  box j that is the column of a near pair whose row box another
                  group computes (one all_gather; packing / unpacking are
                  cached block-copy programs)
    merge(l)      merging level l into a group-computed level l-1 < L0: each
                  rank writes the child blocks it contributes into zeroed parent
                  blocks, then ONE AllReduce per parent near block over the union
                  group of its two boxes (Eq. 34) — the event list of
                  comm_sim.simulate_factor exactly (merge_events, golden-tested)
    solve_halo    cross-group off-diagonal factor blocks (T_ij[:, :r_j], L(s)_ji)
                  also land on the column box's group, so the solve only moves
                  vectors
  solve           forward merges into group-computed levels: one AllReduce per
                  parent box over its group (simulate_solve's merge events);
                  within a level the segments each rank contributes are summed
                  across ranks (all_reduce of a masked level vector — simpler
                  than simulate_solve's per-pair neighbour reduce / broadcast)
"""

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from .program import Program

F64 = torch.float64


class Partition:
    """Box ownership over P = 2^L0 ranks (comm_sim.ProcAssignment semantics,
    comm_sim.py:17-37): at a level l >= L0 box i has the single owner
    i >> (l - L0) (contiguous leaf ranges); at a level l < L0 it is computed by
    its process group [i * P/2^l, (i+1) * P/2^l) — the replication the
    reference's simulator assumes (replicated_work, comm_sim.py:151-167), so a
    rank computes ONE box per replicated level and the root."""

    def __init__(self, p, depth):
        if p < 1 or p & (p - 1):
            raise ValueError("process count must be a power of 2")
        if p > 2 ** depth:
            raise ValueError(f"p = {p} exceeds the leaf count {2 ** depth}")
        self.p = p
        self.depth = depth
        self.L0 = int(math.log2(p))

    def group(self, l, i):
        if l >= self.L0:
            g = i >> (l - self.L0)
            return (g, g + 1)
        span = self.p >> l
        return (i * span, (i + 1) * span)

    def owner(self, l, i):
        return self.group(l, i)[0]

    contributor = owner   # the group member whose copy of a box's blocks enters a sum

    def owned_mask(self, l, rank):
        """Boxes of level l this rank computes (member of their group)."""
        i = np.arange(2 ** l)
        if l < self.L0:
            return i == (rank >> (self.L0 - l))
        return (i >> (l - self.L0)) == rank

    def contrib_mask(self, l, rank):
        """Boxes of level l whose contributor is this rank."""
        i = np.arange(2 ** l)
        if l < self.L0:
            return (i * (self.p >> l)) == rank
        return (i >> (l - self.L0)) == rank

    def union(self, l, i, j):
        gi, gj = self.group(l, i), self.group(l, j)
        return (min(gi[0], gj[0]), max(gi[1], gj[1]))


def merge_events(part, lists, kdims, depth):
    """The factorization's merge AllReduces, a pure function of the structure:
    one per parent near block (pi >= pj) of every level pl < L0 whose union
    group spans >= 2 ranks, over that group, 8 d_pi d_pj bytes (the zero-padded
    contributions of Eq. 34).  Equal to comm_sim.simulate_factor
    (comm_sim.py:92-106).  kdims: {l: array of ranks k}."""
    out = []
    for pl in range(min(depth - 1, part.L0 - 1), -1, -1):
        k = kdims[pl + 1]
        for (pi, pj) in sorted(lists.near[pl]):
            if pi < pj:
                continue
            g = part.union(pl, pi, pj)
            if g[1] - g[0] < 2:
                continue
            di, dj = int(k[2 * pi] + k[2 * pi + 1]), int(k[2 * pj] + k[2 * pj + 1])
            out.append(("factor", pl, "allreduce", g, 8 * di * dj, (pi, pj)))
    return out


@dataclass
class CommEvent:
    phase: str
    level: int
    kind: str
    bytes: int
    participants: tuple = None


@dataclass
class Comm:
    """Thin torch.distributed wrapper that also records a communication trace."""

    rank: int = 0
    world: int = 1
    group: object = None
    host_staged: bool = False      # gloo: collectives on host copies
    trace: list = field(default_factory=list)
    groups: dict = field(default_factory=dict)   # (lo, hi) -> process group of ranks [lo, hi)

    @classmethod
    def from_env(cls, group=None):
        import torch.distributed as dist

        if not dist.is_initialized():
            return cls()
        backend = dist.get_backend(group)
        return cls(rank=dist.get_rank(group), world=dist.get_world_size(group), group=group,
                   host_staged=(backend != "nccl"))

    def _log(self, phase, level, kind, nbytes, participants=None):
        self.trace.append(CommEvent(phase, level, kind, int(nbytes),
                                    participants if participants is not None else (0, self.world)))

    def make_groups(self, ranges):
        """Create the sub-communicators of the rank ranges [lo, hi) — collectively:
        every rank calls this with the same list (plan construction is replicated)."""
        import torch.distributed as dist

        for lo, hi in sorted(set(ranges)):
            if (lo, hi) in self.groups:
                continue
            if lo == 0 and hi == self.world:
                self.groups[(lo, hi)] = self.group
            else:
                self.groups[(lo, hi)] = dist.new_group(ranks=list(range(lo, hi)))

    def group_all_reduce_(self, t, rng, phase="factor", level=-1):
        """Sum over the ranks [lo, hi); a rank outside the range does nothing."""
        import torch.distributed as dist

        lo, hi = rng
        if not (lo <= self.rank < hi):
            return t
        self._log(phase, level, "allreduce", t.numel() * t.element_size(), (lo, hi))
        g = self.groups[(lo, hi)]
        if self.host_staged:
            h = t.cpu()
            dist.all_reduce(h, group=g)
            t.copy_(h)
        else:
            dist.all_reduce(t, group=g)
        return t

    def all_gather(self, t, phase="factor", level=-1):
        import torch.distributed as dist

        self._log(phase, level, "all_gather", t.numel() * t.element_size() * self.world)
        if self.host_staged:
            h = t.cpu()
            out = [torch.empty_like(h) for _ in range(self.world)]
            dist.all_gather(out, h, group=self.group)
            return [o.to(t.device) for o in out]
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return out

    def all_gather_into(self, out, t, phase="factor", level=-1):
        """out (world x t.numel(), contiguous) <- every rank's t."""
        import torch.distributed as dist

        self._log(phase, level, "all_gather", t.numel() * t.element_size() * self.world)
        if self.host_staged:
            h = t.cpu()
            parts = [torch.empty_like(h) for _ in range(self.world)]
            dist.all_gather(parts, h, group=self.group)
            out.copy_(torch.cat(parts).to(out.device))
        else:
            dist.all_gather_into_tensor(out, t, group=self.group)
        return out

    def all_reduce_(self, t, op="sum", phase="solve", level=-1):
        import torch.distributed as dist

        self._log(phase, level, "all_reduce", t.numel() * t.element_size())
        rop = dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MIN
        if self.host_staged:
            h = t.cpu()
            dist.all_reduce(h, op=rop, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=rop, group=self.group)
        return t

    def allreduce_min_(self, t):
        return self.all_reduce_(t, op="min", phase="factor", level=0)

    def all_max(self, x):
        import torch.distributed as dist

        t = torch.tensor([float(x)], dtype=F64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


# --------------------------------------------------------------------------- factorization exchanges

def _view(t, off, rows, cols, ld):
    return t.as_strided((rows, cols), (ld, 1), t.storage_offset() + off)


def _ptr(buf, off):
    return buf.ptr(off) if hasattr(buf, "ptr") else buf.data_ptr() + 8 * int(off)


def _has(buf, off):
    if not hasattr(buf, "hoff"):
        return True
    return buf.lo <= int(off) < buf.hi or int(off) in buf.hoff


class _ExchangeProgram:
    """Static pack / unpack of one exchange: ONE block-copy launch gathers this rank's
    exports into the send buffer, ONE scatters the other ranks' blocks out of the
    gathered buffer (h2g_block_copy; built once per plan and exchange)."""

    def __init__(self, plan, blocks):
        comm, dev = plan.comm, plan.device
        sizes = np.zeros(comm.world, dtype=np.int64)
        for own, _, _, rows, cols, _ in blocks:
            sizes[own] += rows * cols
        self.cap = int(sizes.max())
        if self.cap == 0:
            return
        self.send = torch.zeros(self.cap, dtype=F64, device=dev)
        self.recv = torch.zeros(comm.world * self.cap, dtype=F64, device=dev)
        pack, unpack = [], []
        cursor = np.zeros(comm.world, dtype=np.int64)
        for own, t, off, rows, cols, ld in blocks:
            c = int(cursor[own])
            if rows * cols:
                if own == comm.rank:
                    pack.append((_ptr(t, off), self.send.data_ptr() + 8 * c, rows, cols, ld, cols, 0))
                elif _has(t, off):      # a rank keeps only the halo blocks it reads
                    unpack.append((self.recv.data_ptr() + 8 * (own * self.cap + c), _ptr(t, off), rows, cols, cols,
                                   ld, 0))
            cursor[own] = c + rows * cols
        self.pack = Program(dev)
        self.pack.copy(pack)
        self.pack.finalize()
        self.unpack = Program(dev)
        self.unpack.copy(unpack)
        self.unpack.finalize()

    def run(self, comm, phase, level):
        if self.cap == 0:
            return
        self.pack.run()
        comm.all_gather_into(self.recv, self.send, phase=phase, level=level)
        self.unpack.run()


def _exchange_blocks(plan, blocks, phase, level, tag=None):
    """all_gather of per-rank block exports.

    blocks: list of (owner_rank, flat device tensor, offset, rows, cols, ld) —
    strided sub-blocks (only the slabs the receiver reads, e.g. V_j = R_j[:, :r_j],
    not all of R_j); every rank lists the same blocks in the same order; after the
    call each rank's copy of every block equals its owner's.  On the GPU the
    packing is a cached pair of block-copy programs (tag = the exchange)."""
    comm = plan.comm
    if plan.device.type == "cuda":
        cache = plan.__dict__.setdefault("_exchange_programs", {})
        key = tag if tag is not None else id(blocks)
        if key not in cache:
            cache[key] = _ExchangeProgram(plan, blocks)
        cache[key].run(comm, phase, level)
        return
    # host tensors (the CPU unit test of the exchange pattern)
    sizes = np.zeros(comm.world, dtype=np.int64)
    for own, _, _, rows, cols, _ in blocks:
        sizes[own] += rows * cols
    cap = int(sizes.max())
    if cap == 0:
        return
    send = torch.zeros(cap, dtype=F64, device=plan.device)
    pos = 0
    for own, t, off, rows, cols, ld in blocks:
        if own == comm.rank and rows * cols:
            send[pos:pos + rows * cols].view(rows, cols).copy_(_view(t, off, rows, cols, ld))
            pos += rows * cols
    recv = comm.all_gather(send, phase=phase, level=level)
    cursor = np.zeros(comm.world, dtype=np.int64)
    for own, t, off, rows, cols, ld in blocks:
        c = int(cursor[own])
        if own != comm.rank and rows * cols:
            _view(t, off, rows, cols, ld).copy_(recv[own][c:c + rows * cols].view(rows, cols))
        cursor[own] = c + rows * cols


def solve_merge_events(part, kdims, depth):
    """The forward sweep's merge AllReduces: merging level l into a group-computed
    level l-1 < L0, one per parent box whose group spans >= 2 ranks, over that
    group, 8 d bytes per right-hand side (comm_sim.simulate_solve, comm_sim.py:138-147)."""
    out = []
    for l in range(depth, 0, -1):
        if l - 1 >= part.L0:
            continue
        k = kdims[l]
        for pbox in range(2 ** (l - 1)):
            g = part.group(l - 1, pbox)
            if g[1] - g[0] < 2:
                continue
            out.append(("forward", l - 1, "allreduce", g, 8 * int(k[2 * pbox] + k[2 * pbox + 1])))
    return out


def cross_pairs(part, l, pairs):
    """Near pairs (i, j) whose boxes are computed by different process groups."""
    return [(i, j) for (i, j) in pairs if part.group(l, i) != part.group(l, j)]


def _halo_v_blocks(plan, l):
    """V_j (n_j x r_j, the first r_j columns of R_j) of the column boxes of cross-group near pairs
    (the row box's group forms T_ij = Q_i^T A_ij [V_j | q_skel_j]), from j's contributor."""
    part, B = plan.part, plan.bufs[l]
    lay = B.lay
    need = sorted({j for (i, j) in cross_pairs(part, l, lay.off_pairs)})
    return [(part.contributor(l, j), B.R, int(lay.qoff[j]), int(lay.n[j]), int(lay.r[j]), int(lay.n[j]))
            for j in need]


def _merge_allreduce(plan, l):
    """Merge of level l into the group-computed parent level l - 1: every rank wrote
    the child blocks it contributes into the zeroed parent buffer; one AllReduce
    per parent near block over its union group completes it (Eq. 34,
    comm_sim.simulate_factor)."""
    comm = plan.comm
    abuf, aoff, pn = plan.parent_buf[l]
    for (_, pl, _, g, _, (pi, pj)) in plan.merge_schedule[l]:
        seg = abuf[aoff[(pi, pj)]: aoff[(pi, pj)] + pn[pi] * pn[pj]]
        comm.group_all_reduce_(seg, g, phase="factor", level=pl)


def _solve_halo_blocks(plan):
    """Cross-group off-diagonal factor blocks for the column box's group: lr_off_ij and L(s)_ij
    (T_ij[:, :r_j]) and the mirror L(s)_ji, from the row box's contributor."""
    part = plan.part
    out = []
    for l, B in sorted(plan.bufs.items(), reverse=True):
        lay = B.lay
        for (i, j) in cross_pairs(part, l, lay.off_pairs):
            oi = part.contributor(l, i)
            out.append((oi, B.T, int(B.toff[(i, j)]), int(lay.n[i]), int(lay.r[j]), int(lay.n[j])))
            out.append((oi, B.LSm, int(B.lsoff[(i, j)]), int(lay.k[j]), int(lay.r[i]), int(lay.r[i])))
    return out


def run_exchange(plan, seg):
    kind, l = seg
    if plan.comm.host_staged:
        torch.cuda.current_stream(plan.device).synchronize()
    if kind == "halo_v":
        _exchange_blocks(plan, _halo_v_blocks(plan, l), "factor", l, tag=seg)
    elif kind == "merge":
        _merge_allreduce(plan, l)
    elif kind == "solve_halo":
        _exchange_blocks(plan, _solve_halo_blocks(plan), "factor", -1, tag=seg)
    else:
        raise ValueError(f"unknown exchange {kind}")


def run_segments(plan, stream=None):
    for seg in plan.segments:
        if isinstance(seg, Program):
            seg.launch(stream)
        else:
            run_exchange(plan, seg)


# --------------------------------------------------------------------------- public API

def factorize_distributed(h2, comm=None):
    """Sharded factorization of `h2` over the ranks of `comm` (default: the
    initialized torch.distributed world).  Every rank passes the same H2
    (construction is replicated); returns ULVFactors whose distributed levels
    hold this rank's boxes (``factors.partition``) and whose replicated top
    levels and root are complete on every rank."""
    from . import _native as nat
    from .h2_device import DeviceH2
    from .ulv_factor import FactorPlan, factors_from_plan

    nat.lib()
    comm = comm or Comm.from_env()
    if comm.world == 1 or h2.tree.depth == 0:
        from .ulv_factor import factorize

        return factorize(h2)
    part = Partition(comm.world, h2.tree.depth)
    dh2 = getattr(h2, "_device", None) or DeviceH2.from_host(h2)
    plan = FactorPlan(dh2, h2.lists, part=part, comm=comm)
    plan.run()
    plan.check_pivots()
    f = factors_from_plan(h2, plan)
    f.partition = part
    f.comm = comm
    return f


def solve_distributed(factors, b, mode="parallel"):
    """Distributed solve; every rank passes b (user order) and gets x."""
    from . import _native as nat
    from .ulv_solve import solve

    if getattr(factors, "partition", None) is None:
        return solve(factors, b, mode=mode)
    if mode != "parallel":
        raise ValueError("the distributed solve implements the parallel substitution")
    nat.lib()
    return solve(factors, b, mode=mode)
