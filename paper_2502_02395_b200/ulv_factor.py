"""H²-ULV factorization on the GPU — drop-in for `h2ulv.ulv_factor`.

`factorize(h2, batched=True, retain=False) -> ULVFactors` keeps the
reference signature and output contract (ulv_factor.py:154-316): per level
`lr_diag[i]`, `lr_off[(i, j)]`, `ls[(a, b)]`, `v[i]`, `dims[i]`, the root
factor, `merge_map`, the flop report and the write audit.  The blocks stay
in HBM; the numpy views materialize lazily on first access.

Per level l (fine to coarse) the whole level is a handful of batched launches
on five lanes (CUDA streams joined by events; the whole factorization is one
`Program`, replayed as one CUDA graph):

  lane 2  GEMM NN  MO_ij[:, r_j:] = A_ij q_skel_j                     off_mul1, skeleton part
          GEMM TN  SS_ij = q_skel_i^T MO_ij[:, r_j:]                   off_mul2, skeleton part
  lane 0  GEMM NN M_i = A_ii Q_i; TN H_i = Q_i^T M_i                        diag_mul1/2 (189-200)
          for p in 0, 64, ...: PANEL chol(H[p:p+b,p:p+b]) + inverse; TRSM of the rows below;
                               NEXT = update of the next block column          partial Cholesky
  lane 1  REST = the remaining trailing update (lower tiles)             (217-241): H becomes
  lane 4  V ride-along: R[:, :r] <- q_red L^-T, block column by block column (left-looking)
  lane 3  (deferred, only the solve reads it)
          GEMM NN  MO_ij[:, :r_j] = A_ij V_j ; GEMM TN T_ij[:, :r_j] = Q_i^T MO  -> lr_off, L(s)_ij
          GEMM TN  L(s)_ji = (A_ij q_skel_j)^T V_i = (L(r)_ii^-1 RS_ij)^T        off_mirror (282-286)
  lane 0  COPY parent near blocks <- 2x2 child SS / couplings             merge (289-303)
root: the same PANEL/GEMM loop on the merged d x d block (309-314).

Only the diagonal transform, the Cholesky panels and the merge are on the
critical path: the off-diagonal skeleton blocks SS_ij = q_skel_i^T A_ij
q_skel_j do not depend on the level's Cholesky (lane 2 runs them as soon as
the parent blocks exist), and the remaining off-diagonal factor blocks are
not read by the next level at all (lane 3 overlaps them with it).

`batched` is accepted for signature compatibility: there is only the batched
GPU path, and it is deterministic (no atomics in any reduction), so repeated
runs are bitwise identical — the property test_ulv_factor.py:227-241 checks.
"""

import os
import weakref
from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np
import torch

from .trace import ranged
from . import _native as nat
from .dense_core import PhaseFlops
from .errors import NotPositiveDefiniteError, StructureError
from .h2_device import DeviceH2
from .program import Program

INT_MAX = 2 ** 31 - 1
F64 = torch.float64
# fused per-box partial Cholesky (h2g_chol_box) for levels with at least this many boxes of
# size <= CHOL_BOX_MAX_N; the panel-step chain otherwise (few large boxes: the upper levels)
CHOL_BOX_MIN = int(os.environ.get("H2G_CHOL_BOX_MIN", "4096"))
CHOL_BOX_MAX_N = int(os.environ.get("H2G_CHOL_BOX_MAX_N", "512"))
CHOL_BOX_V = os.environ.get("H2G_CHOL_BOX_V", "0") == "1"
WY_TRANSFORM = os.environ.get("H2G_WY", "1") != "0"   # compact-WY diag transform where the bases carry it
def _wy_cfg():
    """Tile configs of the WY launches (A/B knob, read when a plan is built; "" = the
    planner's choice): W = A Yt, X, U, the relabelled update."""
    return [int(c) if c else None for c in os.environ.get("H2G_WY_CFG", ",,,11").split(",")]
PANEL_ROWS_PER_CTA = 128


class _LazyBlocks(Mapping):
    """Read-only dict whose values are downloaded from HBM on first access."""

    def __init__(self, keys, fetch, shared=None):
        # shared: a (key list, key set) pair cached with the plan (never mutated), so a new
        # factors object over the same structure costs O(1) per mapping instead of O(boxes)
        if shared is not None:
            self._keys, self._set = shared
        else:
            self._keys = list(keys)
            self._set = set(self._keys)
        self._fetch = fetch
        self._cache = {}

    def __getitem__(self, key):
        if key not in self._set:
            raise KeyError(key)
        if key not in self._cache:
            self._cache[key] = self._fetch(key)
        return self._cache[key]

    def __iter__(self):
        return iter(self._keys)

    def __len__(self):
        return len(self._keys)


@dataclass
class ULVLevel:
    lr_diag: Mapping = field(default_factory=dict)
    lr_off: Mapping = field(default_factory=dict)
    ls: Mapping = field(default_factory=dict)
    v: Mapping = field(default_factory=dict)
    dims: dict = field(default_factory=dict)


class ULVFactors:
    """Factor container with the reference's attributes (ulv_factor.py:34-47).

    Device factors (`plan` given, from factorize): the blocks stay in HBM and
    `levels[l].lr_diag[i]` etc. download lazily.  Host factors (`plan` None,
    the reference's own constructor signature `ULVFactors(h2=...)`, e.g. from
    storage.load_factors): numpy blocks filled in by the caller; the first
    solve uploads them into the device layout (plan_from_host_factors)."""

    def __init__(self, h2, plan=None, levels=None, root=None, merge_map=None, flops=None, audit=None,
                 retained=None):
        self.h2 = h2
        self._plan = plan
        self.levels = {} if levels is None else levels
        self.merge_map = {} if merge_map is None else merge_map
        self.flops = plan.flops if plan is not None else ({} if flops is None else flops)
        self.audit = plan.audit if plan is not None else ({} if audit is None else audit)
        self.retained = retained
        self._root = root
        self._host = plan is None

    @property
    def depth(self):
        return self._plan.depth if self._plan is not None else self.h2.tree.depth

    @property
    def root(self):
        if self._root is None and self._plan is not None:
            self._root = self._plan.download_root()
        return self._root

    @root.setter
    def root(self, value):
        self._root = value

    @property
    def device(self):
        """The FactorPlan whose HBM buffers hold these factors (uploaded on first use for host factors)."""
        if self._plan is None:
            self._plan = plan_from_host_factors(self)
        return self._plan


def factor_plan_of(factors):
    """FactorPlan of any factor container: ours, or a duck-typed host one
    (e.g. the reference's own ULVFactors dataclass), uploaded once."""
    if isinstance(factors, ULVFactors):
        return factors.device
    plan = factors.__dict__.get("_b200_plan")
    if plan is None:
        plan = plan_from_host_factors(factors)
        factors.__dict__["_b200_plan"] = plan
    return plan


def plan_from_host_factors(factors):
    """Device layout of host (numpy) factors: the bases / leaf blocks of
    factors.h2 (DeviceH2) and every factor block the substitution reads —
    L(r)_ii and L(s)_ii into H_i, lr_off / L(s)_ij into T_ij, L(s)_ji into
    the mirror slab, L_00 into the root buffer — placed exactly where the
    factorization leaves them, so the same solve program runs on them."""
    h2 = factors.h2
    dh2 = getattr(h2, "_device", None)
    if dh2 is None:
        dh2 = DeviceH2.from_host(h2)
    plan = FactorPlan(dh2, h2.lists)
    for l, B in plan.bufs.items():
        lay = B.lay
        lvl = factors.levels[l]
        n, r = lay.n, lay.r
        H = np.zeros(B.H.numel())
        for i in range(lay.nb):
            ni, ri = int(n[i]), int(r[i])
            blk = H[int(lay.qoff[i]):int(lay.qoff[i]) + ni * ni].reshape(ni, ni)
            blk[:ri, :ri] = lvl.lr_diag[i]
            blk[ri:, :ri] = lvl.ls[(i, i)]
        T = np.zeros(B.T.numel())
        LS = np.zeros(B.LSm.numel())
        for (i, j), off in B.toff.items():
            ni, nj, ri, rj = int(n[i]), int(n[j]), int(r[i]), int(r[j])
            blk = T[off:off + ni * nj].reshape(ni, nj)
            blk[:ri, :rj] = lvl.lr_off[(i, j)]
            blk[ri:, :rj] = lvl.ls[(i, j)]
            kj = nj - rj
            o = B.lsoff[(i, j)]
            LS[o:o + kj * ri] = np.asarray(lvl.ls[(j, i)], dtype=np.float64).reshape(-1)
        bufs = [(B.H, H), (B.T, T), (B.LSm, LS)]
        vs = getattr(lvl, "v", None) or {}
        if plan.has_v and all(i in vs for i in range(lay.nb) if r[i] > 0):
            R = np.zeros(B.R.numel())        # V_i (n_i x r_i, ulv_factor.py:31) where the factorization puts it
            for i in range(lay.nb):
                ni, ri = int(n[i]), int(r[i])
                if ri:
                    R[int(lay.qoff[i]):int(lay.qoff[i]) + ni * ni].reshape(ni, ni)[:, :ri] = vs[i]
            bufs.append((B.R, R))
        else:
            plan.has_v = False
        for dst, src in bufs:
            dst.tensor.copy_(torch.from_numpy(src))      # one GPU: the windows span everything
    d = plan.root_dim
    plan.root_buf[:d * d].copy_(torch.from_numpy(np.ascontiguousarray(factors.root, dtype=np.float64).reshape(-1)))
    plan.generation = 1
    torch.cuda.synchronize(plan.device)
    return plan


def _mat(t, off, rows, cols, ld, r0=0, c0=0):
    """Strided view of a row-major block inside flat tensor `t` (or a _Win, `off`
    global), as numpy."""
    if rows == 0 or cols == 0:
        return np.zeros((rows, cols))
    if isinstance(t, _Win):
        off, t = t.local(off), t.tensor
    base = off + r0 * ld + c0
    v = t[base: base + (rows - 1) * ld + cols].as_strided((rows, cols), (ld, 1))
    return v.cpu().numpy().copy()


class _LevelBuffers:
    pass


class _Win:
    """A level buffer holding only what this rank touches: a contiguous window
    [lo, hi) of the level's global offset space (the boxes / pairs it computes)
    plus individually placed halo blocks (global start offset -> size: the V_j
    it receives, the off-diagonal factor blocks of cross-group pairs).  One GPU:
    the whole space, no halo.  `data_ptr()` is the VIRTUAL base, so
    `data_ptr() + 8 * off` addresses window entries by their global offset;
    `ptr(off)` also resolves halo blocks."""

    def __init__(self, lo, hi, device, halo=None):
        halo = {int(o): int(sz) for o, sz in (halo or {}).items() if not (lo <= o < hi)}
        self.lo, self.hi = int(lo), int(hi)
        self.hoff, acc = {}, max(self.hi - self.lo, 0)
        for o in sorted(halo):
            self.hoff[o] = acc
            acc += halo[o]
        self.tensor = torch.empty(max(acc, 1), dtype=F64, device=device)

    def data_ptr(self):
        return self.tensor.data_ptr() - 8 * self.lo

    def ptr(self, off):
        off = int(off)
        if self.lo <= off < self.hi:
            return self.tensor.data_ptr() + 8 * (off - self.lo)
        return self.tensor.data_ptr() + 8 * self.hoff[off]

    def local(self, off):
        """Index into `tensor` of global offset `off` (window or halo block start)."""
        off = int(off)
        return off - self.lo if self.lo <= off < self.hi else self.hoff[off]

    def numel(self):
        return self.tensor.numel()


class _Session:
    """ctypes handle of h2g_session_* (include/h2ulv_b200.h): the plan's single program
    captured into a CUDA graph, launched asynchronously; the pivot statuses are decoded
    natively into (pivot, level, box) — the NotPositiveDefiniteError contract."""

    def __init__(self, plan):
        import ctypes

        prog = plan.program
        lib = nat.lib()
        base = np.zeros(plan.depth + 1, dtype=np.int32)
        for l, b in plan.slot_base.items():
            base[l] = b
        self._base = base
        side = torch.cuda.Stream(device=plan.device)
        torch.cuda.current_stream(plan.device).synchronize()
        h = ctypes.c_void_p()
        nat.check(lib.h2g_session_create(prog.steps.ctypes.data_as(ctypes.c_void_p), len(prog.steps),
                                         max(prog.n_events, 1), ctypes.c_void_p(plan.npd.data_ptr()), plan.depth,
                                         base.ctypes.data_as(ctypes.c_void_p), nat.stream_ptr(side),
                                         ctypes.byref(h)), "h2g_session_create")
        self.handle = h
        self._status = np.zeros(1, dtype=nat.NPD_STATUS_DT)

    def launch(self, stream=None):
        nat.check(nat.lib().h2g_session_factor_async(self.handle, nat.stream_ptr(stream)), "h2g_session_factor_async")

    def status(self, stream=None):
        """None, or (pivot, level, box) of the reported breakdown (synchronizes)."""
        rc = nat.lib().h2g_session_status(self.handle, nat.stream_ptr(stream),
                                          self._status.ctypes.data_as(nat.ctypes_void_p()))
        if rc == nat.H2G_ENPD:
            st = self._status[0]
            return int(st["pivot"]), int(st["level"]), int(st["box"])
        nat.check(rc, "h2g_session_status")
        return None

    def __del__(self):
        try:
            nat.load_library().h2g_session_destroy(self.handle)
        except Exception:
            pass


class FactorPlan:
    """Device buffers + the static step program(s) of one factorization.

    Single GPU: one Program.  Distributed (`part` = Partition, `comm` = Comm):
    every rank computes the boxes it owns at the distributed levels
    (l >= log2 P) and everything above; the program is cut into segments
    with collective exchanges in between (distributed.py)."""

    def __init__(self, dh2: DeviceH2, lists, part=None, comm=None, level_cuts=False):
        self.dh2 = dh2
        self.depth = dh2.depth
        self.generation = 0      # bumped whenever the buffers receive new factors (solve inverses follow)
        self.has_v = True        # R holds V_i = q_red L^-T (the factorization forms it; host uploads may not)
        self._session = None     # native factorization session (single program), see capture()
        self.part = part
        self.comm = comm
        self.dist = part is not None and part.p > 1
        self.merge_schedule, self.parent_buf = {}, {}
        if self.dist and dh2.depth >= 1:
            from .distributed import merge_events

            kdims = {l: lay.k for l, lay in dh2.levels.items()}
            for ev in merge_events(part, lists, kdims, dh2.depth):
                self.merge_schedule.setdefault(ev[1] + 1, []).append(ev)
            # the merge sub-communicators (factor: union groups of parent near blocks; solve: the
            # parent boxes' groups), created collectively in the same order on every rank
            comm.make_groups([ev[3] for evs in self.merge_schedule.values() for ev in evs] +
                             [part.group(l, i) for l in range(min(part.L0, dh2.depth)) for i in range(2 ** l)
                              if part.group(l, i)[1] - part.group(l, i)[0] >= 2])
        dev = dh2.device
        self.device = dev
        depth = self.depth
        self.segments = []
        self._programs = []
        prog = self._new_program()
        # pivot status: one slot per box of every level plus the root
        self.slot_base = {}
        acc = 0
        for l in range(depth, 0, -1):
            self.slot_base[l] = acc
            acc += 2 ** l
        self.slot_base[0] = acc
        self.npd = torch.full((acc + 1,), INT_MAX, dtype=torch.int32, device=dev)
        self._npd_init = torch.full((acc + 1,), INT_MAX, dtype=torch.int32, device=dev)
        prog.memcpy(self.npd.data_ptr(), self._npd_init.data_ptr(), 4 * (acc + 1))
        self.bufs = {}
        self.merge_pairs = {}
        self._keep = []

        if depth == 0:
            d = int(dh2.root_a.shape[0])
            self.root_buf = torch.empty(d * d, dtype=F64, device=dev)
            self.root_dim = d
            prog.memcpy(self.root_buf.data_ptr(), dh2.root_a.data_ptr(), 8 * d * d)
            self._cholesky_steps(prog, self.root_buf.data_ptr(), d, d, self.slot_base[0])
        else:
            a_buf, a_off = dh2.leaf_a, dh2.aoff
            merge_ev = None
            for l in range(depth, 0, -1):
                if level_cuts:
                    # streamed upload: level l's segment starts once its operands landed
                    prog = self._cut(prog, ("upload", l))
                    merge_ev = None
                lay = dh2.levels[l]
                B = _LevelBuffers()
                self.bufs[l] = B
                B.lay = lay
                n, k, r = lay.n, lay.k, lay.r
                nb = lay.nb
                mine = self.mine(l)
                # boxes this rank computes are contiguous (distributed.Partition): H, M and R hold
                # only them (+ the V_j halo in R), the pair buffers only the own / received pairs
                mi = np.flatnonzero(mine)
                sq = np.asarray(n, dtype=np.int64) ** 2
                wlo, whi = (int(lay.qoff[mi[0]]), int(lay.qoff[mi[-1]] + sq[mi[-1]])) if mi.size else (0, 0)
                if not self.dist:
                    wlo, whi = 0, max(lay.qsize, 1)
                from .distributed import cross_pairs
                cross = cross_pairs(self.part, l, lay.off_pairs) if self.dist else []
                halo_r = {int(lay.qoff[j]): int(sq[j]) for (i, j) in cross if mine[i] and not mine[j]}
                B.M = _Win(wlo, whi, dev)
                B.H = _Win(wlo, whi, dev)
                B.R = _Win(wlo, whi, dev, halo_r)
                B.a, B.aoff = a_buf, a_off
                qp, Hp, Rp, Mp = dh2.q[l].data_ptr(), B.H.data_ptr(), B.R.data_ptr(), B.M.data_ptr()
                ap = a_buf.data_ptr()
                qo = lay.qoff
                for (i, j) in lay.near_pairs:
                    if (i, j) not in a_off and mine[i]:
                        raise StructureError(f"missing near block ({l}, {i}, {j})")
                # ---- off-diagonal skeleton products (lane 2): chain-independent, needed by the merge
                #   MO[:, r_j:] = A_ij q_skel_j            (kept: the mirror's left operand)
                #   T[r_i:, r_j:] = q_skel_i^T MO[:, r_j:] = SS_ij
                offp = lay.off_pairs
                B.toff, B.lsoff = {}, {}
                tacc = lacc = 0
                for (i, j) in offp:
                    B.toff[(i, j)] = tacc
                    tacc += int(n[i] * n[j])
                    B.lsoff[(i, j)] = lacc
                    lacc += int(k[j] * r[i])
                own = [p for p in offp if mine[p[0]]]
                if not self.dist:
                    tw, lw = (0, max(tacc, 1)), (0, max(lacc, 1))
                elif own:
                    a_, b_ = own[0], own[-1]
                    tw = (B.toff[a_], B.toff[b_] + int(n[b_[0]] * n[b_[1]]))
                    lw = (B.lsoff[a_], B.lsoff[b_] + int(k[b_[1]] * r[b_[0]]))
                else:
                    tw, lw = (0, 0), (0, 0)
                recv = [(i, j) for (i, j) in cross if mine[j] and not mine[i]]   # solve_halo targets
                B.MO = _Win(tw[0], tw[1], dev)
                B.T = _Win(tw[0], tw[1], dev, {B.toff[p]: int(n[p[0]] * n[p[1]]) for p in recv})
                B.LSm = _Win(lw[0], lw[1], dev, {B.lsoff[p]: int(k[p[1]] * r[p[0]]) for p in recv})
                MOp, Tp, LSp = B.MO.data_ptr(), B.T.data_ptr(), B.LSm.data_ptr()
                own_off = [(i, j) for (i, j) in offp if mine[i]]
                prog.lane = 2
                if merge_ev is not None:
                    prog.wait(merge_ev)
                prog.gemm(0, 0, [(ap + 8 * a_off[(i, j)], qp + 8 * (qo[j] + r[j]), MOp + 8 * (B.toff[(i, j)] + r[j]),
                                  int(n[i]), int(k[j]), int(n[j]), int(n[j]), int(n[j]), int(n[j]), 0, 1.0, 0.0)
                                 for (i, j) in own_off])
                prog.role = "transform"
                prog.gemm(1, 0, [(qp + 8 * (qo[i] + r[i]), MOp + 8 * (B.toff[(i, j)] + r[j]),
                                  Tp + 8 * (B.toff[(i, j)] + r[i] * n[j] + r[j]),
                                  int(k[i]), int(k[j]), int(n[i]), int(n[i]), int(n[j]), int(n[j]), 0, 1.0, 0.0)
                                 for (i, j) in own_off])
                prog.role = None
                ev_ss = prog.event()
                prog.record(ev_ss)
                # ---- diagonal phase (lane 0 = the critical chain)
                prog.lane = 0
                wy = getattr(dh2, "wy", {}).get(l) if WY_TRANSFORM and not self.dist else None
                if wy is not None:
                    self._wy_transform(prog, wy, lay, ap, a_off, Hp)
                else:
                    prob = []
                    for i in range(nb):
                        if not mine[i]:
                            continue
                        ni = int(n[i])
                        prob.append((ap + 8 * a_off[(i, i)], qp + 8 * qo[i], Mp + 8 * qo[i], ni, ni, ni, ni, ni, ni,
                                     0, 1.0, 0.0))
                    prog.gemm(0, 0, prob, split=True)
                    # H = Q^T (A Q) is symmetric and only its lower half is ever read
                    # (partial Cholesky, L(s)_ii, the SS merge): lower tiles only
                    prob = [(qp + 8 * qo[i], Mp + 8 * qo[i], Hp + 8 * qo[i], int(n[i]), int(n[i]), int(n[i]),
                             int(n[i]), int(n[i]), int(n[i]), nat.GEMM_LOWER, 1.0, 0.0) for i in range(nb) if mine[i]]
                    prog.role = "transform"
                    prog.gemm(1, 0, prob, split=True)
                    prog.role = None
                B.linv, B.loff, ev_v = self._partial_cholesky_steps(prog, Hp, Rp, qo, n, r, self.slot_base[l], mine,
                                                                    Qp=qp)
                if self.dist and self._cross(l, lay):
                    # V_j of boxes computed by another group but coupled to mine by a near pair
                    prog = self._cut(prog, ("halo_v", l))
                    ev_v = ev_ss = None          # the cut joined every lane
                # ---- deferred off-diagonal factor blocks (lane 3): read only by the solve
                #   MO[:, :r_j] = A_ij V_j
                #   T[:, :r_j]  = Q_i^T MO[:, :r_j]        -> lr_off (rows < r_i), L(s)_ij (rows >= r_i)
                #   L(s)_ji     = (A_ij q_skel_j)^T V_i     = (L(r)_ii^-1 RS_ij)^T   off_mirror (282-286)
                prog.lane = 3
                for ev in (ev_v, ev_ss):
                    if ev is not None:
                        prog.wait(ev)
                prog.gemm(0, 0, [(ap + 8 * a_off[(i, j)], B.R.ptr(qo[j]), MOp + 8 * B.toff[(i, j)],
                                  int(n[i]), int(r[j]), int(n[j]), int(n[j]), int(n[j]), int(n[j]), 0, 1.0, 0.0)
                                 for (i, j) in own_off])
                prob = []
                for (i, j) in own_off:
                    ni, nj, ri, rj, kj = int(n[i]), int(n[j]), int(r[i]), int(r[j]), int(k[j])
                    mo = MOp + 8 * B.toff[(i, j)]
                    prob.append((qp + 8 * qo[i], mo, Tp + 8 * B.toff[(i, j)], ni, rj, ni, ni, nj, nj, 0, 1.0, 0.0))
                    prob.append((mo + 8 * rj, Rp + 8 * qo[i], LSp + 8 * B.lsoff[(i, j)], kj, ri, ni, nj, ni, ri,
                                 0, 1.0, 0.0))
                prog.role = "transform"
                prog.gemm(1, 0, prob)
                prog.role = None
                prog.lane = 0
                # ---- merge into the parent level (or the root)
                if ev_ss is not None:
                    prog.wait(ev_ss)
                if self.dist and l - 1 < self.part.L0:
                    # group-computed parent level: each rank writes the child blocks it contributes
                    # into the zeroed parent blocks; one AllReduce per parent near block over its
                    # union group completes them (Eq. 34; comm_sim.simulate_factor)
                    a_buf, a_off = self._merge_steps(prog, l, B, lists, dh2, group=True)
                    prog = self._cut(prog, ("merge", l))
                    merge_ev = None
                else:
                    a_buf, a_off = self._merge_steps(prog, l, B, lists, dh2)
                    merge_ev = prog.event()
                    prog.record(merge_ev)
            d = self._root_d
            self.root_dim = d
            self.root_buf = a_buf
            self._cholesky_steps(prog, a_buf.data_ptr(), d, d, self.slot_base[0])

        self.flops = flop_report({l: (B.lay.n, B.lay.k, B.lay.off_pairs) for l, B in self.bufs.items()},
                                 self.root_dim)
        if self.dist and depth >= 1 and any(self._cross(l, B.lay) for l, B in self.bufs.items()):
            # cross-group off-diagonal factor blocks also go to the column box's group (solve)
            prog = self._cut(prog, ("solve_halo", -1))
        self.segments.append(prog.finalize())
        self.audit = self._audit()
        self.program = self.segments[0] if len(self.segments) == 1 else None

    # ------------------------------------------------------------------ distribution hooks
    def mine(self, l):
        """Boolean mask of the level-l boxes this rank computes (distributed.Partition)."""
        nb = 2 ** l
        if not self.dist:
            return np.ones(nb, dtype=bool)
        return self.part.owned_mask(l, self.comm.rank)

    def device_bytes(self):
        """Bytes of the per-level factorization buffers this rank holds (H, M, R, MO, T, L(s) mirror)."""
        return sum(8 * getattr(B, x).numel() for B in self.bufs.values() for x in ("H", "M", "R", "MO", "T", "LSm"))

    def _cross(self, l, lay):
        from .distributed import cross_pairs

        return bool(cross_pairs(self.part, l, lay.off_pairs))

    def distributed_level(self, l):
        return self.part is not None and self.part.p > 1 and l >= self.part.L0

    def _new_program(self):
        prog = Program(self.device)
        prog.record_writes = True       # the write audit is derived from the programs' extents
        self._programs.append(prog)
        return prog

    def _cut(self, prog, tag):
        self.segments.append(prog.finalize())
        self.segments.append(tag)
        return self._new_program()

    # ------------------------------------------------------------------ steps
    @staticmethod
    def _wy_transform(prog, lq, lay, ap, a_off, Hp):
        """diag_mul1/2 (ulv_factor.py:189-200) through the compact-WY form of the
        bases (basis_qr.build_wy): Q = I - V Vt^T (Vt = V T), so
            H' = Q^T A Q = A - W V^T - V U^T,  W = A Vt,  U = W - V (Vt^T W)
        — 2n^2k + 2n^2k + 4nk^2 flops instead of 3n^3 (n = 256, k ~ 43 at the N = 1M
        leaf: ~4x fewer).  Four grouped GEMMs: W into P[:, :k]; X = Vt^T W; U = W - V X
        into Qm[:, k:] (beta term from W: a separate Cin); then ONE lower NT GEMM with
        K = 2k, H = relabel(A - [W | V] [V | U]^T), whose epilogue writes H' entry
        (a, b) to H in q_full = [q_red | q_skel s] order with id_basis's signs (the
        relabel store of h2g_gemm_grouped_ext).  Same matrix as Q^T (A Q) up to rounding."""
        n, k, qo = lay.n, lay.k, lay.qoff
        boxes = range(lay.nb)
        P = {i: lq.ptr(lq.wy_p, lq.wy_poff[i]) for i in boxes}
        Qm = {i: lq.ptr(lq.wy_q, lq.wy_poff[i]) for i in boxes}
        Vt = {i: lq.ptr(lq.wy_vt, lq.zoff[i]) for i in boxes}
        X = {i: lq.ptr(lq.wy_x, lq.foff[i]) for i in boxes}
        A = {i: ap + 8 * a_off[(i, i)] for i in boxes}
        ni = {i: int(n[i]) for i in boxes}
        ki = {i: int(k[i]) for i in boxes}
        _WY_CFG = _wy_cfg()
        prog.gemm(0, 0, [(A[i], Vt[i], P[i], ni[i], ki[i], ni[i], ni[i], ki[i], 2 * ki[i], 0, 1.0, 0.0)
                         for i in boxes], tile_cfg=_WY_CFG[0])                              # W = A Vt
        prog.gemm(1, 0, [(Vt[i], P[i], X[i], ki[i], ki[i], ni[i], ki[i], 2 * ki[i], ki[i], 0, 1.0, 0.0)
                         for i in boxes], tile_cfg=_WY_CFG[1])                              # X = Vt^T W
        prog.gemm(0, 0, [(Qm[i], X[i], Qm[i] + 8 * ki[i], ni[i], ki[i], ki[i], 2 * ki[i], ki[i], 2 * ki[i], 0,
                          -1.0, 1.0, (P[i], 0, 2 * ki[i], -1)) for i in boxes], tile_cfg=_WY_CFG[2])   # U = W - V X
        prog.role = "transform"
        sg = {i: lq.ptr(lq.wy_sgn, lq.tauoff[i]) for i in boxes}
        prog.gemm(0, 1, [(P[i], Qm[i], Hp + 8 * int(qo[i]), ni[i], ni[i], 2 * ki[i], 2 * ki[i], 2 * ki[i], ni[i],
                          nat.GEMM_LOWER, -1.0, 1.0, (A[i], sg[i], ni[i], ki[i])) for i in boxes],
                  tile_cfg=_WY_CFG[3])
        prog.role = None

    def _partial_cholesky_steps(self, prog, Hp, Rp, qo, n, r, slot0, mine=None, Qp=0):
        return partial_cholesky_steps(prog, self.device, self.npd.data_ptr(), Hp, Rp, qo, n, r, slot0, mine, Qp)

    def _cholesky_steps(self, prog, ptr, d, ld, slot):
        """Root: full Cholesky of the merged d x d block (the solve forms its
        explicit inverse from L_00 itself, ulv_solve.SolvePlan._build_prepare)."""
        assert d == ld
        self.root_linv, _, _ = self._partial_cholesky_steps(prog, ptr, 0, np.array([0]), np.array([d]),
                                                            np.array([d]), slot)

    def _merge_steps(self, prog, l, B, lists, dh2, group=False):
        """Parent near blocks of level l-1 from the child SS blocks / couplings.
        group=True (distributed, group-computed parent level): only the child blocks
        this rank contributes are written, into zeroed parent blocks (the merge
        AllReduce sums them)."""
        lay = B.lay
        n, k, r = lay.n, lay.k, lay.r
        parents = sorted((pi, pj) for (pi, pj) in lists.near[l - 1] if pi >= pj)
        self.merge_pairs[l] = parents
        if group:
            rank, part = self.comm.rank, self.part
            built = [(pi, pj) for (pi, pj) in parents
                     if part.union(l - 1, pi, pj)[0] <= rank < part.union(l - 1, pi, pj)[1]]
        else:
            pmine = self.mine(l - 1) if l - 1 >= 1 else np.ones(1, dtype=bool)
            built = [(pi, pj) for (pi, pj) in parents if pmine[pi]]
        pn = {p: int(k[2 * p] + k[2 * p + 1]) for p in range(2 ** (l - 1))}
        aoff, acc = {}, 0
        for (pi, pj) in parents:
            aoff[(pi, pj)] = acc
            acc += pn[pi] * pn[pj]
        abuf = torch.empty(max(acc, 1), dtype=F64, device=self.device)
        if group:
            zero = torch.zeros_like(abuf)
            self._keep.append(zero)
            prog.memcpy(abuf.data_ptr(), zero.data_ptr(), 8 * abuf.numel())
            self.parent_buf[l] = (abuf, aoff, pn)
        if l == 1:
            self._root_d = pn[0]
        Hp, Tp, Sp = B.H.data_ptr(), B.T.data_ptr(), dh2.s[l].data_ptr()
        qo = lay.qoff
        descs = []
        for (pi, pj) in built:
            dst0 = abuf.data_ptr() + 8 * aoff[(pi, pj)]
            ldd = pn[pj]
            for a in (0, 1):
                ci = 2 * pi + a
                ro = 0 if a == 0 else int(k[2 * pi])
                for b in (0, 1):
                    cj = 2 * pj + b
                    co = 0 if b == 0 else int(k[2 * pj])
                    dst = dst0 + 8 * (ro * ldd + co)
                    kci, kcj = int(k[ci]), int(k[cj])
                    if group:   # exactly one member of the union group contributes each child block
                        hi_ = max(ci, cj)
                        near_child = ci == cj or (hi_, min(ci, cj)) in B.toff
                        who = (self.part.contributor(l, hi_) if near_child
                               else self.part.union(l - 1, pi, pj)[0])
                        if who != rank:
                            continue
                    if ci == cj:
                        src = Hp + 8 * int(qo[ci] + r[ci] * n[ci] + r[ci])
                        descs.append((src, dst, kci, kcj, int(n[ci]), ldd, 2))
                        continue
                    hi, lo = (ci, cj) if ci > cj else (cj, ci)
                    mode = 0 if ci > cj else 1
                    if (hi, lo) in B.toff:
                        src = Tp + 8 * int(B.toff[(hi, lo)] + r[hi] * n[lo] + r[lo])
                        lds = int(n[lo])
                    elif (hi, lo) in lay.soff:
                        src = Sp + 8 * int(lay.soff[(hi, lo)])
                        lds = int(k[lo])
                    else:
                        raise StructureError(f"missing child SS block ({l}, {ci}, {cj})")
                    descs.append((src, dst, kci, kcj, lds, ldd, mode))
        prog.copy(descs)
        return abuf, aoff

    def _audit(self):
        """Write audit of the reference's slab store (ulv_factor.py:50-67, 319-337),
        derived from the write extents of every step of the program(s): see
        audit_writes.  The slabs are the sparsified diagonal blocks H_i and the
        off-diagonal blocks T_ij of every level."""
        regions = []
        for l, B in self.bufs.items():
            lay = B.lay
            n, r = lay.n, lay.r
            mine = self.mine(l)
            for i in range(lay.nb):
                if mine[i]:
                    regions.append((B.H.data_ptr() + 8 * int(lay.qoff[i]), int(n[i]), int(n[i]), int(r[i]), int(r[i]),
                                    ("diag", l, i, i)))
            for (i, j), off in B.toff.items():
                if mine[i]:
                    regions.append((B.T.data_ptr() + 8 * int(off), int(n[i]), int(n[j]), int(r[i]), int(r[j]),
                                    ("off", l, i, j)))
        writes = [w for prog in self._programs for w in prog.writes]
        for prog in self._programs:
            prog.writes = []
        return audit_writes(regions, writes)

    # ------------------------------------------------------------------ run / check
    def run(self, stream=None):
        self.generation += 1
        if self._session is not None:
            self._session.launch(stream)
            return
        if self.program is not None:
            self.program.launch(stream)
            return
        from .distributed import run_segments

        run_segments(self, stream)

    def launch_streamed(self, post=None):
        """Incremental launcher for a plan built with level_cuts: returns
        (on_level, finish).  on_level(l, event) — called by DeviceH2.from_host
        when level l's operands are on their way — queues every segment up to
        and including level l's after a wait on `event`; finish() queues the
        rest (the root).  post(l), when given, is called right after level l's
        segment is queued (its factor blocks are final once it ran); post(0)
        after the root."""
        stream = torch.cuda.current_stream(self.device)
        segs = self.segments
        state = {"i": 0, "level": None}

        def launched(seg):
            seg.launch(stream)
            if post is not None and state["level"] is not None:
                post(state["level"])
                if state["level"] == 1:
                    post(0)
                state["level"] = None

        def on_level(level, event):
            waited = False
            while state["i"] < len(segs):
                seg = segs[state["i"]]
                if isinstance(seg, Program):
                    launched(seg)
                elif seg[0] == "upload" and seg[1] == level and not waited:
                    state["level"] = level
                    stream.wait_event(event)
                    waited = True
                elif seg[0] == "upload":
                    return              # a later level: wait for its upload
                else:
                    raise ValueError(f"streamed launch does not support the exchange {seg}")
                state["i"] += 1

        def finish():
            while state["i"] < len(segs):
                seg = segs[state["i"]]
                if not isinstance(seg, Program):
                    raise RuntimeError(f"streamed launch: level {seg} was never uploaded")
                launched(seg)
                state["i"] += 1

        self.generation += 1
        return on_level, finish

    def capture(self):
        """Single program (one GPU): a native factorization session (h2g_session_create:
        the program captured into one CUDA graph, pivot statuses decoded in C).
        Segmented plans (distributed / streamed): a CUDA graph per program segment,
        the collectives outside."""
        if self.program is not None and not self.dist:
            if self._session is None:
                self._session = _Session(self)
            return
        for seg in self.segments:
            if isinstance(seg, Program) and seg.graph is None:
                seg.capture()

    def check_pivots(self):
        if self._session is not None:
            st = self._session.status()
            if st is not None:
                raise NotPositiveDefiniteError(st[0], level=st[1], box=st[2])
            return
        if self.comm is not None and self.part is not None and self.part.p > 1:
            self.comm.allreduce_min_(self.npd)
        npd = self.npd.cpu().numpy()
        if (npd == INT_MAX).all():
            return
        for l in list(range(self.depth, 0, -1)) + [0]:
            base = self.slot_base[l]
            cnt = 2 ** l if l > 0 else 1
            seg = npd[base:base + cnt]
            bad = np.flatnonzero(seg != INT_MAX)
            if bad.size:
                box = int(bad[0])
                raise NotPositiveDefiniteError(int(seg[box]), level=l, box=box)

    # ------------------------------------------------------------------ views
    def download_root(self):
        d = self.root_dim
        return np.tril(_mat(self.root_buf, 0, d, d, d))

    def level_views(self, l):
        B = self.bufs[l]
        lay = B.lay
        n, k, r, qo = lay.n, lay.k, lay.r, lay.qoff
        nb = lay.nb
        lvl = ULVLevel()
        # the structure (dims, key lists) is the plan's: built once, shared by every factors object
        st = self.__dict__.setdefault("_view_struct", {}).get(l)
        if st is None:
            mine = self.mine(l)           # distributed: only the blocks this rank computed
            boxes = [i for i in range(nb) if mine[i]]
            pairs = [p for p in lay.off_pairs if mine[p[0]]]
            keys = [(i, i) for i in boxes] + list(pairs) + [(j, i) for (i, j) in pairs]
            st = ({i: (int(r[i]), int(k[i])) for i in range(nb)},
                  (boxes, set(boxes)), (pairs, set(pairs)), (keys, set(keys)))
            self._view_struct[l] = st
        dims, sb, sp_, sk = st
        lvl.dims = dict(dims)
        lvl.lr_diag = _LazyBlocks(None, lambda i: np.tril(_mat(B.H, int(qo[i]), int(r[i]), int(r[i]), int(n[i]))),
                                  shared=sb)
        lvl.v = _LazyBlocks(None, lambda i: _mat(B.R, int(qo[i]), int(n[i]), int(r[i]), int(n[i])), shared=sb)
        lvl.lr_off = _LazyBlocks(None, lambda p: _mat(B.T, B.toff[p], int(r[p[0]]), int(r[p[1]]), int(n[p[1]])),
                                 shared=sp_)

        def ls_fetch(key):
            a, b = key
            if a == b:
                return _mat(B.H, int(qo[a]), int(k[a]), int(r[a]), int(n[a]), r0=int(r[a]))
            if a > b:
                return _mat(B.T, B.toff[(a, b)], int(k[a]), int(r[b]), int(n[b]), r0=int(r[a]))
            return _mat(B.LSm, B.lsoff[(b, a)], int(k[a]), int(r[b]), int(r[b]))

        lvl.ls = _LazyBlocks(None, ls_fetch, shared=sk)
        return lvl


def partial_cholesky_steps(prog, device, npd_ptr, Hp, Rp, qo, n, r, slot0, mine=None, Qp=0):
    """Right-looking partial Cholesky of every box's H (and the V ride-along
    rows in R), panels of W = 64 columns, one fused kernel per panel on the
    critical lane:

      lane 0:  [wait REST(q-2)] -> PANEL(q) -> [wait REST(q-1)] -> PANEL(q+1) ...
      lane 1:          [wait PANEL(q)] -> REST(q)
      lane 4:          [wait last PANEL] -> ROWS_V (all block columns, one launch)

    PANEL(q) (h2g_chol_panel: a diag kernel and a row-chunk kernel) applies
    panel q-1 to block column q, factors the diagonal block and TRSMs the
    rows below; REST(q) applies panel q to the columns < r right of block
    column q+1 (lower tiles of RR, all SR rows); the SS corner receives its
    single Schur update SS -= L(s) L(s)^T (K = r) after the last panel.
    ROWS_V (h2g_trsm_rows, left-looking, one CTA per 64 rows walking all
    block columns) forms R = Q_red L^-T = V from Q (Qp) off the critical
    lane; with Qp == 0 (the root) the identity rides along panel by panel
    and R becomes L^-T (the root's explicit inverse for the solve).  Returns
    (linv, loff, event after the last R column or None)."""
    nb = len(n)
    mine = np.ones(nb, dtype=bool) if mine is None else mine
    rmax = int(np.asarray(r)[mine].max()) if mine.any() else 0
    W = nat.PANEL_WIDTH
    nblk = -(-np.asarray(r, dtype=np.int64) // W)
    loff = np.concatenate([[0], np.cumsum(nblk)[:-1]]).astype(np.int64)
    linv = torch.zeros(max(int(nblk.sum()), 1) * W * W, dtype=F64, device=device)
    if rmax == 0:
        return linv, loff, None
    lp = linv.data_ptr()
    nmine = int(mine.sum())
    if Qp and nmine >= CHOL_BOX_MIN and int(np.asarray(n)[mine].max()) <= CHOL_BOX_MAX_N:
        # many boxes: the whole elimination of a box in ONE CTA (h2g_chol_box), all boxes in
        # one launch — no panel-by-panel launch chain, REST or separate SYRK
        # V = q_red L^-T: in the same CTA, panel by panel (H2G_CHOL_BOX_V=1), or one trsm_rows
        # launch on lane 4 (default).  M1: 27.10 vs 26.80 ms — the GPU is saturated either way
        # (the separate launch costs 4.0 ms of wall time in the lane ablation, the fused rows 3.2 ms
        # of critical-lane time).
        fuse_v = CHOL_BOX_V
        prog.chol_box([(Hp + 8 * int(qo[i]), lp + 8 * int(loff[i]) * W * W, int(n[i]), int(r[i]), int(n[i]),
                        slot0 + i) + ((Qp + 8 * int(qo[i]), Rp + 8 * int(qo[i])) if fuse_v else (0, 0))
                       for i in range(nb) if mine[i] and r[i] > 0], npd_ptr)
        prog.role = None
        if not fuse_v:
            ev_fp = prog.event()
            prog.record(ev_fp)
            prog.lane = 4
            prog.wait(ev_fp)
            prog.trsm_rows([(Hp + 8 * int(qo[i]), Qp + 8 * int(qo[i]), Rp + 8 * int(qo[i]),
                             lp + 8 * int(loff[i]) * W * W, int(n[i]), int(r[i]), 0, int(nblk[i]), int(n[i]),
                             int(n[i])) for i in range(nb) if mine[i] and r[i] > 0])
        ev_v = prog.event()
        prog.record(ev_v)
        prog.lane = 0
        return linv, loff, ev_v
    rest_ev = []                      # rest_ev[q]: REST(q) done (None: no REST launch)
    for q, p in enumerate(range(0, rmax, W)):
        descs, rest, rows = [], [], []
        for i in range(nb):
            ri, ni = int(r[i]), int(n[i])
            if ri <= p or not mine[i]:
                continue
            b = min(W, ri - p)
            h = Hp + 8 * int(qo[i])
            li = lp + 8 * (int(loff[i]) + q) * W * W
            descs.append((h, li, ni, W, ni, p, b, slot0 + i))
            q0 = p + b                               # first column right of the panel
            c0 = q0 + (min(W, ri - q0) if ri > q0 else 0)   # right of the next panel
            if ri > c0:
                # columns c0 .. r only: the SS corner gets its single Schur update at the end
                x = h + 8 * (c0 * ni + p)            # panel rows c0.. : H[c0:, p:p+b]
                rest.append((x, x, h + 8 * (c0 * ni + c0), ri - c0, ri - c0, b, ni, ni, ni,
                             nat.GEMM_LOWER, -1.0, 1.0))
                if ni > ri:                          # SR rows
                    rest.append((h + 8 * (ri * ni + p), x, h + 8 * (ri * ni + c0), ni - ri, ri - c0, b,
                                 ni, ni, ni, 0, -1.0, 1.0))
            if Rp and not Qp:                        # root: L^-T panel by panel (rows < p + b)
                rows.append((h, 0, Rp + 8 * int(qo[i]), lp + 8 * int(loff[i]) * W * W, ni, ri, q, q + 1,
                             ni, ni))
        done = [e for e in rest_ev[:max(q - 1, 0)] if e is not None]
        if done:
            prog.wait(done[-1])              # block column q has all updates of panels <= q-2
        prog.role = "factor"
        prog.chol_panel(descs, npd_ptr)
        ev_fp = prog.event()
        prog.record(ev_fp)
        ev_rest = None
        if rest:
            prog.lane = 1
            prog.wait(ev_fp)
            prog.gemm(0, 1, rest)     # role "factor": the in-place trailing update of RR / SR
            ev_rest = prog.event()
            prog.record(ev_rest)
        rest_ev.append(ev_rest)
        if rows:
            prog.lane = 4
            prog.wait(ev_fp)
            prog.trsm_rows(rows)
        prog.lane = 0
    if Rp and Qp:
        # V = Q_red L^-T for every box in ONE launch once all panels are factored:
        # each CTA walks the block columns of its 64 rows (left-looking)
        prog.lane = 4
        prog.wait(ev_fp)
        prog.trsm_rows([(Hp + 8 * int(qo[i]), Qp + 8 * int(qo[i]), Rp + 8 * int(qo[i]),
                         lp + 8 * int(loff[i]) * W * W, int(n[i]), int(r[i]), 0, int(nblk[i]), int(n[i]), int(n[i]))
                        for i in range(nb) if mine[i] and r[i] > 0])
        prog.lane = 0
    ev_v = None
    if Rp:
        ev_v = prog.event()
        prog.lane = 4
        prog.record(ev_v)
        prog.lane = 0
    last = [e for e in rest_ev if e is not None]
    if last:
        prog.wait(last[-1])                  # lane 1 is in order: the last REST covers all
    # the single Schur update SS_ii -= L(s) L(s)^T with K = r (ulv_factor.py:236-241)
    schur = []
    for i in range(nb):
        ri, ni = int(r[i]), int(n[i])
        if mine[i] and ri > 0 and ni > ri:
            ls = Hp + 8 * int(qo[i] + ri * ni)  # H[r:, 0:r]
            schur.append((ls, ls, ls + 8 * ri, ni - ri, ni - ri, ri, ni, ni, ni, nat.GEMM_LOWER, -1.0, 1.0))
    prog.role = "schur"
    prog.gemm(0, 1, schur)
    prog.role = None
    return linv, loff, ev_v


def audit_writes(regions, writes):
    """The reference's write audit (ulv_factor.py:50-67, 319-337) from program extents.

    regions: (ptr, rows, cols, r_split, c_split, key) of every slab block —
      key ("diag", l, i, i) for H_i, ("off", l, i, j) for T_ij; its sub-blocks
      are rr = [:r_split, :c_split], rs, sr, ss as in the reference.
    writes: (step, role, ptr, rows, cols, ld, lower) of every step descriptor
      (Program.writes); roles: "transform" — the U^T A V GEMM that stores the
      sparsified block (the reference's _Slabs.init), "factor" — the in-place
      partial Cholesky of the box's own RR / SR (panels + their trailing
      updates: the reference keeps L(r) / L(s) outside its slab store, so these
      overwrite factor OUTPUT, not a slab), "schur" — the SS_ii -= L(s) L(s)^T
      update; anything else (or any write of a wrong role) is a post-init update.

    Returns the reference's dict: offdiag_ss_post_init_writes,
    rr_rs_sr_post_init_writes, diag_ss_update_counts (sorted distinct per-box
    counts; a box with r = 0 or k = 0 receives the reference's vacuous update,
    counted once), diag_ss_blocks, plus in_place_factor_writes,
    uninitialized_slabs and initialized_twice (structure checks)."""
    import bisect

    regions = sorted(regions)
    starts = [g[0] for g in regions]
    hits = {}                                   # (region index, slab) -> list of roles
    pieces = {}                                 # (region index, slab) -> transform rectangles

    def hit(g, slab, role, box=None):
        hits.setdefault((g, slab), []).append(role)
        if role == "transform" and box is not None:
            pieces.setdefault((g, slab), []).append(box)

    def rect(g, r0, c0, rows, cols, role):
        _, nr, nc, rs, cs, _ = regions[g]
        r1, c1 = min(r0 + rows, nr), min(c0 + cols, nc)
        if r0 < rs and c0 < cs:
            hit(g, "rr", role, (r0, c0, min(r1, rs), min(c1, cs)))
        if r0 < rs and c1 > cs:
            hit(g, "rs", role, (r0, max(c0, cs), min(r1, rs), c1))
        if r1 > rs and c0 < cs:
            hit(g, "sr", role, (max(r0, rs), c0, r1, min(c1, cs)))
        if r1 > rs and c1 > cs:
            hit(g, "ss", role, (max(r0, rs), max(c0, cs), r1, c1))

    def overlapping(boxes):
        for a in range(len(boxes)):
            for b in range(a + 1, len(boxes)):
                p, q = boxes[a], boxes[b]
                if p[0] < q[2] and q[0] < p[2] and p[1] < q[3] and q[1] < p[3]:
                    return True
        return False

    for (_, role, ptr, rows, cols, ld, lower) in writes:
        if rows <= 0 or cols <= 0:
            continue
        g = bisect.bisect_right(starts, ptr) - 1
        if rows == 1 and cols == ld:            # flat copy: every region it overlaps, whole
            end = ptr + 8 * cols
            g = max(g, 0)
            while g < len(regions) and regions[g][0] < end:
                st, nr, nc = regions[g][0], regions[g][1], regions[g][2]
                if st + 8 * nr * nc > ptr:
                    rect(g, 0, 0, nr, nc, role)
                g += 1
            continue
        if g < 0:
            continue
        st, nr, nc = regions[g][0], regions[g][1], regions[g][2]
        off = (ptr - st) // 8
        if off >= nr * nc:
            continue                             # not a slab (scratch, factors, next level's inputs)
        if ld != nc:
            hit(g, "mismatched_ld", role)
            continue
        rect(g, off // nc, off % nc, rows, cols, role)

    offdiag_ss = rr_rs_sr = in_place = twice = 0
    uninit = []
    diag_counts = []
    for g, (_, nr, nc, rs, cs, key) in enumerate(regions):
        kind = key[0]
        for slab in ("rr", "rs", "sr", "ss", "mismatched_ld"):
            roles = hits.get((g, slab), [])
            init = sum(1 for x in roles if x == "transform")
            if init > 1 and not overlapping(pieces.get((g, slab), [])):
                init = 1       # one transform stored in disjoint pieces (edge-carved GEMM launches)
            post = [x for x in roles if x != "transform"]
            area = {"rr": rs * cs, "rs": rs * (nc - cs), "sr": (nr - rs) * cs, "ss": (nr - rs) * (nc - cs)}.get(slab, 1)
            if slab == "mismatched_ld":
                rr_rs_sr += len(roles)
                continue
            if init > 1:
                twice += 1
            if init == 0 and area > 0 and slab != "rs":     # RS_ij of the reference is never formed here
                uninit.append((slab,) + key[1:])
            if kind == "diag" and slab == "ss":
                # every writer counts (the SYRK is the one expected): an extra one shows as a count > 1
                diag_counts.append(len(post) + (1 if (rs == 0 or nr == rs) else 0))
                continue
            if kind == "off" and slab == "ss":
                offdiag_ss += len(post)
                continue
            if kind == "diag" and slab in ("rr", "sr"):
                in_place += sum(1 for x in post if x == "factor")
                rr_rs_sr += sum(1 for x in post if x != "factor")
                continue
            rr_rs_sr += len(post)
    return {"offdiag_ss_post_init_writes": offdiag_ss, "rr_rs_sr_post_init_writes": rr_rs_sr,
            "diag_ss_update_counts": sorted(set(diag_counts)), "diag_ss_blocks": len(diag_counts),
            "in_place_factor_writes": in_place, "uninitialized_slabs": len(uninit),
            "initialized_twice": twice}


def flop_report(levels, root_dim):
    """The reference's flop dict from box dimensions alone.

    levels: {l: (n array, k array, sorted near pairs i > j)}.  Phases and op
    order as issued by ulv_factor.factorize (ulv_factor.py:189-313); padded
    counts follow plan_batches (dense_core.py:229-248).
    """
    fl = PhaseFlops()
    for l in sorted(levels, reverse=True):
        n, k, offp = levels[l]
        r = np.asarray(n) - np.asarray(k)
        nb = len(n)
        fl.record(l, "diag_mul1", [("multiply", (n[i], n[i], n[i])) for i in range(nb)])
        fl.record(l, "diag_mul2", [("multiply", (n[i], n[i], n[i])) for i in range(nb)])
        fl.record(l, "diag_chol", [("cholesky", (r[i],)) for i in range(nb)])
        fl.record(l, "diag_trsm", [op for i in range(nb)
                                   for op in (("tri_solve", (r[i], k[i])), ("tri_solve", (r[i], n[i])))])
        fl.record(l, "diag_schur", [("multiply", (k[i], k[i], r[i])) for i in range(nb)])
        fl.record(l, "off_mul1", [("multiply", (n[i], n[j], n[j])) for (i, j) in offp])
        fl.record(l, "off_mul2", [("multiply", (n[i], n[j], n[i])) for (i, j) in offp])
        fl.record(l, "off_mirror", [("tri_solve", (r[i], k[j])) for (i, j) in offp])
    fl.record(0, "root", [("cholesky", (root_dim,))])
    return fl.flops


_PLAN_CACHE = {}       # structure signature -> (DeviceH2, FactorPlan, weakref to the live factors' lease)


class _Lease:
    """Held (strongly) by a ULVFactors and by every view into its HBM buffers
    (level maps, retained slabs, BlockVectors through the factors); the plan
    cache holds it weakly.  It references nothing itself, so dropping the
    factors and all views frees it at once (no reference cycle waiting for
    the garbage collector) and the next factorization of the same structure
    reuses the buffers, while a surviving view keeps them reserved."""
    __slots__ = ("__weakref__",)
_PLAN_CACHE_MAX = 2


def clear_cache():
    """Drop the cached device layouts / factorization programs."""
    _PLAN_CACHE.clear()


def _cached_plan(h2):
    """DeviceH2 + FactorPlan for h2, reusing the program and HBM buffers of an
    earlier factorization with the same structure (dims + interaction lists)
    once no live ULVFactors references them.  The numeric upload is redone
    every call; only the symbolic part (layout, descriptors, CUDA graph) is
    reused — the symbolic/numeric split of a direct solver."""
    own = getattr(h2, "_device", None)
    if own is not None:  # operands already in HBM (GPU construct)
        key = ("dev", id(own))
        ent = _PLAN_CACHE.get(key)
        if ent is not None and ent[0] is own and (ent[2] is None or ent[2]() is None):
            return ent[0], ent[1]
        plan = FactorPlan(own, h2.lists)
        _remember(key, own, plan)
        return own, plan
    if h2.tree.depth == 0:
        dh2 = DeviceH2.from_host(h2)
        return dh2, FactorPlan(dh2, h2.lists)
    levels = DeviceH2.layouts_from_host(h2)
    from .h2_device import _signature

    arena = getattr(h2, "_arena", None)
    wy = tuple(getattr(arena, "wy_levels", ())) if arena is not None and arena.intact(h2) else ()
    key = ("host", _signature(h2.tree.depth, h2.count, levels), wy)
    ent = _PLAN_CACHE.get(key)
    if ent is not None and (ent[2] is None or ent[2]() is None):
        dh2 = DeviceH2.from_host(h2, into=ent[0])
        return dh2, ent[1]
    dh2 = DeviceH2.from_host(h2)
    plan = FactorPlan(dh2, h2.lists)
    _remember(key, dh2, plan)
    return dh2, plan


def _remember(key, dh2, plan):
    if key not in _PLAN_CACHE and len(_PLAN_CACHE) >= _PLAN_CACHE_MAX:
        _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))
    _PLAN_CACHE[key] = (dh2, plan, None)


_UPLOAD_STREAM = {}


def _upload_stream(device):
    st = _UPLOAD_STREAM.get(device)
    if st is None:
        st = torch.cuda.Stream(device=device)
        _UPLOAD_STREAM[device] = st
    return st


def _factorize_streamed(h2):
    """Host-resident H2 (the reference's numpy data model): the upload runs level
    by level from the leaves up on a copy stream, and each level's factorization
    segment is queued as soon as its operands are in flight, so the GPU factors
    level l while the host gathers and copies the levels above.  The symbolic
    part (layout, descriptors, per-level CUDA graphs) is cached per structure."""
    from .h2_device import _signature

    arena = getattr(h2, "_arena", None)
    if arena is not None and arena.intact(h2):   # a to_pinned_host matrix carries its signature
        key = ("stream", arena.signature)
    else:
        key = ("stream", _signature(h2.tree.depth, h2.count, DeviceH2.layouts_from_host(h2)))
    ent = _PLAN_CACHE.get(key)
    if ent is not None and (ent[2] is None or ent[2]() is None):
        dh2, plan = ent[0], ent[1]
    else:
        dh2 = DeviceH2.allocate_for_host(h2)
        plan = FactorPlan(dh2, h2.lists, level_cuts=True)
        plan.capture()
        _remember(key, dh2, plan)
    cur = torch.cuda.current_stream(dh2.device)
    cur.wait_stream(_upload_stream(dh2.device))
    # a cached solve plan of this structure (w = 1, parallel: what solve(f, b) uses): its
    # per-factorization prepare runs level by level right behind the factorization, on a side
    # stream, hidden under the upload of the levels above
    sp = plan.__dict__.get("_solve_plans", {}).get((1, "parallel"))
    post = None
    if sp is not None:
        side = _prepare_stream(dh2.device)
        side.wait_stream(cur)

        def post(l):
            ev = torch.cuda.Event()
            ev.record(cur)
            side.wait_event(ev)
            sp.prepare_level[l].launch(side)
    on_level, finish = plan.launch_streamed(post)
    DeviceH2.from_host(h2, into=dh2, on_level=on_level, stream=_upload_stream(dh2.device))
    finish()
    if sp is not None:
        cur.wait_stream(side)
        sp._prepared = plan.generation
    return dh2, plan


_PREPARE_STREAM = {}


def _prepare_stream(device):
    st = _PREPARE_STREAM.get(device)
    if st is None:
        st = torch.cuda.Stream(device=device)
        _PREPARE_STREAM[device] = st
    return st


@ranged("h2ulv.factorize")
def factorize(h2, batched=True, retain=False):
    """Factor the hierarchy on the GPU; same contract as ulv_factor.py:154.  Runs on
    the device holding a GPU-built H² (else the current device)."""
    nat.lib()
    own = getattr(h2, "_device", None)
    with torch.cuda.device(own.device if own is not None else torch.cuda.current_device()):
        return _factorize(h2, retain)


def _factorize(h2, retain):
    if getattr(h2, "_device", None) is None and h2.tree.depth > 0:
        dh2, plan = _factorize_streamed(h2)
    else:
        dh2, plan = _cached_plan(h2)
        plan.capture()
        plan.run()
    plan.check_pivots()
    f = factors_from_plan(h2, plan)
    if retain:
        f.retained = _retained_views(plan)
        f.retained._owner = f._lease
    for key, ent in list(_PLAN_CACHE.items()):
        if ent[1] is plan:
            _PLAN_CACHE[key] = (ent[0], ent[1], weakref.ref(f._lease))
    return f


def _retained_views(plan):
    """`factors.retained` of factorize(..., retain=True) (ulv_factor.py:161-162,
    210-214, 273-279): the sparsified blocks Q_i^T A_ij Q_j (i >= j near) split
    into rr / rs / sr / ss0, before any elimination.  The level's near blocks
    A_ij and bases stay in HBM after the factorization, so the slabs are formed
    on access (one device GEMM pair per block) instead of being copied eagerly;
    the values are the same."""
    keys, src = [], {}
    for l, B in plan.bufs.items():
        lay = B.lay
        for (i, j) in lay.near_pairs:
            for part in ("rr", "rs", "sr", "ss0"):
                keys.append((part, l, i, j))
            src[(l, i, j)] = B
    cache = {}

    def block(l, i, j):
        if (l, i, j) not in cache:
            B = src[(l, i, j)]
            lay = B.lay
            n = lay.n
            q = plan.dh2.q[l]
            qi = q[int(lay.qoff[i]): int(lay.qoff[i] + n[i] * n[i])].view(int(n[i]), int(n[i]))
            qj = q[int(lay.qoff[j]): int(lay.qoff[j] + n[j] * n[j])].view(int(n[j]), int(n[j]))
            off = int(B.aoff[(i, j)])
            a = B.a[off: off + int(n[i] * n[j])].view(int(n[i]), int(n[j]))
            if i == j:   # only the lower triangle of a merged diagonal block is maintained
                a = torch.tril(a) + torch.tril(a, -1).T
            cache[(l, i, j)] = (qi.T @ a @ qj).cpu().numpy()
        return cache[(l, i, j)]

    def fetch(key):
        part, l, i, j = key
        h = block(l, i, j)
        lay = plan.bufs[l].lay
        ri, rj = int(lay.r[i]), int(lay.r[j])
        return {"rr": h[:ri, :rj], "rs": h[:ri, rj:], "sr": h[ri:, :rj], "ss0": h[ri:, rj:]}[part].copy()

    return _LazyBlocks(keys, fetch)


def factors_from_plan(h2, plan):
    f = ULVFactors(h2, plan)
    f._lease = _Lease()
    for l in range(plan.depth, 0, -1):
        lvl = plan.level_views(l)
        # the lazy views read the plan's HBM buffers: they hold the lease, so the plan
        # cache (weakref to the lease) never hands those buffers to a new factorization
        for m in (lvl.lr_diag, lvl.lr_off, lvl.ls, lvl.v):
            m._owner = f._lease
        f.levels[l] = lvl
    mm = plan.__dict__.get("_merge_map")
    if mm is None:
        mm = plan._merge_map = {l: {(pi, pj): [(2 * pi + a, 2 * pj + b) for a in (0, 1) for b in (0, 1)]
                                    for (pi, pj) in parents} for l, parents in plan.merge_pairs.items()}
    for l, m in mm.items():
        f.merge_map[l] = dict(m)      # per-factors dicts; the child lists are the plan's (read-only by contract)
    return f


def h2_device_of(h2):
    """The DeviceH2 of `h2`: the cached one (GPU construct) or a fresh upload."""
    dh2 = getattr(h2, "_device", None)
    if dh2 is None:
        dh2 = DeviceH2.from_host(h2)
    return dh2


# --------------------------------------------------------------------------- single-box API (ulv_factor.py:70-132)
from .block_engine import factor_diag, merge_level, sparsify_diag, sparsify_off  # noqa: E402,F401


def inject_couplings(h2, level, ss_sink):
    """Assign the far-pair couplings S_ij (i > j) into their SS slots
    (ulv_factor.py:108-112).  The factorization itself places them on the
    device with the merge's block copy (FactorPlan._merge_steps)."""
    for (i, j) in h2.lists.far[level]:
        if i > j:
            ss_sink((i, j), h2.coupling(level, i, j))
