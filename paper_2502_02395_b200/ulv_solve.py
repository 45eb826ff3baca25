"""Forward/backward substitution through the GPU ULV factors — drop-in for
`h2ulv.ulv_solve` (ulv_solve.py:1-207).

`solve(factors, b, mode="parallel")` permutes b into tree order, runs the
forward sweep (levels fine -> coarse, then the root) and the backward sweep
(root, then coarse -> fine) and permutes back.  The "parallel" form
(ulv_solve.py:98-109, 166-176) is what runs: every phase of a level is one
batched launch over all boxes, so a level costs 5 launches forward and 5
backward independent of the box count.  "naive" (the sequential Algorithm 3
of the reference) is executed box by box with the same kernels.

Vectors live in HBM in split layout per level: all redundant segments
(y_R) back to back, all skeleton segments (b_S) back to back.  The skeleton
segments of level l, concatenated in box order, are exactly the input
segments of level l-1 (n_p = k_2p + k_2p+1), so the merge
`segs[p] = vstack(b_S,2p, b_S,2p+1)` (ulv_solve.py:113) costs nothing.
"""

import os
from dataclasses import dataclass, field

import numpy as np
import torch

from .trace import ranged
from . import _native as nat
from .program import Program

# grouped GEMVs with fewer 64-row chunks than this are split over their terms
# (Program.gemv balance): the upper levels' few outputs with many neighbour terms
GEMV_BALANCE = int(os.environ.get("H2G_GEMV_BALANCE", "592"))
# levels whose transform kernels would launch fewer CTAs than this run them as balanced GEMVs
XFORM_MIN_CTAS = int(os.environ.get("H2G_XFORM_MIN_CTAS", "592"))
# levels with at most this many boxes solve with explicit triangular inverses (see SolvePlan.winv)
WINV_MAX_BOXES = int(os.environ.get("H2G_SOLVE_WINV_MAX_BOXES", "128"))

F64 = torch.float64


@dataclass
class BlockVector:
    """Per-level redundant segments plus the root segment (ulv_solve.py:18-25)."""

    yr: dict = field(default_factory=dict)
    root: np.ndarray = None
    width: int = 1
    vector: bool = True
    _plan: object = None
    _owner: object = None     # the ULVFactors it came from (keeps their HBM buffers reserved)


def _near_sets(lay):
    nb = lay.nb
    below = [[] for _ in range(nb)]
    above = [[] for _ in range(nb)]
    for (i, j) in lay.off_pairs:
        below[i].append(j)
        above[j].append(i)
    return [sorted(x) for x in below], [sorted(x) for x in above]


class SolvePlan:
    """Device vectors and the forward / backward programs for RHS width w."""

    def __init__(self, fplan, w, mode="parallel"):
        self.fp = fplan
        self.w = w
        self.mode = mode
        dev = fplan.device
        self.device = dev
        depth = fplan.depth
        dh2 = fplan.dh2
        self.count = dh2.count
        z = lambda m: torch.zeros(max(int(m), 1) * w, dtype=F64, device=dev)
        self.xin = z(self.count)
        d = fplan.root_dim
        self.yroot, self.xroot = z(d), z(d)
        self.v = {}
        for l in range(depth, 0, -1):
            lay = fplan.bufs[l].lay
            sr, sk, sn = int(lay.r.sum()), int(lay.k.sum()), int(lay.n.sum())
            self.v[l] = dict(BR=z(sr), BS=z(sk), Z=z(sr), Y=z(sr), YB=z(sr), Z2=z(sr), XR=z(sr), FULL=z(sn),
                             offR=np.concatenate([[0], np.cumsum(lay.r)[:-1]]).astype(np.int64),
                             offS=np.concatenate([[0], np.cumsum(lay.k)[:-1]]).astype(np.int64),
                             offX=np.concatenate([[0], np.cumsum(lay.n)[:-1]]).astype(np.int64))
        self.dist = fplan.part is not None and fplan.part.p > 1
        # The stored V_i = q_red L_ii^-T (ulv_factor.py:31) folds triangular solves into the
        # basis transforms: backward B3 q_red L_ii^-T t + q_skel x_S = [V_i | q_skel] [t; x_S]
        # on every level, and on levels whose boxes have no near neighbour (every third level
        # of a cube tree, the N = 1M leaf among them) forward P1 z_i = V_i^T b_i = y_i too, so
        # such a level has no TRSV at all.  The prepare step puts q_skel next to V_i in R.
        self.use_v = mode == "parallel" and fplan.has_v
        # (neighbour-free levels are the same computation in both modes — there is no chain to
        # order — so naive and parallel share the fused form and agree bit for bit, e.g. on
        # HSS trees, test_ulv_solve.py:90-96)
        self.fused = {l: fplan.has_v and not fplan.bufs[l].lay.off_pairs for l in range(depth, 0, -1)}
        # levels with few boxes: a one-CTA-per-box TRSV is a long serial chain on a few SMs, so
        # they get explicit Wt_i = L_ii^-T (from the stored L, in the prepare step) and every
        # triangular solve becomes a balanced GEMV
        self.winv = {}
        for l in range(depth, 0, -1):
            lay = fplan.bufs[l].lay
            mine = fplan.mine(l)
            nbox = int(sum(1 for i in range(lay.nb) if mine[i] and lay.r[i] > 0))
            self.winv[l] = self.use_v and not self.fused[l] and 0 < nbox <= WINV_MAX_BOXES
        self._build_prepare()
        self._segs = []
        self._masks = {}
        self.fwd_segments = self._finish(self._build_forward())
        self.bwd_segments = self._finish(self._build_backward())
        self.fwd = self.fwd_segments[0] if len(self.fwd_segments) == 1 else None
        self.bwd = self.bwd_segments[0] if len(self.bwd_segments) == 1 else None
        self.output = self.v[depth]["FULL"] if depth >= 1 else self.xroot

    # -------------------------------------------------------------- triangular inverses
    def _build_prepare(self):
        """The inverses the substitution reads are formed from the stored factor
        blocks themselves, once per factorization (h2g_tri_inv: the 64 x 64
        diagonal blocks of every L(r)_ii; the root's explicit W = L_00^-T by
        the row solve of the identity), not taken from the Cholesky's own
        by-products.  The solve is then a pure function of the factor blocks
        (lr_diag, lr_off, ls, v, root; ulv_factor.py:27-43) — like the
        reference's — so factors read back from storage solve to the same bits
        (test_storage.py:90-98).

        One program with the levels on separate lanes (they are independent; the
        root's latency-bound inverse chain alone on lane 0), plus the same steps
        as one program per level (`prepare_level[l]`, l = 0 the root) that a
        streamed factorization queues right behind each level (ulv_factor.
        _factorize_streamed), hidden under the upload of the levels above."""
        dev = self.device
        self._tri_status = torch.full((1,), 2 ** 31 - 1, dtype=torch.int32, device=dev)
        self.linv, self.loff, self.wt, self.mblk = {}, {}, {}, {}
        prog = Program(dev)
        levels = [0] + list(range(self.fp.depth, 0, -1))
        for l in levels:
            prog.lane = 0 if l == 0 else 1 + (self.fp.depth - l) % 4
            self._emit_prepare(prog, l, alloc=True)
        prog.lane = 0
        self.prepare = prog.finalize()
        self.prepare.capture()
        self.prepare_level = {}
        for l in levels:
            pl = Program(dev)
            self._emit_prepare(pl, l, alloc=False)
            self.prepare_level[l] = pl.finalize()
        self._prepared = None

    def _emit_prepare(self, prog, l, alloc):
        """The prepare steps of level l (l = 0: the root) into `prog`; `alloc` creates the
        buffers they write, otherwise the ones a first call created are reused."""
        fp = self.fp
        dev = self.device
        W = nat.PANEL_WIDTH
        if l == 0:
            d = fp.root_dim
            nb0 = -(-d // W)
            if alloc:
                self.root_linv = torch.zeros(max(nb0, 1) * W * W, dtype=F64, device=dev)
                self.root_w = torch.zeros(max(d * d, 1), dtype=F64, device=dev)
            rp = fp.root_buf.data_ptr()
            prog.triinv([(rp, self.root_linv.data_ptr(), d, d, 0)], self._tri_status.data_ptr())
            prog.trsm_rows([(rp, 0, self.root_w.data_ptr(), self.root_linv.data_ptr(), d, d, 0, nb0, d, d)])
            return
        B = fp.bufs[l]
        lay = B.lay
        nblk = -(-np.asarray(lay.r, dtype=np.int64) // W)
        loff = np.concatenate([[0], np.cumsum(nblk)[:-1]]).astype(np.int64)
        mine = self._mine(l)
        lt = None
        if self.fused[l]:
            # no TRSV reads a fused level's inverses (both modes transform only): just the
            # zero-diagonal check that raises SingularTriangularError
            if alloc:
                self.linv[l], self.loff[l] = None, loff
            prog.triinv([(B.H.data_ptr() + 8 * int(lay.qoff[i]), 0, int(lay.r[i]), int(lay.n[i]), 0)
                         for i in range(lay.nb) if mine[i] and lay.r[i] > 0], self._tri_status.data_ptr())
        else:
            if alloc:
                self.linv[l] = torch.zeros(max(int(nblk.sum()), 1) * W * W, dtype=F64, device=dev)
                self.loff[l] = loff
            lt = self.linv[l]
            prog.triinv([(B.H.data_ptr() + 8 * int(lay.qoff[i]), lt.data_ptr() + 8 * int(loff[i]) * W * W,
                          int(lay.r[i]), int(lay.n[i]), 0) for i in range(lay.nb) if mine[i] and lay.r[i] > 0],
                        self._tri_status.data_ptr())
        if self.winv[l]:
            roff = np.concatenate([[0], np.cumsum(np.asarray(lay.r, dtype=np.int64) ** 2)[:-1]])
            if alloc:
                wt_ = torch.zeros(max(int((np.asarray(lay.r, dtype=np.int64) ** 2).sum()), 1), dtype=F64, device=dev)
                self.wt[l] = (wt_, roff)
            wt = self.wt[l][0]
            prog.trsm_rows([(B.H.data_ptr() + 8 * int(lay.qoff[i]), 0, wt.data_ptr() + 8 * int(roff[i]),
                             lt.data_ptr() + 8 * int(loff[i]) * W * W, int(lay.r[i]), int(lay.r[i]), 0,
                             int(nblk[i]), int(lay.n[i]), int(lay.r[i]))
                            for i in range(lay.nb) if mine[i] and lay.r[i] > 0])
            if not self.dist:
                # M_ij = L_ii^-1 L(r)_ij (i > j near): P2+P3 become y_i = z_i - sum_j M_ij z_j
                # and B2' x_R-terms t_i = y_i - sum_j M_ji^T y_j — one GEMV each, no TRSV
                pairs = [(i, j) for (i, j) in lay.off_pairs if lay.r[i] > 0 and lay.r[j] > 0]
                if alloc:
                    moff, acc = {}, 0
                    for (i, j) in pairs:
                        moff[(i, j)] = acc
                        acc += int(lay.r[i]) * int(lay.r[j])
                    self.mblk[l] = (torch.zeros(max(acc, 1), dtype=F64, device=dev), moff)
                mt, moff = self.mblk[l]
                prog.gemm(1, 0, [(wt.data_ptr() + 8 * int(roff[i]), B.T.ptr(B.toff[(i, j)]),
                                  mt.data_ptr() + 8 * moff[(i, j)], int(lay.r[i]), int(lay.r[j]), int(lay.r[i]),
                                  int(lay.r[i]), int(lay.n[j]), int(lay.r[j]), 0, 1.0, 0.0) for (i, j) in pairs])
        if self.use_v or self.fused[l]:
            # R_i = [V_i | q_skel_i]: the spare columns of V's n x n slot take q_skel
            q = fp.dh2.q[l]
            prog.copy([(q.data_ptr() + 8 * int(lay.qoff[i] + lay.r[i]), B.R.ptr(int(lay.qoff[i] + lay.r[i])),
                        int(lay.n[i]), int(lay.k[i]), int(lay.n[i]), int(lay.n[i]), 0)
                       for i in range(lay.nb) if mine[i] and lay.k[i] > 0])
            if self.fused[l]:
                # no near neighbours: L(s)_ii is the only L(s) block of box i, so P4
                # (b_S -= L(s)_ii y) and B1 (y_R -= L(s)_ii^T x_S) fold into the transforms
                # through q_skel~ = q_skel - V_i L(s)_ii^T:  b_S - L(s) V^T b = q_skel~^T b,
                # V (y - L(s)^T x_S) + q_skel x_S = V y + q_skel~ x_S
                gm = []
                for i in range(lay.nb):
                    ni, ri, ki = int(lay.n[i]), int(lay.r[i]), int(lay.k[i])
                    if mine[i] and ri > 0 and ki > 0:
                        o = int(lay.qoff[i])
                        gm.append((B.R.ptr(o), B.H.data_ptr() + 8 * (o + ri * ni), B.R.ptr(o + ri),
                                   ni, ki, ri, ni, ni, ni, 0, -1.0, 1.0))
                prog.gemm(0, 1, gm)

    def ensure_prepared(self, stream=None):
        """Run the inverse program if the factors changed since the last solve."""
        gen = self.fp.generation
        if self._prepared != gen:
            self.prepare.launch(stream)
            self._prepared = gen

    # -------------------------------------------------------------- distribution
    def _mine(self, l):
        return self.fp.mine(l) if l >= 1 else np.ones(1, dtype=bool)

    def _cut(self, prog, tag):
        """End the current program segment; `tag` = (vector, level, offsets key)
        is all-reduced across ranks (owned segments only) before the next one."""
        if not self.dist:
            return prog
        self._segs.append(prog.finalize())
        self._segs.append(tag)
        return Program(self.device)

    def _finish(self, prog):
        segs = self._segs + [prog.finalize()]
        self._segs = []
        return segs

    def _mask(self, l, offkey):
        """0/1 row mask (x w columns) of the segments this rank contributes to the sum of a
        level-l vector (one member per box's process group: the masked all-reduce leaves every
        rank with the complete vector)."""
        key = (l, offkey)
        if key not in self._masks:
            lay = self.fp.bufs[l].lay
            sizes = {"offR": lay.r, "offS": lay.k, "offX": lay.n}[offkey]
            mine = self.fp.part.contrib_mask(l, self.fp.comm.rank)
            m = np.repeat(mine.astype(np.float64), np.asarray(sizes, dtype=np.int64))
            self._masks[key] = torch.from_numpy(np.repeat(m, self.w)).to(self.device)
        return self._masks[key]

    def _run_segments(self, segs, stream=None):
        for seg in segs:
            if isinstance(seg, Program):
                seg.launch(stream)
                continue
            name, l, offkey = seg
            vec = self.v[l][name]
            m = self._mask(l, offkey)
            vec[:m.numel()].mul_(m)
            if name == "BS" and l - 1 < self.fp.part.L0:
                # merge into the group-computed parent level: one AllReduce per parent box over
                # its process group, 8 d w bytes — simulate_solve's merge events (comm_sim.py:138-147)
                self._merge_reduce(vec, l)
            else:
                self.fp.comm.all_reduce_(vec[:m.numel()], phase="solve", level=l)

    def _merge_reduce(self, vec, l):
        part, comm, w = self.fp.part, self.fp.comm, self.w
        lay = self.fp.bufs[l].lay
        offS = self.v[l]["offS"]
        for pbox in range(2 ** (l - 1)):
            g = part.group(l - 1, pbox)
            if g[1] - g[0] < 2:
                continue
            a, b = int(offS[2 * pbox]) * w, (int(offS[2 * pbox + 1]) + int(lay.k[2 * pbox + 1])) * w
            comm.group_all_reduce_(vec[a:b], g, phase="forward", level=l - 1)

    # -------------------------------------------------------------- pointers
    def _p(self, t, off_rows=0):
        return t.data_ptr() + 8 * int(off_rows) * self.w

    def _ls(self, l, a, b):
        """(pointer, ld) of L(s)_ab at level l."""
        B = self.fp.bufs[l]
        lay = B.lay
        n, r = lay.n, lay.r
        if a == b:
            return B.H.data_ptr() + 8 * int(lay.qoff[a] + r[a] * n[a]), int(n[a])
        if a > b:
            return B.T.ptr(B.toff[(a, b)]) + 8 * int(r[a] * n[b]), int(n[b])
        return B.LSm.ptr(B.lsoff[(b, a)]), int(r[b])

    def _ls_keys(self, lay):
        keys = [(i, i) for i in range(lay.nb)] + list(lay.off_pairs) + [(j, i) for (i, j) in lay.off_pairs]
        return [(a, b) for (a, b) in keys if lay.k[a] > 0 and lay.r[b] > 0]

    def _L(self, l, i):
        B = self.fp.bufs[l]
        return B.H.data_ptr() + 8 * int(B.lay.qoff[i]), int(B.lay.n[i])

    def _tr(self, l, i, x):
        """TRSV descriptor (L, Linv, x, n, ld) of box i at level l (l = 0: root)."""
        if l == 0:
            d = self.fp.root_dim
            return (self.fp.root_buf.data_ptr(), self.root_linv.data_ptr(), x, d, d)
        B = self.fp.bufs[l]
        lay = B.lay
        return (B.H.data_ptr() + 8 * int(lay.qoff[i]), self.linv[l].data_ptr() + 8 * int(self.loff[l][i]) * 4096, x,
                int(lay.r[i]), int(lay.n[i]))

    def _root_solve(self, prog, y, x, trans):
        """y = L_00^-1 x (trans 0) or L_00^-T x (trans 1) with the root's explicit
        W = L_00^-T from the factorization: one grouped GEMV instead of a TRSV."""
        d = self.fp.root_dim
        wp = self.root_w.data_ptr()
        prog.gemv([(y.data_ptr(), 0, 0, d, 0, nat.GEMV_PLUS, [(wp, x.data_ptr(), d, 1 - trans, d)])], self.w)

    # -------------------------------------------------------------- forward
    def _build_forward(self):
        fp, w = self.fp, self.w
        prog = Program(self.device)
        depth = fp.depth
        if depth == 0:
            d = fp.root_dim
            self._root_solve(prog, self.yroot, self.xin, 0)
            return prog
        xin = self.xin
        for l in range(depth, 0, -1):
            V = self.v[l]
            lay = fp.bufs[l].lay
            n, k, r, nb = lay.n, lay.k, lay.r, lay.nb
            offR, offS, offX = V["offR"], V["offS"], V["offX"]
            below, _ = _near_sets(lay)
            q = fp.dh2.q[l]
            mine = self._mine(l)
            if self.fused[l]:
                # G1 + P1-P4 of a level without near neighbours: [y_R; b_S] = [V | q_skel~]^T seg
                R = fp.bufs[l].R
                self._xform_t(prog, [(R.ptr(int(lay.qoff[i])), self._p(xin, offX[i]), self._p(V["Y"], offR[i]),
                               self._p(V["BS"], offS[i]), int(n[i]), int(r[i]), int(n[i]))
                              for i in range(nb) if mine[i]], w)
                if self.dist:
                    prog = self._cut(prog, ("Y", l, "offR"))
                # (P4 is in the transform: R carries q_skel~, see _build_prepare)
                if self.dist and l - 1 < fp.part.L0:
                    prog = self._cut(prog, ("BS", l, "offS"))
                xin = V["BS"]
                continue
            if self.use_v:
                # G1 + P1: [z; b_S] = [V | q_skel]^T seg  (z_i = L_ii^-1 q_red^T seg_i)
                R = fp.bufs[l].R
                self._xform_t(prog, [(R.ptr(int(lay.qoff[i])), self._p(xin, offX[i]), self._p(V["Z"], offR[i]),
                               self._p(V["BS"], offS[i]), int(n[i]), int(r[i]), int(n[i]))
                              for i in range(nb) if mine[i]], w)
                prog = self._forward_parallel_level_v(prog, l, V, lay, below)
                if self.dist and l - 1 < fp.part.L0:
                    prog = self._cut(prog, ("BS", l, "offS"))
                xin = V["BS"]
                continue
            # G1: [b_R; b_S] = q_full^T seg   (_transform_in, ulv_solve.py:33-41)
            self._xform_t(prog, [(q.data_ptr() + 8 * int(lay.qoff[i]), self._p(xin, offX[i]), self._p(V["BR"], offR[i]),
                           self._p(V["BS"], offS[i]), int(n[i]), int(r[i]), int(n[i])) for i in range(nb) if mine[i]], w)
            if self.mode == "parallel":
                prog = self._forward_parallel_level(prog, l, V, lay, below)
            else:
                self._forward_naive_level(prog, l, V, lay)
            if self.dist and l - 1 < fp.part.L0:
                prog = self._cut(prog, ("BS", l, "offS"))   # the parent level is group-computed
            xin = V["BS"]
        d = fp.root_dim
        self._root_solve(prog, self.yroot, xin, 0)
        return prog

    def _forward_parallel_level(self, prog, l, V, lay, below):
        w = self.w
        n, k, r, nb = lay.n, lay.k, lay.r, lay.nb
        offR, offS = V["offR"], V["offS"]
        B = self.fp.bufs[l]
        mine = self._mine(l)
        dist = self.dist
        # P1  z_i = L_ii^-1 b_R,i
        prog.memcpy(V["Z"].data_ptr(), V["BR"].data_ptr(), 8 * int(r.sum()) * w)
        prog.trsv([self._tr(l, i, self._p(V["Z"], offR[i])) for i in range(nb) if mine[i]], 0, w)
        if dist:
            prog = self._cut(prog, ("Z", l, "offR"))
        # P2  t_i = b_R,i - sum_{j<i near} L(r)_ij z_j ;  P3  y_i = L_ii^-1 t_i.
        # A box without lower near neighbours has t_i = b_R,i, so y_i = z_i (the same
        # TRSV on the same input): Y starts as a copy of Z and P2 / P3 run only for the
        # boxes with neighbours (none at a cube-shaped leaf level).
        prog.memcpy(V["Y"].data_ptr(), V["Z"].data_ptr(), 8 * int(r.sum()) * w)
        nbr = [i for i in range(nb) if mine[i] and any(r[j] > 0 for j in below[i])]
        outs = []
        for i in nbr:
            terms = [(B.T.ptr(B.toff[(i, j)]), self._p(V["Z"], offR[j]), int(n[j]), 0, int(r[j]))
                     for j in below[i] if r[j] > 0]
            outs.append((self._p(V["Y"], offR[i]), 0, self._p(V["BR"], offR[i]), int(r[i]), 0, 0, terms))
        prog.gemv(outs, w, balance=GEMV_BALANCE)
        prog.trsv([self._tr(l, i, self._p(V["Y"], offR[i])) for i in nbr], 0, w)
        if dist:
            prog = self._cut(prog, ("Y", l, "offR"))
        # P4  b_S,a -= sum_b L(s)_ab y_b
        self._ls_update_forward(prog, l, V, lay, owned=mine)
        return prog

    def _xform_t(self, prog, descs, w):
        """[y1; y2] = Q^T x per box: the column-chunked transform kernel when the level
        fills the GPU, else a balanced grouped GEMV (SPLIT rows r | k) whose rows (the K
        axis) are spread over many CTAs — the upper levels' few large boxes."""
        descs = [d for d in descs if d[4] > 0]
        if sum(-(-int(d[4]) // 128) for d in descs) >= XFORM_MIN_CTAS:
            prog.xform_t(descs, w)
            return
        prog.gemv([(y1, y2, 0, n, split, nat.GEMV_PLUS | nat.GEMV_SPLIT, [(q, x, ldq, 1, n)])
                   for (q, x, y1, y2, n, split, ldq) in descs], w, balance=GEMV_BALANCE)

    def _xform_n(self, prog, descs, w):
        """out = Q [xr; xs] per box (see _xform_t for the choice of kernel)."""
        descs = [d for d in descs if d[4] > 0]
        if sum(-(-int(d[4]) // 32) for d in descs) >= XFORM_MIN_CTAS:
            prog.xform_n(descs, w)
            return
        outs = []
        for (q, xr, xs, out, n, r, ldq) in descs:
            terms = ([(q, xr, ldq, 0, r)] if r > 0 else []) + ([(q + 8 * r, xs, ldq, 0, n - r)] if n > r else [])
            outs.append((out, 0, 0, n, 0, nat.GEMV_PLUS, terms))
        prog.gemv(outs, w, balance=GEMV_BALANCE)

    def _forward_parallel_level_v(self, prog, l, V, lay, below):
        """P1-P3 with Z = L^-1 b_R already formed through V (the transform):
        y_i = L_ii^-1 (b_R,i - u_i) = z_i - L_ii^-1 u_i, u_i = sum_{j<i near} L(r)_ij z_j,
        so only the boxes with lower near neighbours run a TRSV (on u_i)."""
        w = self.w
        n, r, nb = lay.n, lay.r, lay.nb
        offR = V["offR"]
        B = self.fp.bufs[l]
        mine = self._mine(l)
        if self.dist:
            prog = self._cut(prog, ("Z", l, "offR"))
        if l in self.mblk:
            # y_i = z_i - sum_{j<i near} M_ij z_j  (M_ij = L_ii^-1 L(r)_ij from the prepare step)
            mt, moff = self.mblk[l]
            prog.gemv([(self._p(V["Y"], offR[i]), 0, self._p(V["Z"], offR[i]), int(r[i]), 0, 0,
                        [(mt.data_ptr() + 8 * moff[(i, j)], self._p(V["Z"], offR[j]), int(r[j]), 0, int(r[j]))
                         for j in below[i] if r[j] > 0]) for i in range(nb) if mine[i] and r[i] > 0], w,
                      balance=GEMV_BALANCE)
            self._ls_update_forward(prog, l, V, lay, owned=mine)     # P4
            return prog
        prog.memcpy(V["Y"].data_ptr(), V["Z"].data_ptr(), 8 * int(r.sum()) * w)
        nbr = [i for i in range(nb) if mine[i] and any(r[j] > 0 for j in below[i])]
        if nbr:
            U = V["BR"]          # free on this path: holds u_i, then L_ii^-1 u_i
            prog.gemv([(self._p(U, offR[i]), 0, 0, int(r[i]), 0, nat.GEMV_PLUS,
                        [(B.T.ptr(B.toff[(i, j)]), self._p(V["Z"], offR[j]), int(n[j]), 0, int(r[j]))
                         for j in below[i] if r[j] > 0]) for i in nbr], w, balance=GEMV_BALANCE)
            if self.winv[l]:          # y_i = z_i - L_ii^-1 u_i = z_i - Wt_i^T u_i
                wt, roff = self.wt[l]
                prog.gemv([(self._p(V["Y"], offR[i]), 0, self._p(V["Z"], offR[i]), int(r[i]), 0, 0,
                            [(wt.data_ptr() + 8 * int(roff[i]), self._p(U, offR[i]), int(r[i]), 1, int(r[i]))])
                           for i in nbr], w, balance=GEMV_BALANCE)
            else:
                prog.trsv([self._tr(l, i, self._p(U, offR[i])) for i in nbr], 0, w)
                prog.gemv([(self._p(V["Y"], offR[i]), 0, self._p(V["Z"], offR[i]), int(r[i]), 0, 0,
                            [(0, self._p(U, offR[i]), 0, 0, int(r[i]))]) for i in nbr], w)
        if self.dist:
            prog = self._cut(prog, ("Y", l, "offR"))
        self._ls_update_forward(prog, l, V, lay, owned=mine)     # P4
        return prog

    def _ls_update_forward(self, prog, l, V, lay, only_b=None, owned=None):
        w = self.w
        offR, offS = V["offR"], V["offS"]
        terms = {}
        for (a, b) in self._ls_keys(lay):
            if only_b is not None and b != only_b:
                continue
            if owned is not None and not owned[a]:
                continue
            ptr, ld = self._ls(l, a, b)
            terms.setdefault(a, []).append((b, (ptr, self._p(V["Y"], offR[b]), ld, 0, int(lay.r[b]))))
        # terms in box order (a structural order: the summation order — hence the bits — must not
        # depend on where the buffers happen to live, so reloaded factors solve identically)
        outs = [(self._p(V["BS"], offS[a]), 0, self._p(V["BS"], offS[a]), int(lay.k[a]), 0, 0,
                 [tm for _, tm in sorted(t, key=lambda x: x[0])])
                for a, t in sorted(terms.items())]
        prog.gemv(outs, w, balance=GEMV_BALANCE)

    def _forward_naive_level(self, prog, l, V, lay):
        """Algorithm 3 order (ulv_solve.py:90-97): box by box."""
        w = self.w
        offR = V["offR"]
        B = self.fp.bufs[l]
        _, above = _near_sets(lay)
        prog.memcpy(V["Y"].data_ptr(), V["BR"].data_ptr(), 8 * int(lay.r.sum()) * w)
        for i in range(lay.nb):
            prog.trsv([self._tr(l, i, self._p(V["Y"], offR[i]))], 0, w)
            outs = []
            for j in above[i]:
                if lay.r[i] == 0 or lay.r[j] == 0:
                    continue
                outs.append((self._p(V["Y"], offR[j]), 0, self._p(V["Y"], offR[j]), int(lay.r[j]), 0, 0,
                             [(B.T.ptr(B.toff[(j, i)]), self._p(V["Y"], offR[i]), int(lay.n[i]), 0,
                               int(lay.r[i]))]))
            prog.gemv(outs, w, balance=GEMV_BALANCE)
            self._ls_update_forward(prog, l, V, lay, only_b=i)

    # -------------------------------------------------------------- backward
    def _build_backward(self):
        fp, w = self.fp, self.w
        prog = Program(self.device)
        depth = fp.depth
        d = fp.root_dim
        self._root_solve(prog, self.xroot, self.yroot, 1)
        xs = self.xroot
        for l in range(1, depth + 1):
            V = self.v[l]
            lay = fp.bufs[l].lay
            n, k, r, nb = lay.n, lay.k, lay.r, lay.nb
            offR, offS, offX = V["offR"], V["offS"], V["offX"]
            B = fp.bufs[l]
            mine = self._mine(l)
            dist = self.dist
            if dist and l >= 2:
                prog = self._cut(prog, ("FULL", l - 1, "offX"))   # x_S of neighbours computed elsewhere
            if self.fused[l]:
                # B1-B3 without near neighbours: full_i = [V_i | q_skel~_i] [y_R,i; x_S,i]
                self._xform_n(prog, [(B.R.ptr(int(lay.qoff[i])), self._p(V["Y"], offR[i]), self._p(xs, offS[i]),
                                      self._p(V["FULL"], offX[i]), int(n[i]), int(r[i]), int(n[i]))
                                     for i in range(nb) if mine[i]], w)
                xs = V["FULL"]
                continue
            # B1  y_R,i -= sum_a L(s)_ai^T x_S,a
            src = {}
            for (a, b) in self._ls_keys(lay):
                if not mine[b]:
                    continue          # the column box is computed elsewhere (its blocks may not be here)
                ptr, ld = self._ls(l, a, b)
                src.setdefault(b, []).append((a, (ptr, self._p(xs, offS[a]), ld, 1, int(k[a]))))
            outs = [(self._p(V["YB"], offR[i]), 0, self._p(V["Y"], offR[i]), int(r[i]), 0, 0,
                     [tm for _, tm in sorted(src.get(i, []), key=lambda x: x[0])])
                    for i in range(nb) if mine[i]]
            prog.gemv(outs, w, balance=GEMV_BALANCE)
            if self.mode == "parallel" and l in self.mblk:
                # t_i = y_i - sum_{j>i near} L(r)_ji^T L_jj^-T y_j = y_i - sum_j M_ji^T y_j
                _, above = _near_sets(lay)
                mt, moff = self.mblk[l]
                prog.gemv([(self._p(V["XR"], offR[i]), 0, self._p(V["YB"], offR[i]), int(r[i]), 0, 0,
                            [(mt.data_ptr() + 8 * moff[(j, i)], self._p(V["YB"], offR[j]), int(r[i]), 1, int(r[j]))
                             for j in above[i] if r[j] > 0]) for i in range(nb) if mine[i] and r[i] > 0], w,
                          balance=GEMV_BALANCE)
            elif self.mode == "parallel":
                _, above = _near_sets(lay)
                if self.winv[l]:      # z2_i = L_ii^-T y_i = Wt_i y_i
                    wt, roff = self.wt[l]
                    prog.gemv([(self._p(V["Z2"], offR[i]), 0, 0, int(r[i]), 0, nat.GEMV_PLUS,
                                [(wt.data_ptr() + 8 * int(roff[i]), self._p(V["YB"], offR[i]), int(r[i]), 0,
                                  int(r[i]))]) for i in range(nb) if mine[i] and r[i] > 0], w, balance=GEMV_BALANCE)
                else:
                    prog.memcpy(V["Z2"].data_ptr(), V["YB"].data_ptr(), 8 * int(r.sum()) * w)
                    prog.trsv([self._tr(l, i, self._p(V["Z2"], offR[i])) for i in range(nb) if mine[i]], 1, w)
                if dist:
                    prog = self._cut(prog, ("Z2", l, "offR"))
                # boxes without upper near neighbours: x_R,i = z2_i (same TRSV, same input);
                # with V, XR carries t_i = y_R,i instead (B3 applies L^-T through V)
                prog.memcpy(V["XR"].data_ptr(), (V["YB"] if self.use_v else V["Z2"]).data_ptr(),
                            8 * int(r.sum()) * w)
                nbr = [i for i in range(nb) if mine[i] and any(r[j] > 0 for j in above[i])]
                outs = []
                for i in nbr:
                    terms = [(B.T.ptr(B.toff[(j, i)]), self._p(V["Z2"], offR[j]), int(n[i]), 1,
                              int(r[j])) for j in above[i] if r[j] > 0]
                    outs.append((self._p(V["XR"], offR[i]), 0, self._p(V["YB"], offR[i]), int(r[i]), 0, 0, terms))
                prog.gemv(outs, w, balance=GEMV_BALANCE)
                if not self.use_v:
                    prog.trsv([self._tr(l, i, self._p(V["XR"], offR[i])) for i in nbr], 1, w)
            else:
                self._backward_naive_level(prog, l, V, lay)
            # B3  full_i = q_red x_R + q_skel x_S = q_full [x_R; x_S]; with the stored V_i
            # (use_v): x_R,i = L_ii^-T t_i, so q_red x_R,i = V_i t_i and full_i = [V_i | q_skel_i] [t_i; x_S,i]
            # — XR holds t_i (the second TRSV is not run)
            if self.use_v:
                qptr = {i: B.R.ptr(int(lay.qoff[i])) for i in range(nb) if mine[i]}
            else:
                qptr = {i: fp.dh2.q[l].data_ptr() + 8 * int(lay.qoff[i]) for i in range(nb) if mine[i]}
            self._xform_n(prog, [(qptr[i], self._p(V["XR"], offR[i]), self._p(xs, offS[i]),
                           self._p(V["FULL"], offX[i]), int(n[i]), int(r[i]), int(n[i]))
                          for i in range(nb) if mine[i]], w)
            xs = V["FULL"]
        if self.dist and depth >= 1:
            prog = self._cut(prog, ("FULL", depth, "offX"))     # assemble x on every rank
        return prog

    def _backward_naive_level(self, prog, l, V, lay):
        """ulv_solve.py:157-162: reversed box order."""
        w = self.w
        offR = V["offR"]
        B = self.fp.bufs[l]
        _, above = _near_sets(lay)
        prog.memcpy(V["XR"].data_ptr(), V["YB"].data_ptr(), 8 * int(lay.r.sum()) * w)
        for i in reversed(range(lay.nb)):
            terms = [(B.T.ptr(B.toff[(j, i)]), self._p(V["XR"], offR[j]), int(lay.n[i]), 1,
                      int(lay.r[j])) for j in above[i] if lay.r[j] > 0]
            if terms:
                prog.gemv([(self._p(V["XR"], offR[i]), 0, self._p(V["XR"], offR[i]), int(lay.r[i]), 0, 0, terms)], w)
            prog.trsv([self._tr(l, i, self._p(V["XR"], offR[i]))], 1, w)

    # -------------------------------------------------------------- run
    def run_forward(self, stream=None):
        self.ensure_prepared(stream)
        if self.fwd is not None:
            self.fwd.launch(stream)
        else:
            self._run_segments(self.fwd_segments, stream)

    def run_backward(self, stream=None):
        self.ensure_prepared(stream)
        if self.bwd is not None:
            self.bwd.launch(stream)
        else:
            self._run_segments(self.bwd_segments, stream)

    def block_vector(self, vector):
        bv = BlockVector(width=self.w, vector=vector, _plan=self)
        for l in range(self.fp.depth, 0, -1):
            V = self.v[l]
            lay = self.fp.bufs[l].lay
            y = V["Y"].view(-1, self.w)[:int(lay.r.sum())].cpu().numpy()   # one D2H per level
            for i in range(lay.nb):
                o = int(V["offR"][i])
                bv.yr[(l, i)] = y[o:o + int(lay.r[i])].copy()
        bv.root = self.yroot.view(-1, self.w)[:self.fp.root_dim].cpu().numpy()
        return bv


def _plan_for(factors, w, mode):
    """Solve programs live with the factorization program they read, so a
    re-factorization with a cached FactorPlan reuses them too."""
    from .ulv_factor import factor_plan_of

    fp = factor_plan_of(factors)
    cache = fp.__dict__.setdefault("_solve_plans", {})
    key = (w, mode)
    if key not in cache:
        sp = SolvePlan(fp, w, mode)
        for seg in sp.fwd_segments + sp.bwd_segments:
            if isinstance(seg, Program):
                seg.capture()
        cache[key] = sp
    return cache[key]


def _to_tree_order(factors, b):
    bm = np.asarray(b, dtype=np.float64)
    vector = bm.ndim == 1
    bm = bm.reshape(factors.h2.count, -1)
    return bm, vector


def forward_parallel(factors, b):
    return _forward(factors, b, "parallel")


def forward_naive(factors, b):
    return _forward(factors, b, "naive")


def _forward(factors, b, mode):
    """b in TREE order (as the reference's forward_* expect)."""
    nat.lib()
    bm, vector = _to_tree_order(factors, b)
    sp = _plan_for(factors, bm.shape[1], mode)
    sp.xin.view(-1, sp.w)[:factors.h2.count].copy_(torch.from_numpy(np.ascontiguousarray(bm)))
    sp.run_forward()
    bv = sp.block_vector(vector)
    bv._owner = factors
    return bv


def backward_parallel(factors, y):
    return _backward(factors, y, "parallel")


def backward_naive(factors, y):
    return _backward(factors, y, "naive")


def _backward(factors, y, mode):
    """The backward sweep is a pure function of `y` (ulv_solve.py:127-188): the
    host BlockVector is packed into the device layout and uploaded every call,
    so in-place edits of y.yr / y.root and an interleaved forward of another
    right-hand side cannot leak into the result."""
    nat.lib()
    sp = _plan_for(factors, y.width, mode)
    fp = sp.fp
    with torch.cuda.device(sp.device):
        for l in range(fp.depth, 0, -1):
            V = sp.v[l]
            lay = fp.bufs[l].lay
            host = np.empty((int(lay.r.sum()), sp.w), dtype=np.float64)
            for i in range(lay.nb):
                o = int(V["offR"][i])
                host[o:o + int(lay.r[i])] = np.asarray(y.yr[(l, i)], dtype=np.float64).reshape(-1, sp.w)
            V["Y"].view(-1, sp.w)[:host.shape[0]].copy_(torch.from_numpy(host))
        sp.yroot.view(-1, sp.w)[:fp.root_dim].copy_(
            torch.from_numpy(np.asarray(y.root, dtype=np.float64).reshape(-1, sp.w)))
        sp.run_backward()
        x = sp.output.view(-1, sp.w)[:factors.h2.count].cpu().numpy()
    return x[:, 0] if y.vector else x


@ranged("h2ulv.solve")
def solve(factors, b, mode="parallel"):
    """Solve A x = b with b in the ORIGINAL input order (ulv_solve.py:191-207)."""
    if mode not in ("naive", "parallel"):
        raise ValueError(f"unknown mode '{mode}'")
    nat.lib()
    bm = np.asarray(b, dtype=np.float64)
    vector = bm.ndim == 1
    bm = bm.reshape(factors.h2.count, -1)
    sp = _plan_for(factors, bm.shape[1], mode)
    with torch.cuda.device(sp.device):
        return _solve_on(factors, sp, bm, vector)


def _solve_on(factors, sp, bm, vector):
    dev = sp.device
    # the tree permutation is structure (like the cached plans): uploaded once per cloud / device
    cloud = factors.h2.cloud
    cached = cloud.__dict__.get("_perm_dev")
    if cached is not None and cached[0] is cloud.perm and cached[1].device == dev:
        perm = cached[1]
    else:
        perm = torch.from_numpy(np.asarray(cloud.perm, dtype=np.int64)).to(dev, non_blocking=True)
        try:
            cloud._perm_dev = (cloud.perm, perm)
        except AttributeError:   # a frozen / slotted cloud: no cache
            pass
    b_dev = torch.from_numpy(np.ascontiguousarray(bm)).to(dev)
    sp.xin.view(-1, sp.w)[:factors.h2.count] = b_dev.index_select(0, perm)
    sp.run_forward()
    sp.run_backward()
    x_dev = torch.empty_like(b_dev)
    x_dev[perm] = sp.output.view(-1, sp.w)[:factors.h2.count]
    x = x_dev.cpu().numpy()
    return x[:, 0] if vector else x
