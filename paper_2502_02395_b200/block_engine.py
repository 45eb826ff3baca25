"""GPU execution of the reference's dense block primitives and batch planner.

The reference funnels every dense operation of the factorization through
`dense_core.cholesky / tri_solve / multiply` and the batch planner
`plan_batches` / `run_plan` (dense_core.py:51-93, 184-284), which groups the
ops of one level/phase by kind and then runs them one LAPACK/BLAS call at a
time.  Here a `BatchGroup` is what its name says: ONE batched launch of the
library's kernels over all of its ops —

  multiply   one grouped DMMA GEMM launch (h2g_gemm_grouped), op(A)/op(B)
             through the kernel's transpose modes, `accumulate` preloaded
             into C (beta = 1), `scale` as alpha;
  cholesky   the device asymmetry check (h2g_sym_check, the ValueError of
             dense_core.py:56-59) and the partial-Cholesky panel program
             with r = n (the same CHOL_PANEL / GEMM steps the factorization
             runs), pivot status -> NotPositiveDefiniteError(pivot, *context);
  tri_solve  the 64x64 diagonal-block inverses of the triangle
             (h2g_tri_inv, zero diagonal -> SingularTriangularError) and the
             left-looking row solve X = C M^-T (h2g_trsm_rows); the four
             side/transpose modes are reduced to that form by transposing /
             reversing the operands on the host (M = L, or M = P L^T P with
             P the reversal, which is lower triangular).

Operands go up in one pinned copy per group and the results come back in
one.  The tile configuration is pinned per kind, so an op's result does not
depend on which other ops share its launch: `run_plan` and `run_sequential`
agree bit for bit (test_dense_core.py:244-258).  There is no CPU path: every
call needs the CUDA library (NativeUnavailableError otherwise).
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .errors import NotPositiveDefiniteError, SingularTriangularError
from .program import Program

INT_MAX = 2 ** 31 - 1
GEMM_CFG = 2          # 64x64 DMMA tiles for every block-engine GEMM (bitwise batch independence)


def _device():
    nat.lib()
    return torch.device("cuda", torch.cuda.current_device())


class _Arena:
    """Packs host arrays into one pinned buffer, one H2D copy, device pointers."""

    def __init__(self):
        self.parts = []
        self.size = 0

    def add(self, arr):
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        off = self.size
        self.parts.append((off, arr))
        self.size += max(arr.size, 1)
        self.size = -(-self.size // 32) * 32          # 256-byte aligned blocks
        return off

    def reserve(self, n):
        return self.add(np.zeros(max(int(n), 1)))

    def upload(self, device):
        host = torch.empty(max(self.size, 1), dtype=torch.float64, pin_memory=True)
        hv = host.numpy()
        for off, arr in self.parts:
            hv[off:off + arr.size] = arr.reshape(-1)
        self.dev = host.to(device, non_blocking=True)
        self._host = host
        self.base = self.dev.data_ptr()
        return self

    def ptr(self, off):
        return self.base + 8 * int(off)

    def download(self):
        return self.dev.cpu().numpy()


def _run(prog, device):
    prog.finalize()
    prog.run(torch.cuda.current_stream(device))


# --------------------------------------------------------------------------- multiply

def multiply_batch(items):
    """items: (a, b, transpose_a, transpose_b, accumulate_into, scale) tuples ->
    list of scale * op(A) op(B) (+ accumulate_into), one grouped GEMM launch
    per transpose combination (dense_core.multiply, dense_core.py:84-93)."""
    shapes = []
    for a, b, ta, tb, acc, scale in items:
        a = np.asarray(a, dtype=np.float64)
        b = np.asarray(b, dtype=np.float64)
        sa = a.shape[::-1] if ta else a.shape
        sb = b.shape[::-1] if tb else b.shape
        if sa[1] != sb[0]:
            raise ValueError(f"inner dimensions {tuple(sa)} x {tuple(sb)} do not conform")
        shapes.append((int(sa[0]), int(sb[1]), int(sa[1])))
    if not items:
        return []
    dev = _device()
    ar = _Arena()
    offs = []
    for (a, b, ta, tb, acc, scale), (m, n, k) in zip(items, shapes):
        oa, ob = ar.add(np.asarray(a, dtype=np.float64)), ar.add(np.asarray(b, dtype=np.float64))
        if acc is not None:
            acc = np.broadcast_to(np.asarray(acc, dtype=np.float64), (m, n))
            oc = ar.add(acc)
        else:
            oc = ar.reserve(m * n)
        offs.append((oa, ob, oc))
    ar.upload(dev)
    prog = Program(dev)
    groups = {}
    for q, ((a, b, ta, tb, acc, scale), (m, n, k), (oa, ob, oc)) in enumerate(zip(items, shapes, offs)):
        lda = int(np.shape(a)[1]) if np.ndim(a) == 2 else 1
        ldb = int(np.shape(b)[1]) if np.ndim(b) == 2 else 1
        groups.setdefault((bool(ta), bool(tb)), []).append(
            (ar.ptr(oa), ar.ptr(ob), ar.ptr(oc), m, n, k, max(lda, 1), max(ldb, 1), max(n, 1), 0, float(scale),
             1.0 if acc is not None else 0.0))
    for (ta, tb), probs in groups.items():
        prog.gemm(int(ta), int(tb), probs, tile_cfg=GEMM_CFG)
    _run(prog, dev)
    host = ar.download()
    out = []
    for (m, n, k), (oa, ob, oc) in zip(shapes, offs):
        out.append(host[oc:oc + m * n].reshape(m, n).copy())
    return out


# --------------------------------------------------------------------------- cholesky

def _sym_verdict(host_u64, q):
    dmax = host_u64[2 * q: 2 * q + 1].view(np.float64)[0]
    amax = host_u64[2 * q + 1: 2 * q + 2].view(np.float64)[0]
    return amax > 0 and dmax > 1e-10 * amax


def cholesky_batch(mats, contexts=None):
    """Lower Cholesky factors of every matrix (dense_core.cholesky,
    dense_core.py:51-66): asymmetry beyond 1e-10 relative -> ValueError,
    a non-positive pivot -> NotPositiveDefiniteError(pivot, level, box) with
    the op's context; errors surface in op order."""
    from .ulv_factor import partial_cholesky_steps

    mats = [np.asarray(a, dtype=np.float64) for a in mats]
    contexts = contexts or [None] * len(mats)
    res = [np.zeros((0, 0)) if a.shape[0] == 0 else None for a in mats]
    live = [q for q, a in enumerate(mats) if a.shape[0] > 0]
    if not live:
        return res
    dev = _device()
    ar = _Arena()
    offs = {q: ar.add(mats[q]) for q in live}
    ar.upload(dev)
    # H: every matrix back to back (the Cholesky works in place); qo in doubles from H's base
    n = np.array([mats[q].shape[0] for q in live], dtype=np.int64)
    qo = np.concatenate([[0], np.cumsum(n * n)[:-1]]).astype(np.int64)
    H = torch.empty(max(int((n * n).sum()), 1), dtype=torch.float64, device=dev)
    sym = torch.zeros(2 * len(live), dtype=torch.int64, device=dev)
    npd = torch.full((len(live),), INT_MAX, dtype=torch.int32, device=dev)
    prog = Program(dev)
    prog.symcheck([(ar.ptr(offs[q]), int(mats[q].shape[0]), int(mats[q].shape[0])) for q in live], sym.data_ptr())
    for t, q in enumerate(live):
        prog.memcpy(H.data_ptr() + 8 * int(qo[t]), ar.ptr(offs[q]), 8 * int(n[t] * n[t]))
    linv, _, _ = partial_cholesky_steps(prog, dev, npd.data_ptr(), H.data_ptr(), 0, qo, n, n.copy(), 0)
    _run(prog, dev)
    sym_h = sym.cpu().numpy().view(np.uint64)
    npd_h = npd.cpu().numpy()
    Hh = H.cpu().numpy()
    for t, q in enumerate(live):
        if _sym_verdict(sym_h, t):
            raise ValueError("matrix is not symmetric to 1e-10 relative")
        if npd_h[t] != INT_MAX:
            lvl, box = contexts[q] if contexts[q] is not None else (None, None)
            raise NotPositiveDefiniteError(int(npd_h[t]), level=lvl, box=box)
        nt = int(n[t])
        res[q] = np.tril(Hh[qo[t]:qo[t] + nt * nt].reshape(nt, nt))
    del linv
    return res


# --------------------------------------------------------------------------- tri_solve

def _to_rows_form(l, b, side, transposed):
    """(M, C, finish): op(L) X = B (left) / X op(L) = B (right) as X' = C M^-T
    with M lower triangular, X = finish(X')."""
    vec = b.ndim == 1
    if side == "left":
        bb = b[:, None] if vec else b
        if not transposed:                 # X = L^-1 B  ->  X^T = B^T L^-T
            m, c = l, bb.T
            fin = lambda x: x.T
        else:                              # X = L^-T B  ->  X^T = B^T L^-1 = ((B^T P) M^-T) P
            m, c = l.T[::-1, ::-1], bb.T[:, ::-1]
            fin = lambda x: x[:, ::-1].T
    else:
        bb = b[None, :] if vec else b
        if transposed:                     # X = B L^-T
            m, c = l, bb
            fin = lambda x: x
        else:                              # X = B L^-1 = ((B P) M^-T) P
            m, c = l.T[::-1, ::-1], bb[:, ::-1]
            fin = lambda x: x[:, ::-1]
    if vec:
        return m, c, lambda x, f=fin: np.ascontiguousarray(f(x)).reshape(-1)
    return m, c, lambda x, f=fin: np.ascontiguousarray(f(x))


def tri_solve_batch(items):
    """items: (l, b, side, transposed) -> list of X with op(L) X = B (left) or
    X op(L) = B (right) (dense_core.tri_solve, dense_core.py:69-81); a zero
    diagonal entry raises SingularTriangularError (in op order)."""
    out = [None] * len(items)
    live = []
    for q, (l, b, side, transposed) in enumerate(items):
        l = np.asarray(l, dtype=np.float64)
        b = np.asarray(b, dtype=np.float64)
        if l.shape[0] == 0 or b.size == 0:
            out[q] = np.zeros_like(b)
            continue
        live.append((q, *_to_rows_form(l, b, side, transposed)))
    if not live:
        return out
    dev = _device()
    ar = _Arena()
    W = nat.PANEL_WIDTH
    descs = []
    for q, m, c, fin in live:
        nn = int(m.shape[0])
        om, oc = ar.add(m), ar.add(c)
        ol = ar.reserve(-(-nn // W) * W * W)
        descs.append((om, oc, ol, nn, int(c.shape[0])))
    ar.upload(dev)
    status = torch.full((len(live),), INT_MAX, dtype=torch.int32, device=dev)
    prog = Program(dev)
    prog.triinv([(ar.ptr(om), ar.ptr(ol), nn, nn, t) for t, (om, oc, ol, nn, rows) in enumerate(descs)],
                status.data_ptr())
    prog.trsm_rows([(ar.ptr(om), ar.ptr(oc), ar.ptr(oc), ar.ptr(ol), rows, nn, 0, -(-nn // W), nn, nn)
                    for (om, oc, ol, nn, rows) in descs])
    _run(prog, dev)
    st = status.cpu().numpy()
    host = ar.download()
    for t, ((q, m, c, fin), (om, oc, ol, nn, rows)) in enumerate(zip(live, descs)):
        if st[t] != INT_MAX:
            raise SingularTriangularError("zero diagonal entry in triangular factor")
        out[q] = fin(host[oc:oc + rows * nn].reshape(rows, nn))
    return out


# --------------------------------------------------------------------------- the reference's planner

def flop_count(kind, dims):
    from .dense_core import flop_count as fc

    return fc(kind, dims)


@dataclass
class BlockOp:
    """One dense operation destined for a batch group (dense_core.py:184-207):
    dims are the true dimensions, (n,) cholesky, (n, m) tri_solve, (m, n, k)
    multiply; `sink` receives the true-region result."""

    kind: str
    dims: tuple
    a: np.ndarray = None
    b: np.ndarray = None
    transpose_a: bool = False
    transpose_b: bool = False
    scale: float = 1.0
    accumulate: np.ndarray = None
    side: str = "left"
    transposed: bool = False
    context: tuple = None
    sink: object = None


@dataclass
class BatchGroup:
    kind: str
    padded_dims: tuple
    ops: list


@dataclass
class BatchPlan:
    groups: list = field(default_factory=list)
    true_flops: int = 0
    padded_flops: int = 0

    @property
    def op_count(self):
        return sum(len(g.ops) for g in self.groups)


def _round4(x):
    return max(4, -(-x // 4) * 4) if x > 0 else 0


def plan_batches(level_ops, budget_blocks=None):
    """Group by kind, pad each dim to the per-kind maximum rounded to 4 (the
    flop accounting of the padded model), split groups to at most
    `budget_blocks` ops (dense_core.py:229-248).  Padding is only accounted:
    each group runs as one batched launch over the TRUE sizes."""
    plan = BatchPlan()
    by_kind = {}
    for op in level_ops:
        by_kind.setdefault(op.kind, []).append(op)
    for kind, ops in by_kind.items():
        width = len(ops[0].dims)
        maxdims = tuple(_round4(max(op.dims[d] for op in ops)) for d in range(width))
        chunk = len(ops) if not budget_blocks else max(1, budget_blocks)
        for s in range(0, len(ops), chunk):
            plan.groups.append(BatchGroup(kind=kind, padded_dims=maxdims, ops=ops[s:s + chunk]))
        for op in ops:
            plan.true_flops += flop_count(kind, op.dims)
            plan.padded_flops += flop_count(kind, maxdims)
    return plan


def run_group(kind, ops):
    """One batched launch for the ops of one kind; sinks called in op order."""
    if kind == "cholesky":
        res = cholesky_batch([op.a for op in ops], [op.context for op in ops])
    elif kind == "tri_solve":
        res = tri_solve_batch([(op.a, op.b, op.side, op.transposed) for op in ops])
    elif kind == "multiply":
        res = multiply_batch([(op.a, op.b, op.transpose_a, op.transpose_b, op.accumulate, op.scale) for op in ops])
    else:
        raise ValueError(f"unknown op kind '{kind}'")
    for op, r in zip(ops, res):
        if op.sink is not None:
            op.sink(r)
    return res


def run_op(op):
    """Execute a single BlockOp on its true region (dense_core.py:251-266)."""
    return run_group(op.kind, [op])[0]


def run_plan(plan):
    """Execute a BatchPlan: one batched GPU launch per group (dense_core.py:269-274)."""
    for group in plan.groups:
        run_group(group.kind, group.ops)


def run_sequential(level_ops):
    """One launch per op (dense_core.py:277-281)."""
    for op in level_ops:
        run_op(op)


# --------------------------------------------------------------------------- one-box ULV steps

def sparsify_diag(basis, a_ii):
    """Q^T A_ii Q split into (rr, rs, sr, ss), redundant slab first
    (ulv_factor.py:70-75): GEMM NN (A Q) then TN (Q^T M) in one program."""
    q = np.ascontiguousarray(basis.q_full, dtype=np.float64)
    a = np.asarray(a_ii, dtype=np.float64)
    n = q.shape[0]
    r = basis.n - basis.rank
    if n == 0:
        h = np.zeros((0, 0))
    else:
        dev = _device()
        ar = _Arena()
        oa, oq, om, oh = ar.add(a), ar.add(q), ar.reserve(n * n), ar.reserve(n * n)
        ar.upload(dev)
        prog = Program(dev)
        prog.gemm(0, 0, [(ar.ptr(oa), ar.ptr(oq), ar.ptr(om), n, n, n, n, n, n, 0, 1.0, 0.0)], tile_cfg=GEMM_CFG)
        prog.gemm(1, 0, [(ar.ptr(oq), ar.ptr(om), ar.ptr(oh), n, n, n, n, n, n, 0, 1.0, 0.0)], tile_cfg=GEMM_CFG)
        _run(prog, dev)
        h = ar.download()[oh:oh + n * n].reshape(n, n)
    return (h[:r, :r].copy(), h[:r, r:].copy(), h[r:, :r].copy(), h[r:, r:].copy())


def factor_diag(rr, sr, ss, basis, context=None):
    """Eliminate the redundant part of one diagonal block (ulv_factor.py:78-84):
    (L(r), L(s) = SR L^-T, SS - L(s) L(s)^T, V = q_red L^-T) — ONE partial
    Cholesky of [[RR, .], [SR, SS]] (the factorization's own panel program:
    panels, TRSM of the SR rows, the single SYRK Schur update of SS, and the
    row solve of V riding along on q_full), plus the asymmetry check of RR."""
    from .ulv_factor import partial_cholesky_steps

    rr = np.asarray(rr, dtype=np.float64)
    sr = np.asarray(sr, dtype=np.float64)
    ss = np.asarray(ss, dtype=np.float64)
    r = rr.shape[0]
    k = ss.shape[0]
    n = r + k
    q_full = np.ascontiguousarray(basis.q_full, dtype=np.float64)
    if r == 0:
        return np.zeros((0, 0)), np.zeros_like(sr), ss - np.zeros((k, k)), np.zeros_like(basis.q_red)
    h = np.zeros((n, n))
    h[:r, :r] = rr
    h[r:, :r] = sr
    h[r:, r:] = ss
    dev = _device()
    ar = _Arena()
    oh, oq, orr, ov = ar.add(h), ar.add(q_full), ar.add(rr), ar.reserve(n * n)
    ar.upload(dev)
    sym = torch.zeros(2, dtype=torch.int64, device=dev)
    npd = torch.full((1,), INT_MAX, dtype=torch.int32, device=dev)
    prog = Program(dev)
    prog.symcheck([(ar.ptr(orr), r, r)], sym.data_ptr())
    linv, _, _ = partial_cholesky_steps(prog, dev, npd.data_ptr(), ar.ptr(oh), ar.ptr(ov), np.array([0]),
                                        np.array([n]), np.array([r]), 0, Qp=ar.ptr(oq))
    _run(prog, dev)
    if _sym_verdict(sym.cpu().numpy().view(np.uint64), 0):
        raise ValueError("matrix is not symmetric to 1e-10 relative")
    bad = int(npd.cpu().numpy()[0])
    if bad != INT_MAX:
        lvl, box = context if context is not None else (None, None)
        raise NotPositiveDefiniteError(bad, level=lvl, box=box)
    host = ar.download()
    H = host[oh:oh + n * n].reshape(n, n)
    V = host[ov:ov + n * n].reshape(n, n)
    del linv
    ssl = np.tril(H[r:, r:])
    ss_up = ssl + np.tril(ssl, -1).T       # the SYRK maintains the lower triangle
    return np.tril(H[:r, :r]), H[r:, :r].copy(), ss_up, V[:, :r].copy()


def sparsify_off(basis_i, a_ij, v_j, basis_j, lr_ii=None):
    """Transform one near off-diagonal block, i > j (ulv_factor.py:87-105):
    T = Q_i^T (A_ij [V_j | q_skel_j]) by two grouped GEMMs; with lr_ii the
    mirror L(s)_ji = (L(r)_ii^-1 RS)^T = RS^T L(r)_ii^-T by the row solve on
    the transposed RS slab (one program)."""
    a = np.asarray(a_ij, dtype=np.float64)
    right = np.hstack([np.asarray(v_j, dtype=np.float64), basis_j.q_skel])
    q = np.ascontiguousarray(basis_i.q_full, dtype=np.float64)
    ni, nj = a.shape
    ri = basis_i.n - basis_i.rank
    rj = basis_j.n - basis_j.rank
    kj = basis_j.rank
    want_mirror = lr_ii is not None and ri > 0 and kj > 0
    if ni == 0 or nj == 0:
        t = np.zeros((ni, right.shape[1]))
        host = None
    else:
        dev = _device()
        ar = _Arena()
        oa, orr, oq = ar.add(a), ar.add(right), ar.add(q)
        om, ot = ar.reserve(ni * nj), ar.reserve(ni * nj)
        prog_descs = None
        if want_mirror:
            ol = ar.add(np.asarray(lr_ii, dtype=np.float64))
            oc = ar.reserve(kj * ri)
            olinv = ar.reserve(-(-ri // nat.PANEL_WIDTH) * nat.PANEL_WIDTH ** 2)
        ar.upload(dev)
        prog = Program(dev)
        prog.gemm(0, 0, [(ar.ptr(oa), ar.ptr(orr), ar.ptr(om), ni, nj, nj, nj, nj, nj, 0, 1.0, 0.0)],
                  tile_cfg=GEMM_CFG)
        prog.gemm(1, 0, [(ar.ptr(oq), ar.ptr(om), ar.ptr(ot), ni, nj, ni, ni, nj, nj, 0, 1.0, 0.0)],
                  tile_cfg=GEMM_CFG)
        status = torch.full((1,), INT_MAX, dtype=torch.int32, device=dev)
        if want_mirror:
            # C = RS^T (k_j x r_i) from T[:r_i, r_j:] by the transposing copy, then C L^-T
            prog.copy([(ar.ptr(ot + rj), ar.ptr(oc), kj, ri, nj, ri, 1)])
            prog.triinv([(ar.ptr(ol), ar.ptr(olinv), ri, ri, 0)], status.data_ptr())
            prog.trsm_rows([(ar.ptr(ol), ar.ptr(oc), ar.ptr(oc), ar.ptr(olinv), kj, ri, 0,
                             -(-ri // nat.PANEL_WIDTH), ri, ri)])
        _run(prog, dev)
        if want_mirror and int(status.cpu().numpy()[0]) != INT_MAX:
            raise SingularTriangularError("zero diagonal entry in triangular factor")
        host = ar.download()
        t = host[ot:ot + ni * nj].reshape(ni, nj)
    ls_ji = None
    if lr_ii is not None:
        ls_ji = host[oc:oc + kj * ri].reshape(kj, ri).copy() if want_mirror else np.zeros((kj, ri))
    return t[:ri, :rj].copy(), t[ri:, :rj].copy(), t[ri:, rj:].copy(), ls_ji


def merge_level(ss_of, lists, level, ranks):
    """2x2-assemble child SS blocks into the parent near blocks of level-1
    (ulv_factor.py:115-132): every child block goes up once and ONE
    block-copy launch places all of them; a missing child -> StructureError."""
    from .errors import StructureError

    parents = [(pi, pj) for (pi, pj) in lists.near[level - 1] if pi >= pj]
    kids = {}
    for (pi, pj) in parents:
        for ci in (2 * pi, 2 * pi + 1):
            for cj in (2 * pj, 2 * pj + 1):
                blk = ss_of(ci, cj)
                if blk is None:
                    raise StructureError(f"missing child SS block ({level}, {ci}, {cj})")
                kids[(pi, pj, ci, cj)] = np.asarray(blk, dtype=np.float64)
    if not parents:
        return {}
    dims = {}
    for (pi, pj, ci, cj), blk in kids.items():
        dims[ci] = blk.shape[0]
        dims[cj] = blk.shape[1]
    ar = _Arena()
    src = {key: ar.add(blk) for key, blk in kids.items()}
    out = {}
    for (pi, pj) in parents:
        mi, mj = dims[2 * pi] + dims[2 * pi + 1], dims[2 * pj] + dims[2 * pj + 1]
        out[(pi, pj)] = (ar.reserve(mi * mj), mi, mj)
    dev = _device()
    ar.upload(dev)
    descs = []
    for (pi, pj, ci, cj), blk in kids.items():
        o, mi, mj = out[(pi, pj)]
        ro = 0 if ci == 2 * pi else dims[2 * pi]
        co = 0 if cj == 2 * pj else dims[2 * pj]
        descs.append((ar.ptr(src[(pi, pj, ci, cj)]), ar.ptr(o + ro * mj + co), blk.shape[0], blk.shape[1],
                      max(blk.shape[1], 1), mj, 0))
    prog = Program(dev)
    prog.copy(descs)
    _run(prog, dev)
    host = ar.download()
    return {key: host[o:o + mi * mj].reshape(mi, mj).copy() for key, (o, mi, mj) in out.items()}
