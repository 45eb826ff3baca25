"""CPU ORACLE for the H²-ULV factorize / solve path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this module, and only as the checker or the
timed CPU baseline; the product package (paper_2502_02395_b200) never
imports it and has no CPU fallback.

A plain numpy/scipy restatement of the reference algorithm
(/root/reference/pkg/src/h2ulv, the un-vendored LAPACK/BLAS it calls is
scipy 1.18.1 / numpy 2.3.5 with scipy-openblas 0.3.30 in this image):

  factorize      ulv_factor.py:154-316 (diag transform 189-200, partial
                 Cholesky 217-241, off-diagonal transform 243-272, mirror
                 282-286, couplings 108-112/289, merge 115-132/292-303,
                 root 309-314)
  solve          ulv_solve.py:66-207 (parallel and naive forward/backward)
  h2_matvec      h2_build.py:232-282
  complete_qr    dense_core.py:136-148 (the ① complementary basis)
  flop model     dense_core.py:166-181 / 229-248
  dense_assemble oracle.py:34-40 (the dense kernel matrix, capped) and the
                 exact residual / refinement checks built on it

Parity pinned: tests/test_oracle.py checks this module against golden
vectors produced by running the reference itself (tests/golden/make_golden.py):
block-by-block factors, root, solution and the flop report of three small
reference H2 matrices, plus the reference's known-answer tests.
"""

import numpy as np
import scipy.linalg

from paper_2502_02395_b200.errors import NotPositiveDefiniteError  # exception type only


# ----------------------------------------------------------------------------- dense kernels

def chol(a, level=None, box=None):
    """dpotrf (lower) with the reference's error contract (dense_core.py:51-66)."""
    a = np.asarray(a, dtype=np.float64)
    if a.shape[0] == 0:
        return np.zeros((0, 0))
    scale = np.abs(a).max()
    if scale > 0 and np.abs(a - a.T).max() > 1e-10 * scale:
        raise ValueError("matrix is not symmetric to 1e-10 relative")
    c, info = scipy.linalg.lapack.dpotrf(a, lower=1)
    if info > 0:
        raise NotPositiveDefiniteError(info - 1, level=level, box=box)
    return np.tril(c)


def trsm_right_lt(l, b):
    """X with X L^T = B (dense_core.tri_solve side=right, transposed=True)."""
    if l.shape[0] == 0 or b.size == 0:
        return np.zeros_like(b)
    return scipy.linalg.solve_triangular(l, b.T, lower=True, trans="N").T


def trsv(l, b, transposed=False):
    if l.shape[0] == 0 or b.size == 0:
        return np.zeros_like(b)
    return scipy.linalg.solve_triangular(l, b, lower=True, trans="T" if transposed else "N")


def complete_qr(z, k):
    """q_full = [q_red | q_skel] and frame of Z (n x k), sign-fixed (dense_core.py:136-148)."""
    n = z.shape[0]
    if k == 0:
        return np.eye(n), np.zeros((0, 0))
    q, r = np.linalg.qr(z, mode="complete")
    s = np.sign(np.diag(r[:k, :k]))
    s[s == 0] = 1.0
    return np.hstack([q[:, k:], q[:, :k] * s]), s[:, None] * r[:k, :]


# ----------------------------------------------------------------------------- flop model

def _flops(kind, dims):
    if kind == "cholesky":
        return dims[0] ** 3 // 3
    if kind == "tri_solve":
        return dims[0] * dims[0] * dims[1]
    return 2 * dims[0] * dims[1] * dims[2]


def _r4(x):
    return 0 if x <= 0 else max(4, -(-x // 4) * 4)


class FlopReport:
    def __init__(self):
        self.d = {"levels": {}, "total_true": 0, "total_padded": 0}

    def add(self, level, phase, ops):
        groups = {}
        for kind, dims in ops:
            groups.setdefault(kind, []).append(tuple(int(x) for x in dims))
        t = p = 0
        for kind, lst in groups.items():
            mx = tuple(_r4(max(d[a] for d in lst)) for a in range(len(lst[0])))
            t += sum(_flops(kind, d) for d in lst)
            p += len(lst) * _flops(kind, mx)
        e = self.d["levels"].setdefault(level, {}).setdefault(phase, {"true": 0, "padded": 0, "count": 0})
        e["true"] += t
        e["padded"] += p
        e["count"] += len(ops)
        self.d["total_true"] += t
        self.d["total_padded"] += p


# ----------------------------------------------------------------------------- factorize

class OracleFactors:
    def __init__(self, h2):
        self.h2 = h2
        self.levels = {}
        self.root = None
        self.flops = None

    @property
    def depth(self):
        return self.h2.tree.depth


def factorize(h2):
    """Sequential restatement of ulv_factor.factorize on host numpy blocks."""
    depth = h2.tree.depth
    f = OracleFactors(h2)
    fr = FlopReport()
    if depth == 0:
        a = h2.near_blocks[(0, 0, 0)]
        fr.add(0, "root", [("cholesky", (a.shape[0],))])
        f.root = chol(a, 0, 0)
        f.flops = fr.d
        return f
    cur = {(i, j): h2.near_blocks[(depth, i, j)] for (i, j) in
           [(i, j) for (i, j) in h2.lists.near[depth] if i >= j]}
    for l in range(depth, 0, -1):
        nb = 2 ** l
        B = [h2.bases[(l, i)] for i in range(nb)]
        n = [b.q_skel.shape[0] for b in B]
        k = [b.rank for b in B]
        r = [n[i] - k[i] for i in range(nb)]
        Q = [np.hstack([b.q_red, b.q_skel]) for b in B]
        lvl = {"lr_diag": {}, "lr_off": {}, "ls": {}, "v": {}, "dims": {i: (r[i], k[i]) for i in range(nb)}}
        ss = {}
        fr.add(l, "diag_mul1", [("multiply", (n[i], n[i], n[i])) for i in range(nb)])
        fr.add(l, "diag_mul2", [("multiply", (n[i], n[i], n[i])) for i in range(nb)])
        hs = [Q[i].T @ (cur[(i, i)] @ Q[i]) for i in range(nb)]
        for i in range(nb):
            lvl["lr_diag"][i] = chol(hs[i][:r[i], :r[i]], l, i)
        # errors are raised per box in index order before any TRSM, as in the reference
        fr.add(l, "diag_chol", [("cholesky", (r[i],)) for i in range(nb)])
        for i in range(nb):
            h = hs[i]
            ri = r[i]
            lr = lvl["lr_diag"][i]
            ls = trsm_right_lt(lr, h[ri:, :ri])
            lvl["ls"][(i, i)] = ls
            lvl["v"][i] = trsm_right_lt(lr, B[i].q_red)
            ss[(i, i)] = h[ri:, ri:] - ls @ ls.T
        fr.add(l, "diag_trsm", [x for i in range(nb) for x in (("tri_solve", (r[i], k[i])),
                                                               ("tri_solve", (r[i], n[i])))])
        fr.add(l, "diag_schur", [("multiply", (k[i], k[i], r[i])) for i in range(nb)])
        offp = sorted((i, j) for (i, j) in h2.lists.near[l] if i > j)
        fr.add(l, "off_mul1", [("multiply", (n[i], n[j], n[j])) for (i, j) in offp])
        fr.add(l, "off_mul2", [("multiply", (n[i], n[j], n[i])) for (i, j) in offp])
        fr.add(l, "off_mirror", [("tri_solve", (r[i], k[j])) for (i, j) in offp])
        for (i, j) in offp:
            right = np.hstack([lvl["v"][j], B[j].q_skel])
            t = Q[i].T @ (cur[(i, j)] @ right)
            lvl["lr_off"][(i, j)] = t[:r[i], :r[j]]
            lvl["ls"][(i, j)] = t[r[i]:, :r[j]]
            ss[(i, j)] = t[r[i]:, r[j]:]
            lvl["ls"][(j, i)] = trsv(lvl["lr_diag"][i], t[:r[i], r[j]:]).T
        for (i, j) in h2.lists.far[l]:
            if i > j:
                ss[(i, j)] = h2.couplings[(l, i, j)]

        def child(ci, cj):
            return ss[(ci, cj)] if ci >= cj else ss[(cj, ci)].T

        cur = {(pi, pj): np.block([[child(2 * pi + a, 2 * pj + b) for b in (0, 1)] for a in (0, 1)])
               for (pi, pj) in h2.lists.near[l - 1] if pi >= pj}
        f.levels[l] = lvl
    a00 = cur[(0, 0)]
    fr.add(0, "root", [("cholesky", (a00.shape[0],))])
    f.root = chol(a00, 0, 0)
    f.flops = fr.d
    return f


# ----------------------------------------------------------------------------- solve

def _near_lists(lists, l, nb):
    below = [sorted(j for (i, j) in lists.near[l] if i == a and j < a) for a in range(nb)]
    above = [sorted(i for (i, j) in lists.near[l] if j == a and i > a) for a in range(nb)]
    return below, above


def forward(f, bt, parallel=True):
    """Tree-order rhs -> ({(l, i): y_R}, root segment) (ulv_solve.py:66-116)."""
    h2 = f.h2
    bm = np.asarray(bt, dtype=np.float64).reshape(h2.count, -1)
    depth = f.depth
    if depth == 0:
        return {}, trsv(f.root, bm)
    segs = {i: bm[b.begin:b.end] for i, b in enumerate(h2.tree.leaves)}
    yr = {}
    for l in range(depth, 0, -1):
        nb = 2 ** l
        lv = f.levels[l]
        br, bs = {}, {}
        for i in range(nb):
            b = h2.bases[(l, i)]
            w = np.hstack([b.q_red, b.q_skel]).T @ segs[i]
            br[i], bs[i] = w[:lv["dims"][i][0]], w[lv["dims"][i][0]:]
        below, above = _near_lists(h2.lists, l, nb)
        targets = [sorted(a for (a, c) in lv["ls"] if c == i) for i in range(nb)]
        if parallel:
            z = {i: trsv(lv["lr_diag"][i], br[i]) for i in range(nb)}
            y = {}
            for i in range(nb):
                u = np.zeros_like(br[i])
                for j in below[i]:
                    u += lv["lr_off"][(i, j)] @ z[j]
                y[i] = trsv(lv["lr_diag"][i], br[i] - u)
            for i in range(nb):
                for a in targets[i]:
                    bs[a] = bs[a] - lv["ls"][(a, i)] @ y[i]
            br = y
        else:
            for i in range(nb):
                yi = trsv(lv["lr_diag"][i], br[i])
                br[i] = yi
                for j in above[i]:
                    br[j] = br[j] - lv["lr_off"][(j, i)] @ yi
                for a in targets[i]:
                    bs[a] = bs[a] - lv["ls"][(a, i)] @ yi
        for i in range(nb):
            yr[(l, i)] = br[i]
        segs = {p: np.vstack([bs[2 * p], bs[2 * p + 1]]) for p in range(nb // 2)}
    return yr, trsv(f.root, segs[0])


def backward(f, yr, yroot, parallel=True):
    """(ulv_solve.py:127-188) -> tree-order x (N x w)."""
    h2 = f.h2
    depth = f.depth
    xroot = trsv(f.root, yroot, transposed=True)
    if depth == 0:
        return xroot
    parent = xroot
    for l in range(1, depth + 1):
        nb = 2 ** l
        lv = f.levels[l]
        xs, pos = {}, 0
        for i in range(nb):
            kk = lv["dims"][i][1]
            xs[i] = parent[pos:pos + kk]
            pos += kk
        y = {i: yr[(l, i)].copy() for i in range(nb)}
        below, above = _near_lists(h2.lists, l, nb)
        sources = [sorted(a for (a, c) in lv["ls"] if c == i) for i in range(nb)]
        for i in range(nb):
            for a in sources[i]:
                y[i] = y[i] - lv["ls"][(a, i)].T @ xs[a]
        xr = {}
        if parallel:
            z = {i: trsv(lv["lr_diag"][i], y[i], True) for i in range(nb)}
            for i in range(nb):
                u = np.zeros_like(y[i])
                for j in above[i]:
                    u += lv["lr_off"][(j, i)].T @ z[j]
                xr[i] = trsv(lv["lr_diag"][i], y[i] - u, True)
        else:
            for i in reversed(range(nb)):
                acc = y[i]
                for j in above[i]:
                    acc = acc - lv["lr_off"][(j, i)].T @ xr[j]
                xr[i] = trsv(lv["lr_diag"][i], acc, True)
        full = [h2.bases[(l, i)].q_red @ xr[i] + h2.bases[(l, i)].q_skel @ xs[i] for i in range(nb)]
        parent = np.vstack(full)
    return parent


def solve(f, b, mode="parallel"):
    """User-order b -> user-order x (ulv_solve.py:191-207)."""
    b = np.asarray(b, dtype=np.float64)
    vec = b.ndim == 1
    bm = b.reshape(f.h2.count, -1)
    perm = f.h2.cloud.perm
    yr, yroot = forward(f, bm[perm], mode == "parallel")
    xt = backward(f, yr, yroot, mode == "parallel")
    x = np.zeros_like(xt)
    x[perm] = xt
    return x[:, 0] if vec else x


# ----------------------------------------------------------------------------- matvec

def h2_matvec(h2, x):
    """Tree-order y = A x through the H² representation (h2_build.py:232-282)."""
    xm = np.asarray(x, dtype=np.float64).reshape(h2.count, -1)
    tree, depth = h2.tree, h2.tree.depth
    if depth == 0:
        return (h2.near_blocks[(0, 0, 0)] @ xm).reshape(np.shape(x))
    up = {}
    for l in range(depth, 0, -1):
        for i in range(2 ** l):
            if l == depth:
                b = tree.boxes[l][i]
                seg = xm[b.begin:b.end]
            else:
                seg = np.vstack([up[(l + 1, 2 * i)], up[(l + 1, 2 * i + 1)]])
            up[(l, i)] = h2.bases[(l, i)].q_skel.T @ seg
    dn = {key: np.zeros_like(v) for key, v in up.items()}
    for l in range(depth, 0, -1):
        for (i, j) in h2.lists.far[l]:
            s = h2.couplings[(l, i, j)] if i > j else h2.couplings[(l, j, i)].T
            dn[(l, i)] += s @ up[(l, j)]
    y = np.zeros_like(xm)
    for l in range(1, depth + 1):
        for i in range(2 ** l):
            full = h2.bases[(l, i)].q_skel @ dn[(l, i)]
            if l == depth:
                b = tree.boxes[l][i]
                y[b.begin:b.end] += full
            else:
                ka = h2.bases[(l + 1, 2 * i)].rank
                dn[(l + 1, 2 * i)] += full[:ka]
                dn[(l + 1, 2 * i + 1)] += full[ka:]
    for (i, j) in h2.lists.near[depth]:
        bi, bj = tree.boxes[depth][i], tree.boxes[depth][j]
        blk = h2.near_blocks[(depth, i, j)] if i >= j else h2.near_blocks[(depth, j, i)].T
        y[bi.begin:bi.end] += blk @ xm[bj.begin:bj.end]
    return y.reshape(np.shape(x))


def residual(h2, x, b):
    """||A x - b|| / ||b|| through the H² matvec in tree order (cli.py:199-205)."""
    perm = h2.cloud.perm
    r = h2_matvec(h2, np.asarray(x)[perm]) - np.asarray(b)[perm]
    return float(np.linalg.norm(r) / np.linalg.norm(b))


DENSE_CAP = 16384


def dense_assemble(kernel, cloud, cap=DENSE_CAP):
    """Full N x N kernel matrix in the cloud's current (tree) order
    (oracle.py:34-40: gen_block over all points, capped)."""
    from paper_2502_02395_b200 import kernels

    n = cloud.count
    if n > cap:
        raise ValueError(f"N = {n} exceeds the dense-oracle cap {cap}")
    idx = np.arange(n, dtype=np.int64)
    return kernels.gen_block(kernel, idx, idx, cloud)


def exact_residual(a_tree, perm, x, b):
    """||A x - b|| / ||b|| with the dense matrix A in tree order, x / b in input order."""
    r = a_tree @ np.asarray(x)[perm] - np.asarray(b)[perm]
    return float(np.linalg.norm(r) / np.linalg.norm(b))


# ----------------------------------------------------------------------------- construct (CPU)

def construct(kernel, tree, lists, cfg, cloud, workers=None):
    """CPU construction (h2_build.py:170-220) for the CPU baseline arm.

    The skeleton pass is the package's host half (pinned bit-exact to the
    reference by tests/test_host_parity.py); the complementary basis is
    numpy's LAPACK QR (dense_core.py:136-148) and the blocks come from the
    host kernel evaluator (kernels.py:46-64).  Returns an H2Matrix of host
    numpy blocks (leaf near blocks only — the factorization reads no others).
    """
    import os

    import scipy.linalg as sla

    from paper_2502_02395_b200 import kernels
    from paper_2502_02395_b200.dense_core import BasisDecomposition
    from paper_2502_02395_b200.h2_build import H2Matrix, _skel_global, _skeleton_pass

    h2 = H2Matrix(tree=tree, lists=lists, kernel=kernel, cloud=cloud, config=cfg)
    depth = tree.depth
    if depth == 0:
        allp = np.arange(cloud.count, dtype=np.int64)
        h2.near_blocks = {(0, 0, 0): kernels.gen_block(kernel, allp, allp, cloud)}
        return h2
    eff, choice = _skeleton_pass(kernel, tree, lists, cfg, cloud, h2.build_flops, workers or os.cpu_count())
    h2.eff_points = eff
    for l in range(depth, 0, -1):
        for i in range(2 ** l):
            c = choice[(l, i)]
            n = len(eff[(l, i)])
            k = 0 if c is None else c.rank
            if k:
                z = c.t
                if l < depth:
                    w = sla.block_diag(h2.bases[(l + 1, 2 * i)].frame, h2.bases[(l + 1, 2 * i + 1)].frame)
                    z = w @ z
                qf, fr = complete_qr(z, k)
            else:
                qf, fr = np.eye(n), np.zeros((0, 0))
            skel = np.zeros(0, np.int64) if c is None else c.skeleton
            h2.bases[(l, i)] = BasisDecomposition(q_skel=qf[:, n - k:], q_red=qf[:, :n - k], skeleton=skel,
                                                  rank=k, frame=fr)
            h2.skeletons[(l, i)] = _skel_global(eff, choice, l, i)
        for (i, j) in lists.far[l]:
            if i > j:
                g = kernels.gen_block(kernel, h2.skeletons[(l, i)], h2.skeletons[(l, j)], cloud)
                h2.couplings[(l, i, j)] = h2.bases[(l, i)].frame @ g @ h2.bases[(l, j)].frame.T
    for (i, j) in lists.near[depth]:
        if i >= j:
            h2.near_blocks[(depth, i, j)] = kernels.gen_block(kernel, eff[(depth, i)], eff[(depth, j)], cloud)
    return h2
