"""H² construction — drop-in for `h2ulv.h2_build` (h2_build.py:1-282).

Split of the work (north star: skeletons bit-exact, ① on the GPU):

host, per level, boxes in parallel threads (BLAS pinned to 1 thread each)
  * stratified seeded sampling of far / near points (h2_build.py:73-113)
  * Gauss-Seidel close-field prefactor G(B_i, S_C) A_cc^-1 (116-152)
  * pivoted-QR skeleton choice and interpolation operator T (dense_core.py:114-134)
  These define the skeleton indices, which must equal the reference's bit
  for bit, so they use the same LAPACK routines on identical samples.

GPU, one static program for the whole tree (program.Program)
  * Z_i = T_i (leaf) or blockdiag(F_2i, F_2i+1) T_i (h2_build.py:193-197) — grouped GEMM
  * ① batched blocked Householder QR -> q_full_i = [q_red | q_skel], frame F_i (basis_qr)
  * leaf near blocks G(B_i, B_j) (205-208) and skeleton blocks G(SK_i, SK_j) — kernel-block kernel
  * couplings S_ij = F_i G(SK_i, SK_j) F_j^T (209-215) — grouped GEMM
The result keeps every operand in HBM (`h2._device`) so factorize() starts
without a host->device copy; the numpy attributes of the reference's
H2Matrix (bases, near_blocks, couplings) materialize lazily on access.
"""

import os
from collections.abc import Mapping
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import torch

from .trace import ranged
from . import _native as nat
from . import dense_core, kernels
from .basis_qr import LevelQR, build_wy, rebuild_qfull, wy_profitable, wy_signs
from .dense_core import BasisDecomposition, skeleton_selection, solve_triangular
from .errors import CoincidentPointsError, SingularTriangularError, StructureError
from .h2_device import DeviceH2, LevelLayout
from .program import Program

WY_ENABLED = os.environ.get("H2G_WY", "1") != "0"   # compact-WY diag transform (A/B switch)

F64 = torch.float64


@dataclass
class BuildConfig:
    eta: float = 1.0
    leaf_max: int = 64
    rank: int = None
    tol: float = None
    s_far: int = 0
    s_near: int = 0
    gs_sweeps: int = 2
    seed: int = 0

    def __post_init__(self):
        if (self.rank is None) == (self.tol is None):
            raise ValueError("exactly one of rank/tol must be set")
        if self.gs_sweeps < 0:
            raise ValueError("gs_sweeps must be >= 0")


@dataclass
class H2Matrix:
    tree: object
    lists: object
    kernel: object
    cloud: object
    config: object
    bases: Mapping = field(default_factory=dict)
    skeletons: dict = field(default_factory=dict)
    eff_points: dict = field(default_factory=dict)
    near_blocks: Mapping = field(default_factory=dict)
    couplings: Mapping = field(default_factory=dict)
    build_flops: dict = field(default_factory=dict)

    @property
    def count(self):
        return self.cloud.count

    def rank_of(self, l, i):
        return self.bases[(l, i)].rank

    def near_block(self, l, i, j):
        return self.near_blocks[(l, i, j)] if i >= j else self.near_blocks[(l, j, i)].T

    def coupling(self, l, i, j):
        return self.couplings[(l, i, j)] if i > j else self.couplings[(l, j, i)].T


# --------------------------------------------------------------------------- sampling

def _box_rng(seed, level, box):
    return np.random.default_rng(np.random.SeedSequence((seed, level, box)))


def _stratified(pools, budget, rng):
    """Round-robin draw of `budget` ids over randomly permuted pools
    (h2_build.py:77-96); everything (in pool order) when the budget covers it."""
    total = sum(len(p) for p in pools)
    nonempty = [p for p in pools if len(p)]
    if budget == 0 or budget >= total:
        return np.concatenate(nonempty) if nonempty else np.zeros(0, dtype=np.int64)
    # When the budget is below the pool count, the round-robin stops inside its first
    # pass and only takes element 0 of the first `budget` pools; the permutations of
    # the later pools are drawn after those from a generator used nowhere else, so
    # skipping them leaves the result bit-identical (at N = 1M: 512 of 4095 per box).
    if budget <= len(nonempty):
        nonempty = nonempty[:budget]
    shuffled = [p[rng.permutation(len(p))] for p in nonempty]
    picked = []
    depth = 0
    while len(picked) < budget:
        live = False
        for p in shuffled:
            if depth < len(p):
                picked.append(p[depth])
                live = True
                if len(picked) == budget:
                    break
        depth += 1
        if not live:
            break
    return np.sort(np.asarray(picked, dtype=np.int64))


def sample_far(tree, lists, eff_points, level, box, s_far, seed, near_of=None):
    """Far-field sample: every same-level box outside the near list (h2_build.py:99-106)."""
    mine = near_of[box] if near_of is not None else {j for (i, j) in lists.near[level] if i == box}
    pools = [eff_points[(level, j)] for j in range(2 ** level) if j not in mine]
    return _stratified(pools, s_far, _box_rng(seed, level, box))


def sample_near(tree, lists, eff_points, level, box, s_near, seed, near_of=None):
    """Near-field sample from the near, off-diagonal boxes (h2_build.py:109-113)."""
    mine = near_of[box] if near_of is not None else {j for (i, j) in lists.near[level] if i == box}
    pools = [eff_points[(level, j)] for j in sorted(mine) if j != box]
    return _stratified(pools, s_near, _box_rng(seed, level, box))


def gauss_seidel_solve(a, b, sweeps):
    """`sweeps` forward Gauss-Seidel sweeps for a^-1 b from zero (h2_build.py:116-133)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if np.any(np.diag(a) == 0.0):
        raise SingularTriangularError("zero diagonal in Gauss-Seidel")
    if sweeps < 1:
        raise ValueError("sweeps must be >= 1")
    lower = np.tril(a)
    strict_upper = a - lower
    x = np.zeros_like(b)
    for _ in range(sweeps):
        x = solve_triangular(lower, b - strict_upper @ x, lower=True)
    return x


def prefactor_close(kernel, cloud, box_pts, near_samples, gs_sweeps, flops=None):
    """(G(S_C, B_i) solved against A_cc)^T, i.e. G(B_i, S_C) A_cc^-1 (h2_build.py:136-152)."""
    nb, nc = len(box_pts), len(near_samples)
    if nc == 0:
        return np.zeros((nb, 0))
    a_cc = kernels.gen_block(kernel, near_samples, near_samples, cloud)
    g = kernels.gen_block(kernel, near_samples, box_pts, cloud)
    if gs_sweeps == 0:
        x = scipy.linalg.cho_solve(scipy.linalg.cho_factor(a_cc, lower=True), g)
        cost = nc ** 3 // 3 + 2 * nc * nc * nb
    else:
        x = gauss_seidel_solve(a_cc, g, gs_sweeps)
        cost = gs_sweeps * 2 * nc * nc * nb
    if flops is not None:
        flops["prefactor"] = flops.get("prefactor", 0) + cost
    return x.T


def _far_ancestry(lists, level, box):
    i = box
    for l in range(level, 0, -1):
        if any(a == i for (a, _) in lists.far[l]):
            return True
        i //= 2
    return False


# --------------------------------------------------------------------------- lazy host views

class _LazyMap(Mapping):
    def __init__(self, keys, fetch):
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


def _flat(t, off, rows, cols):
    if rows * cols == 0:
        return np.zeros((rows, cols))
    return t[int(off):int(off) + rows * cols].view(rows, cols).cpu().numpy()


# --------------------------------------------------------------------------- construct

def _skeleton_pass(kernel, tree, lists, cfg, cloud, flops, workers):
    """Host half of construction for every level: skeletons and T."""
    depth = tree.depth
    eff = {(depth, i): np.arange(b.begin, b.end, dtype=np.int64) for i, b in enumerate(tree.leaves)}
    choice = {}
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=1), ThreadPoolExecutor(max_workers=workers) as pool:
        for l in range(depth, 0, -1):
            nb = 2 ** l
            near_of = [set() for _ in range(nb)]
            for (i, j) in lists.near[l]:
                near_of[i].add(j)
            box_flops = [dict() for _ in range(nb)]

            def one(i, l=l, near_of=near_of, box_flops=box_flops):
                pts = eff[(l, i)]
                far_pts = sample_far(tree, lists, eff, l, i, cfg.s_far, cfg.seed, near_of)
                near_pts = sample_near(tree, lists, eff, l, i, cfg.s_near, cfg.seed, near_of)
                close = prefactor_close(kernel, cloud, pts, near_pts, cfg.gs_sweeps, box_flops[i])
                samples = np.hstack([kernels.gen_block(kernel, pts, far_pts, cloud), close])
                if samples.shape[1] == 0:
                    return None
                return skeleton_selection(samples, rank=cfg.rank, tol=cfg.tol)

            results = list(pool.map(one, range(nb)))
            for i, res in enumerate(results):
                flops["prefactor"] = flops.get("prefactor", 0) + box_flops[i].get("prefactor", 0)
                if res is None or res.rank == 0:
                    if _far_ancestry(lists, l, i):
                        raise StructureError(f"box ({l}, {i}) got rank 0 but participates in far interactions")
                choice[(l, i)] = res
            if l > 1:
                for p in range(2 ** (l - 1)):
                    eff[(l - 1, p)] = np.concatenate(
                        [_skel_global(eff, choice, l, 2 * p), _skel_global(eff, choice, l, 2 * p + 1)])
    return eff, choice


def _skel_global(eff, choice, l, i):
    c = choice[(l, i)]
    if c is None:
        return np.zeros(0, dtype=np.int64)
    return eff[(l, i)][c.skeleton]


@ranged("h2ulv.construct")
def construct(kernel, tree, lists, cfg, cloud, device=None, workers=None):
    """Build the H² representation (h2_build.py:170-220); operands end in HBM on
    `device` (default: the current CUDA device), every launch bound to it."""
    nat.lib()
    device = torch.device(device or "cuda")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    with torch.cuda.device(device):
        return _construct(kernel, tree, lists, cfg, cloud, device, workers)


def _construct(kernel, tree, lists, cfg, cloud, device, workers):
    workers = workers or min(32, os.cpu_count() or 1)
    h2 = H2Matrix(tree=tree, lists=lists, kernel=kernel, cloud=cloud, config=cfg)
    h2.build_flops.setdefault("prefactor", 0)
    depth = tree.depth
    pts_dev = torch.from_numpy(np.ascontiguousarray(cloud.points, dtype=np.float64)).to(device)
    flag = torch.zeros(2, dtype=torch.int64, device=device)
    fam = kernels.FAMILY_CODE[kernel.family]
    shift, decay = float(kernel.diagonal_shift), float(kernel.device_param)
    prog = Program(device)
    keep = []  # index arrays referenced by the program

    def idx(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(device)
        keep.append(t)
        return t.data_ptr()

    if depth == 0:
        allpts = np.arange(cloud.count, dtype=np.int64)
        h2.eff_points[(0, 0)] = allpts
        d = cloud.count
        root_a = torch.empty(d * d, dtype=F64, device=device)
        ip = idx(allpts)
        prog.kblock([(ip, ip, root_a.data_ptr(), d, d, d)], pts_dev.data_ptr(), fam, shift, decay, flag.data_ptr())
        prog.finalize().run()
        _check_coincident(flag, kernel, cloud, [(allpts, allpts)])
        h2._device = DeviceH2(device, 0, cloud.count, {}, {}, {}, None, {}, root_a=root_a.view(d, d))
        h2.near_blocks = _LazyMap([(0, 0, 0)], lambda key: root_a.view(d, d).cpu().numpy())
        h2.bases, h2.couplings = {}, {}
        return h2

    eff, choice = _skeleton_pass(kernel, tree, lists, cfg, cloud, h2.build_flops, workers)
    h2.eff_points = eff
    for (l, i), c in choice.items():
        h2.skeletons[(l, i)] = _skel_global(eff, choice, l, i)

    levels, lqs, q, s = {}, {}, {}, {}
    for l in range(depth, 0, -1):
        nb = 2 ** l
        n = [len(eff[(l, i)]) for i in range(nb)]
        k = [0 if choice[(l, i)] is None else choice[(l, i)].rank for i in range(nb)]
        lay = LevelLayout(l, n, k, lists.near[l], lists.far[l])
        levels[l] = lay
        lq = LevelQR(device, n, k)
        lqs[l] = lq
        # T_i (host) -> device, then Z_i = T_i or blockdiag(F_2i, F_2i+1) T_i
        tcat = [choice[(l, i)].t.ravel() for i in range(nb) if k[i] > 0]
        if tcat:
            host = np.concatenate(tcat)
            tdev = torch.from_numpy(host).to(device)
            keep.append(tdev)
        toffs, acc = {}, 0
        for i in range(nb):
            if k[i] > 0:
                toffs[i] = acc
                acc += n[i] * k[i]
        if l == depth:
            for i in range(nb):
                if k[i] > 0:
                    prog.memcpy(lq.ptr(lq.Z, lq.zoff[i]), tdev.data_ptr() + 8 * toffs[i], 8 * n[i] * k[i])
        else:
            child = lqs[l + 1]
            prob = []
            for i in range(nb):
                if k[i] == 0:
                    continue
                ka = int(child.k[2 * i])
                kb = int(child.k[2 * i + 1])
                t0 = tdev.data_ptr() + 8 * toffs[i]
                z0 = lq.ptr(lq.Z, lq.zoff[i])
                if ka:
                    prob.append((child.ptr(child.frame, child.foff[2 * i]), t0, z0, ka, k[i], ka, ka, k[i], k[i],
                                 0, 1.0, 0.0))
                if kb:
                    prob.append((child.ptr(child.frame, child.foff[2 * i + 1]), t0 + 8 * ka * k[i],
                                 z0 + 8 * ka * k[i], kb, k[i], kb, kb, k[i], k[i], 0, 1.0, 0.0))
            prog.gemm(0, 0, prob)
        lq.build(prog)
        if WY_ENABLED and wy_profitable(n, k):
            build_wy(lq, prog)          # compact-WY form for the diag transform (FactorPlan)
        q[l] = lq.qfull
        # couplings S_ij = F_i G(SK_i, SK_j) F_j^T for far pairs i > j
        sbuf = torch.empty(max(lay.ssize, 1), dtype=F64, device=device)
        gbuf = torch.empty(max(lay.ssize, 1), dtype=F64, device=device)
        tmp = torch.empty(max(lay.ssize, 1), dtype=F64, device=device)
        kb_desc, g1, g2 = [], [], []
        skel_ptr = {i: idx(h2.skeletons[(l, i)]) for i in range(nb) if k[i] > 0}
        for (i, j), off in lay.soff.items():
            ki, kj = k[i], k[j]
            if ki == 0 or kj == 0:
                continue
            gp = gbuf.data_ptr() + 8 * off
            kb_desc.append((skel_ptr[i], skel_ptr[j], gp, ki, kj, kj))
            tp = tmp.data_ptr() + 8 * off
            g1.append((lq.ptr(lq.frame, lq.foff[i]), gp, tp, ki, kj, ki, ki, kj, kj, 0, 1.0, 0.0))
            g2.append((tp, lq.ptr(lq.frame, lq.foff[j]), sbuf.data_ptr() + 8 * off, ki, kj, kj, kj, kj, kj,
                       0, 1.0, 0.0))
        prog.kblock(kb_desc, pts_dev.data_ptr(), fam, shift, decay, flag.data_ptr())
        prog.gemm(0, 0, g1)
        prog.gemm(0, 1, g2)
        keep.extend([gbuf, tmp])
        s[l] = sbuf

    # leaf near blocks G(B_i, B_j), i >= j
    leaf = levels[depth]
    aoff, acc = {}, 0
    for (i, j) in leaf.near_pairs:
        aoff[(i, j)] = acc
        acc += int(leaf.n[i] * leaf.n[j])
    leaf_a = torch.empty(max(acc, 1), dtype=F64, device=device)
    box_ptr = {i: idx(eff[(depth, i)]) for i in range(2 ** depth)}
    prog.kblock([(box_ptr[i], box_ptr[j], leaf_a.data_ptr() + 8 * off, int(leaf.n[i]), int(leaf.n[j]),
                  int(leaf.n[j])) for (i, j), off in aoff.items()], pts_dev.data_ptr(), fam, shift, decay,
                flag.data_ptr())
    prog.finalize().run()
    torch.cuda.synchronize(device)
    _check_coincident(flag, kernel, cloud, [(eff[(depth, i)], eff[(depth, j)]) for (i, j) in aoff])

    dh2 = DeviceH2(device, depth, cloud.count, levels, q, s, leaf_a, aoff)
    dh2.wy = {}
    for l, lq in lqs.items():
        if hasattr(lq, "wy_vt"):
            wy_signs(lq)
            dh2.wy[l] = lq
    if dh2.wy:
        # q_full of a compact-WY level IS relabel(I - Yt Y^T) (the product a compact upload of
        # to_pinned_host(h2) rebuilds on the device, so both paths hold the same bits)
        p2 = Program(device)
        for l, lq in dh2.wy.items():
            rebuild_qfull(lq, p2, lambda i, lq=lq: lq.ptr(lq.qfull, lq.qoff[i]))
        p2.finalize().run()
        torch.cuda.synchronize(device)
    h2._device = dh2
    h2._build_keep = (lqs, keep)
    h2._choice = choice
    _attach_host_views(h2, dh2, choice, lqs)
    return h2


def _check_coincident(flag, kernel, cloud, pairs):
    if int(flag[0].item()) == 0:
        return
    for rows, cols in pairs:  # locate the pair exactly like kernels.gen_block does
        kernels.gen_block(kernel, rows, cols, cloud)
    raise CoincidentPointsError(-1, -1)


def _attach_host_views(h2, dh2, choice, lqs):
    depth = dh2.depth

    def basis(key):
        l, i = key
        lay, lq = dh2.levels[l], lqs[l]
        n, k = int(lay.n[i]), int(lay.k[i])
        qf = _flat(lq.qfull, lq.qoff[i], n, n)
        fr = _flat(lq.frame, lq.foff[i], k, k)
        c = choice[key]
        skel = c.skeleton if c is not None else np.zeros(0, dtype=np.int64)
        return BasisDecomposition(q_skel=qf[:, n - k:].copy(), q_red=qf[:, :n - k].copy(), skeleton=skel,
                                  rank=k, frame=fr)

    h2.bases = _LazyMap(sorted(choice), basis)

    near_keys = [(l, i, j) for l in range(depth, 0, -1) for (i, j) in sorted(h2.lists.near[l]) if i >= j]

    def near(key):
        l, i, j = key
        if l == depth:
            lay = dh2.levels[l]
            return _flat(dh2.leaf_a, dh2.aoff[(i, j)], int(lay.n[i]), int(lay.n[j]))
        # upper-level near blocks are not used by factorize/solve; evaluated on request
        return kernels.gen_block(h2.kernel, h2.eff_points[(l, i)], h2.eff_points[(l, j)], h2.cloud)

    h2.near_blocks = _LazyMap(near_keys, near)
    cpl_keys = [(l, i, j) for l in range(depth, 0, -1) for (i, j) in dh2.levels[l].far_pairs]

    def cpl(key):
        l, i, j = key
        lay = dh2.levels[l]
        return _flat(dh2.s[l], lay.soff[(i, j)], int(lay.k[i]), int(lay.k[j]))

    h2.couplings = _LazyMap(cpl_keys, cpl)


def to_pinned_host(h2):
    """Host copy of a GPU-built H², in the reference's numpy data model, whose
    blocks all live in ONE pinned host buffer laid out like the upload
    staging of DeviceH2.from_host (per level, leaves first: bases as q_red
    then q_skel per box, couplings, then the leaf near blocks).

    `bases[(l, i)].q_red / q_skel`, `near_blocks[(depth, i, j)]` and
    `couplings[(l, i, j)]` are numpy views into that buffer, so `factorize`
    of this matrix DMAs each level straight from it (no host gather): the
    "inputs in pinned host memory" starting point of an end-to-end run.
    Only the leaf-level near blocks are included (the factorization never
    reads the upper-level ones, ulv_factor.py:175-176)."""
    dh2 = h2._device
    depth = dh2.depth
    if depth == 0:
        raise ValueError("to_pinned_host: depth-0 trees have a single dense block")
    lqs = h2._build_keep[0]
    regions, total = dh2.staging_regions()
    arena_t = torch.empty(max(total, 1), dtype=F64, pin_memory=True)
    arena = arena_t.numpy()
    dev = dh2.device
    # q_full -> [q_red | q_skel] split per box on the device (the inverse of the upload interleave)
    split = {}
    prog = Program(dev)
    for l, lay in dh2.levels.items():
        sp = torch.empty(max(lay.qsize, 1), dtype=F64, device=dev)
        split[l] = sp
        descs = []
        for i in range(lay.nb):
            n, k = int(lay.n[i]), int(lay.k[i])
            r, o = n - k, int(lay.qoff[i])
            descs.append((dh2.q[l].data_ptr() + 8 * o, sp.data_ptr() + 8 * o, n, r, n, r, 0))
            descs.append((dh2.q[l].data_ptr() + 8 * (o + r), sp.data_ptr() + 8 * (o + n * r), n, k, n, k, 0))
        prog.copy(descs)
    prog.finalize().run()
    for kind, l, base, size in regions:
        if kind == "w":   # compact-WY level: Y, Yt, signs (uploaded instead of q_full)
            lq = lqs[l]
            nk, k = int((lq.n * lq.k).sum()), int(lq.k.sum())
            o = base
            for t, m in ((lq.V, nk), (lq.wy_vt, nk), (lq.wy_sgn, k)):
                arena_t[o:o + m].copy_(t[:m])
                o += m
            continue
        src = split[l] if kind == "q" else dh2.s[l] if kind == "s" else dh2.leaf_a
        arena_t[base:base + size].copy_(src[:size])
    torch.cuda.synchronize(dev)
    out = H2Matrix(tree=h2.tree, lists=h2.lists, kernel=h2.kernel, cloud=h2.cloud, config=h2.config)
    out.skeletons, out.eff_points, out.build_flops = h2.skeletons, h2.eff_points, dict(h2.build_flops)
    base_of = {(kind, l): base for kind, l, base, _ in regions}
    flag = [False]
    bases, near, cpl = _TrackedDict(), _TrackedDict(), _TrackedDict()
    for l, lay in dh2.levels.items():
        b0 = base_of[("q", l)]
        lq = lqs[l]
        fr_all = lq.frame.cpu().numpy()
        for i in range(lay.nb):
            n, k = int(lay.n[i]), int(lay.k[i])
            r, o = n - k, b0 + int(lay.qoff[i])
            c = h2._choice[(l, i)]
            fr = fr_all[lq.foff[i]:lq.foff[i] + k * k].reshape(k, k)
            qs, qr = arena[o + n * r:o + n * n].reshape(n, k), arena[o:o + n * r].reshape(n, r)
            if l in dh2.wy:
                # the device rebuilds this level's q_full from the arena's Y / Yt: in-place edits
                # of these views could not reach it, so they are read-only (rebinding still works
                # and sends factorize back to the full upload)
                qs.flags.writeable = False
                qr.flags.writeable = False
            bd = _TrackedBasis(q_skel=qs, q_red=qr, rank=k, frame=fr,
                               skeleton=c.skeleton if c is not None else np.zeros(0, dtype=np.int64))
            object.__setattr__(bd, "_flag", flag)
            dict.__setitem__(bases, (l, i), bd)
        s0 = base_of[("s", l)]
        for (i, j), o in lay.soff.items():
            blk = arena[s0 + o:s0 + o + int(lay.k[i] * lay.k[j])].reshape(int(lay.k[i]), int(lay.k[j]))
            dict.__setitem__(cpl, (l, i, j), blk)
    a0, leaf = base_of[("a", depth)], dh2.levels[depth]
    for (i, j), o in dh2.aoff.items():
        blk = arena[a0 + o:a0 + o + int(leaf.n[i] * leaf.n[j])].reshape(int(leaf.n[i]), int(leaf.n[j]))
        dict.__setitem__(near, (depth, i, j), blk)
    for d in (bases, near, cpl):
        d._flag = flag
    out.bases, out.near_blocks, out.couplings = bases, near, cpl
    out._arena = PinnedArena(arena_t, dh2.signature(),
                             {"bases": bases, "near_blocks": near, "couplings": cpl}, flag)
    out._arena.wy_levels = tuple(sorted(dh2.wy))
    return out


class _TrackedDict(dict):
    """dict that flags its arena when an entry is replaced, added or removed."""

    _flag = None

    def _mark(self):
        if self._flag is not None:
            self._flag[0] = True

    def __setitem__(self, key, value):
        self._mark()
        super().__setitem__(key, value)

    def __delitem__(self, key):
        self._mark()
        super().__delitem__(key)

    def _mutator(name):
        def f(self, *a, **kw):
            self._mark()
            return getattr(dict, name)(self, *a, **kw)
        f.__name__ = name
        return f

    pop = _mutator("pop")
    popitem = _mutator("popitem")
    clear = _mutator("clear")
    update = _mutator("update")
    setdefault = _mutator("setdefault")
    __ior__ = _mutator("__ior__")
    del _mutator


class _TrackedBasis(BasisDecomposition):
    """BasisDecomposition whose q_red / q_skel are arena views: rebinding either flags the arena."""

    _flag = None

    def __setattr__(self, name, value):
        if name in ("q_red", "q_skel") and self._flag is not None:
            self._flag[0] = True
        object.__setattr__(self, name, value)


class PinnedArena:
    """The pinned buffer behind a `to_pinned_host` matrix plus the containers it
    handed out.  `intact(h2)` is true while `h2` still holds those containers and
    no block in them was rebound (a rebound block sends factorize back to the
    gather path).  O(1): the containers flag their own mutation.  In-place edits
    of a block's values write through to the buffer, so they stay intact."""

    def __init__(self, tensor, signature, containers, flag):
        self.wy_levels = ()               # levels shipped in compact-WY form (to_pinned_host)
        self.tensor = tensor
        self.signature = signature
        self.containers = containers      # attribute name -> _TrackedDict handed out
        self._flag = flag                 # [bool], shared with the containers and bases

    def intact(self, h2):
        if self._flag[0]:
            return False
        return all(getattr(h2, name, None) is d for name, d in self.containers.items())


# --------------------------------------------------------------------------- matvec

def h2_matvec(h2, x):
    """y = A x through the hierarchical representation, tree order
    (h2_build.py:232-282), on the GPU: one grouped GEMV launch per level and
    pass (matvec_device.MatvecPlan).  A GPU-built H² uses the operands already
    in HBM; a host (numpy) H² — the reference's data model, e.g. one read back
    by storage.load_h2 — is uploaded with DeviceH2.from_host on every call, so
    the product stays a pure function of the blocks and the two agree bit for
    bit (test_storage.py:49-55).  There is no host path."""
    from .matvec_device import device_matvec

    xm = np.asarray(x, dtype=np.float64)
    if xm.reshape(xm.shape[0], -1).shape[0] != h2.count:
        raise ValueError("length mismatch")
    return device_matvec(h2, xm)


def build_basis_for_box(kernel, cloud, box_pts, far_pts, close_block, rank=None, tol=None, row_weight=None):
    """Composite basis from [G(B_i, far) | close_block] via the ID
    (h2_build.py:155-167): host skeleton choice (bit-exact dgeqp3), the
    complementary basis by the GPU Householder QR (dense_core.id_basis)."""
    far_block = kernels.gen_block(kernel, box_pts, far_pts, cloud)
    samples = np.hstack([far_block, np.asarray(close_block, dtype=np.float64).reshape(len(box_pts), -1)])
    if samples.shape[1] == 0:
        n = len(box_pts)
        return dense_core.BasisDecomposition(q_skel=np.zeros((n, 0)), q_red=np.eye(n),
                                             skeleton=np.zeros(0, dtype=np.int64), rank=0, frame=np.zeros((0, 0)))
    return dense_core.id_basis(samples, rank=rank, tol=tol, row_weight=row_weight)
