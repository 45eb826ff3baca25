"""Host-side parity (no GPU): tree, interaction lists and skeleton indices
are bit-identical to the reference's (golden fixtures c1 = BASELINE C1,
c2 = BASELINE C2), and the flop model reproduces the reference's report."""
import hashlib

import numpy as np
import pytest

import paper_2502_02395_b200 as pkg
from fixtures import arrays, meta
from paper_2502_02395_b200.h2_build import _skel_global, _skeleton_pass
from paper_2502_02395_b200.ulv_factor import flop_report


def sha(*arrays_):
    h = hashlib.sha256()
    for a in arrays_:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def _setup(name):
    cfg = meta(name)["config"]
    gen = pkg.gen_uniform_cube if cfg["shape"] == "cube" else pkg.gen_sphere_surface
    cloud = gen(cfg["n"], seed=0)
    tree = pkg.build_tree(cloud, cfg["leaf"])
    lists = pkg.build_interaction_lists(tree, cfg["eta"])
    kw = {key: cfg[key] for key in ("rank", "tol", "s_far", "s_near") if key in cfg}
    bc = pkg.BuildConfig(eta=cfg["eta"], leaf_max=cfg["leaf"], seed=0, **kw)
    kernel = pkg.KernelSpec(family=cfg["family"], diagonal_shift=cfg["shift"])
    return cloud, tree, lists, bc, kernel


def _structure(tree, lists):
    rng = np.array([(l, b.index_in_level, b.begin, b.end) for l in range(tree.depth + 1) for b in tree.boxes[l]],
                   dtype=np.int64)
    near = np.array([(l, i, j) for l in range(tree.depth + 1) for (i, j) in sorted(lists.near[l])],
                    dtype=np.int64).reshape(-1, 3)
    far = np.array([(l, i, j) for l in range(tree.depth + 1) for (i, j) in sorted(lists.far[l])],
                   dtype=np.int64).reshape(-1, 3)
    return rng, near, far


def _skeletons(tree, eff, choice):
    loc, glob, ranks = [], [], []
    for l in range(tree.depth, 0, -1):
        for i in range(2 ** l):
            c = choice[(l, i)]
            ranks.append(0 if c is None else c.rank)
            loc.append(np.zeros(0, np.int64) if c is None else c.skeleton)
            glob.append(_skel_global(eff, choice, l, i))
    return np.concatenate(loc).astype(np.int64), np.concatenate(glob).astype(np.int64), np.array(ranks, np.int64)


def test_c1_tree_lists_exact():
    cloud, tree, lists, _, _ = _setup("c1")
    z = arrays("c1")
    rng, near, far = _structure(tree, lists)
    assert np.array_equal(cloud.perm, z["perm"])
    assert np.array_equal(rng, z["box_ranges"])
    assert np.array_equal(near, z["near"]) and np.array_equal(far, z["far"])


def test_c2_tree_lists_exact():
    cloud, tree, lists, _, _ = _setup("c2")
    s = meta("c2")["sha"]
    rng, near, far = _structure(tree, lists)
    assert sha(cloud.perm) == s["perm"] and sha(cloud.points) == s["points"]
    assert sha(rng) == s["box_ranges"] and sha(near) == s["near"] and sha(far) == s["far"]


def test_c1_skeletons_exact():
    cloud, tree, lists, bc, kernel = _setup("c1")
    z = arrays("c1")
    flops = {}
    eff, choice = _skeleton_pass(kernel, tree, lists, bc, cloud, flops, workers=8)
    loc, glob, ranks = _skeletons(tree, eff, choice)
    assert np.array_equal(ranks, z["ranks"])
    assert np.array_equal(loc, z["skel_local"]) and np.array_equal(glob, z["skel_global"])


def test_c2_skeletons_exact():
    """BASELINE C2 (N = 65536, sampled 512/512): the full host pass, ~10 s on 8 cores."""
    cloud, tree, lists, bc, kernel = _setup("c2")
    s = meta("c2")["sha"]
    eff, choice = _skeleton_pass(kernel, tree, lists, bc, cloud, {}, workers=8)
    loc, glob, ranks = _skeletons(tree, eff, choice)
    assert sha(ranks) == s["ranks"]
    assert sha(loc) == s["skeleton_local"] and sha(glob) == s["skeleton_global"]


@pytest.mark.parametrize("name", ["c1", "c2", "h2_cube512_rank16", "h2_sphere1024_yukawa_tol"])
def test_flop_model_reproduces_reference(name):
    m = meta(name)
    cloud, tree, lists, _, _ = _setup(name) if name in ("c1", "c2") else (None, None, None, None, None)
    if lists is None:
        from fixtures import load_h2
        h2 = load_h2(name)
        lists = h2.lists
    levels = {}
    for l, dims in m["dims"].items():
        d = np.array(dims, dtype=np.int64)
        r, k = d[:, 0], d[:, 1]
        offp = sorted((i, j) for (i, j) in lists.near[int(l)] if i > j)
        levels[int(l)] = (r + k, k, offp)
    root = int(sum(levels[1][1])) if levels else 0
    got = flop_report(levels, root)
    want = m["flops"]
    assert got["total_true"] == want["total_true"] and got["total_padded"] == want["total_padded"]
    for l, phases in want["levels"].items():
        for ph, ent in phases.items():
            assert got["levels"][int(l)][ph] == ent, (l, ph)


def test_stratified_sampling_matches_reference_algorithm():
    """h2_build._stratified skips the permutations of pools the round-robin never
    reaches (budget < pool count); the draw must stay bit-identical to the
    reference's _stratified (h2_build.py:77-96), restated here literally."""
    from paper_2502_02395_b200.h2_build import _stratified

    def reference(pools, budget, rng):
        total = sum(len(p) for p in pools)
        nonempty = [p for p in pools if len(p)]
        if budget == 0 or budget >= total:
            return np.concatenate(nonempty) if nonempty else np.zeros(0, dtype=np.int64)
        shuffled = [p[rng.permutation(len(p))] for p in nonempty]
        picked, depth = [], 0
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

    g = np.random.default_rng(0)
    for trial in range(200):
        sizes = g.integers(0, 40, size=int(g.integers(1, 600)))
        starts = np.concatenate([[0], np.cumsum(sizes)[:-1]])
        pools = [np.arange(s0, s0 + sz, dtype=np.int64) for s0, sz in zip(starts, sizes)]
        budget = int(g.integers(0, 700))
        seed = np.random.SeedSequence((trial, 3, 7))
        a = reference(pools, budget, np.random.default_rng(seed))
        b = _stratified(pools, budget, np.random.default_rng(np.random.SeedSequence((trial, 3, 7))))
        assert np.array_equal(a, b), trial
