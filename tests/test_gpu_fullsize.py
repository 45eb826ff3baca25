"""Full-size parity at the BASELINE.json configurations, pinned to fixtures
produced by running the unmodified reference (tests/golden/make_golden.py):

  c2        configs[1]  Laplace cube N = 65 536, tol 1e-8, shift 1e5, 512/512
  c3        configs[2]  Yukawa sphere N = 262 144, tol 1e-8, shift 1e5, 512/512
  m1        the metric  Laplace cube N = 1 048 576, tol 1e-8, shift 2e6, 512/512
  m1_tol6   configs[4]  the same at tol 1e-6   (weak-scaling sweep, P = 1)
  m1_tol10  configs[4]  the same at tol 1e-10

For each: the GPU construct's tree, interaction lists, ranks and skeleton
indices are bit-identical to the reference's (sha256 of the same arrays the
generator hashed), the flop report equals the reference's dict exactly, and
the factor + solve residual ||h2_matvec(x) - b|| / ||b|| (cli.py:199-205) is
within 10x of the reference's (the north_star tolerance).

The two breakdown edges of BASELINE.md §3 raise the reference's
NotPositiveDefiniteError at the same (pivot, level, box):
  c2_npd         C2 at shift 1e3 (genuinely indefinite: level 8, box 40)
  sphere65k_npd  Yukawa sphere N = 65 536 at shift 1e3 (approximate-ULV breakdown: level 4, box 1)
"""
import hashlib

import numpy as np
import pytest

from fixtures import flops_equal, meta

pytestmark = pytest.mark.gpu


def sha(*arrays_):
    h = hashlib.sha256()
    for a in arrays_:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def pkg():
    import paper_2502_02395_b200 as p
    return p


def _build(pkg, name):
    cfg = meta(name)["config"]
    gen = pkg.gen_uniform_cube if cfg["shape"] == "cube" else pkg.gen_sphere_surface
    cloud = gen(cfg["n"], seed=0)
    tree = pkg.build_tree(cloud, cfg["leaf"])
    lists = pkg.build_interaction_lists(tree, cfg["eta"])
    kw = {key: cfg[key] for key in ("rank", "tol", "s_far", "s_near") if key in cfg}
    bc = pkg.BuildConfig(eta=cfg["eta"], leaf_max=cfg["leaf"], seed=0, **kw)
    kernel = pkg.KernelSpec(family=cfg["family"], diagonal_shift=cfg["shift"])
    return pkg.construct(kernel, tree, lists, bc, cloud)


def _structure_sha(h2):
    tree, lists = h2.tree, h2.lists
    rng = np.array([(l, b.index_in_level, b.begin, b.end) for l in range(tree.depth + 1) for b in tree.boxes[l]],
                   dtype=np.int64)
    near = np.array([(l, i, j) for l in range(tree.depth + 1) for (i, j) in sorted(lists.near[l])],
                    dtype=np.int64).reshape(-1, 3)
    far = np.array([(l, i, j) for l in range(tree.depth + 1) for (i, j) in sorted(lists.far[l])],
                   dtype=np.int64).reshape(-1, 3)
    loc, glob, ranks = [], [], []
    for l in range(tree.depth, 0, -1):
        for i in range(2 ** l):
            b = h2.bases[(l, i)]
            ranks.append(b.rank)
            loc.append(np.asarray(b.skeleton, dtype=np.int64))
            glob.append(np.asarray(h2.skeletons[(l, i)], dtype=np.int64))
    return {"perm": sha(h2.cloud.perm), "box_ranges": sha(rng), "near": sha(near), "far": sha(far),
            "ranks": sha(np.array(ranks, np.int64)), "skeleton_local": sha(np.concatenate(loc)),
            "skeleton_global": sha(np.concatenate(glob))}


def _per_level_mismatch(h2, m):
    bad = []
    for l, want in m.get("skeleton_sha_per_level", {}).items():
        sk = [np.asarray(h2.bases[(int(l), i)].skeleton, dtype=np.int64) for i in range(2 ** int(l))]
        got = sha(np.concatenate(sk), np.array([len(s) for s in sk], np.int64))
        if got != want:
            bad.append(int(l))
    return bad


@pytest.mark.parametrize("name", ["c2", "c3", "m1", "m1_tol6", "m1_tol10"])
def test_fullsize_structure_flops_residual(pkg, name):
    from paper_2502_02395_b200.ulv_factor import clear_cache

    clear_cache()
    m = meta(name)
    h2 = _build(pkg, name)
    got = _structure_sha(h2)
    for key, want in m["sha"].items():
        if key in got:
            assert got[key] == want, (name, key, "levels with different skeletons:", _per_level_mismatch(h2, m))
    f = pkg.factorize(h2)
    assert flops_equal(f.flops, m["flops"]), name
    for l, dims in m["dims"].items():
        assert [list(f.levels[int(l)].dims[i]) for i in range(len(dims))] == dims
    assert f.root.shape[0] == m["root_dim"]
    b = np.random.default_rng(1).standard_normal(m["config"]["n"])
    x = pkg.solve(f, b)
    perm = h2.cloud.perm
    res = float(np.linalg.norm(pkg.h2_matvec(h2, x[perm]) - b[perm]) / np.linalg.norm(b))
    assert res <= 10 * m["residual"], (name, res, m["residual"])
    if name == "c2":
        # multi-RHS through every solve path at full size (TRSV levels, explicit-inverse
        # levels, neighbour-free levels, balanced GEMVs with w > 1): column j == solve(b_j)
        b2 = np.random.default_rng(2).standard_normal(m["config"]["n"])
        xm = pkg.solve(f, np.stack([b, b2, -3.0 * b, b2, b], axis=1))
        for j, bj in enumerate((b, b2, -3.0 * b, b2, b)):
            xj = x if j in (0, 4) else pkg.solve(f, bj) if j != 2 else -3.0 * x
            assert np.linalg.norm(xm[:, j] - xj) <= 1e-12 * np.linalg.norm(xj), j
        for mode in ("naive",):
            xn = pkg.solve(f, b, mode=mode)
            assert np.linalg.norm(xn - x) <= 1e-9 * np.linalg.norm(x)
    del f, h2
    clear_cache()


@pytest.mark.parametrize("name", ["c2_npd", "sphere65k_npd"])
def test_breakdown_edges_like_reference(pkg, name):
    from paper_2502_02395_b200.ulv_factor import clear_cache

    clear_cache()
    m = meta(name)
    h2 = _build(pkg, name)
    got = _structure_sha(h2)
    assert got["skeleton_global"] == m["sha"]["skeleton_global"] and got["ranks"] == m["sha"]["ranks"]
    with pytest.raises(pkg.NotPositiveDefiniteError) as e:
        pkg.factorize(h2)
    want = m["npd"]
    assert (e.value.pivot, e.value.level, e.value.box) == (want["pivot"], want["level"], want["box"])
    del h2
    clear_cache()


def test_m1_root_breakdown_at_shift_1e5(pkg):
    """the reference at the metric's N = 1M with shift 1e5 (instead of 2e6)
    factors all 12 levels and breaks down at the ROOT (level 0, pivot 60).  Same
    structure through the GPU construct; the breakdown is raised from the native
    session's status decode with the reference's (pivot, level, box)."""
    from paper_2502_02395_b200.ulv_factor import clear_cache

    clear_cache()
    cloud = pkg.gen_uniform_cube(1048576, seed=0)
    tree = pkg.build_tree(cloud, 256)
    lists = pkg.build_interaction_lists(tree, 1.0)
    bc = pkg.BuildConfig(eta=1.0, leaf_max=256, tol=1e-8, s_far=512, s_near=512, seed=0)
    h2 = pkg.construct(pkg.KernelSpec(family="laplace", diagonal_shift=1e5), tree, lists, bc, cloud)
    with pytest.raises(pkg.NotPositiveDefiniteError) as e:
        pkg.factorize(h2)
    assert (e.value.level, e.value.box) == (0, 0)
    assert e.value.pivot == 60
    del h2
    clear_cache()
