"""(f)3 storage of device-resident factors (reference storage.py:158-218,
test_storage.py:23-98): the container round trip is bit-exact, reloaded
(host) factors solve to the same bits on the GPU, and the reference's own
factors, loaded as host blocks, solve on the GPU to the reference's x."""
import numpy as np
import pytest

from fixtures import H2_FIXTURES, load_h2, reference_factors

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def built():
    import paper_2502_02395_b200 as pkg
    cloud = pkg.gen_sphere_surface(2048, seed=0)
    tree = pkg.build_tree(cloud, 128)
    lists = pkg.build_interaction_lists(tree, 1.0)
    h2 = pkg.construct(pkg.KernelSpec(family="laplace", diagonal_shift=1e3), tree, lists,
                       pkg.BuildConfig(eta=1.0, leaf_max=128, tol=1e-8, s_far=256, s_near=256), cloud)
    return pkg, h2, pkg.factorize(h2)


def test_factor_container_bit_exact(built, tmp_path):
    from paper_2502_02395_b200 import storage
    pkg, h2, f = built
    storage.save_h2(h2, tmp_path)
    storage.save_ulv(f, tmp_path)
    h2b, back = storage.load_factors(tmp_path)
    assert set(back.levels) == set(f.levels)
    for l, lvl in f.levels.items():
        blv = back.levels[l]
        assert blv.dims == lvl.dims
        for name in ("lr_diag", "lr_off", "ls", "v"):
            src, dst = getattr(lvl, name), getattr(blv, name)
            assert set(src) == set(dst), (l, name)
            for key in src:
                assert np.array_equal(dst[key], src[key]), (l, name, key)
    assert np.array_equal(back.root, f.root)
    assert back.flops["total_true"] == f.flops["total_true"]
    b = np.random.default_rng(2).standard_normal(h2.count)
    x = pkg.solve(f, b)
    assert np.array_equal(pkg.solve(back, b), x)                 # reloaded host factors: same bits
    x2 = pkg.solve(f, b)
    assert np.array_equal(x2, x)
    assert np.array_equal(pkg.h2_matvec(h2b, x), pkg.h2_matvec(h2, x))


@pytest.mark.parametrize("name", H2_FIXTURES)
def test_reference_factors_solve_on_gpu(name):
    """Host factors holding the REFERENCE's own blocks (golden fixtures) solve on the
    GPU to the reference's solution."""
    import paper_2502_02395_b200 as pkg
    from paper_2502_02395_b200.ulv_factor import ULVFactors, ULVLevel
    h2 = load_h2(name)
    ref = reference_factors(name)
    f = ULVFactors(h2=h2)
    for l in range(1, h2.tree.depth + 1):
        lvl = ULVLevel()
        lvl.lr_diag = {i: v for (ll, i), v in ref["lr_diag"].items() if ll == l}
        lvl.lr_off = {(i, j): v for (ll, i, j), v in ref["lr_off"].items() if ll == l}
        lvl.ls = {(a, b): v for (ll, a, b), v in ref["ls"].items() if ll == l}
        f.levels[l] = lvl
    f.root = ref["root"]
    x = pkg.solve(f, ref["b"])
    assert np.linalg.norm(x - ref["x"]) / np.linalg.norm(ref["x"]) < 1e-10
