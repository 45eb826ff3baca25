"""The CPU oracle is pinned against the reference's own outputs (golden
fixtures made by tests/golden/make_golden.py) before it is trusted as the
checker of the GPU path."""
import numpy as np
import pytest

from fixtures import H2_FIXTURES, arrays, flops_equal, load_h2, meta, reference_factors
from oracle import h2ulv_oracle as orc
from paper_2502_02395_b200.errors import NotPositiveDefiniteError


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("name", H2_FIXTURES)
def test_oracle_factors_match_reference(name):
    h2 = load_h2(name)
    ref = reference_factors(name)
    f = orc.factorize(h2)
    for (l, i), v in ref["lr_diag"].items():
        assert _rel(f.levels[l]["lr_diag"][i], v) < 1e-12
    for (l, i, j), v in ref["lr_off"].items():
        assert _rel(f.levels[l]["lr_off"][(i, j)], v) < 1e-11
    for (l, a, b), v in ref["ls"].items():
        assert _rel(f.levels[l]["ls"][(a, b)], v) < 1e-11
    assert _rel(f.root, ref["root"]) < 1e-11
    assert flops_equal(f.flops, meta(name)["flops"])


@pytest.mark.parametrize("name", H2_FIXTURES)
@pytest.mark.parametrize("mode", ["parallel", "naive"])
def test_oracle_solve_matches_reference(name, mode):
    h2 = load_h2(name)
    ref = reference_factors(name)
    f = orc.factorize(h2)
    x = orc.solve(f, ref["b"], mode=mode)
    want = ref["x"] if mode == "parallel" else ref["x_naive"]
    assert _rel(x, want) < 1e-11
    res = orc.residual(h2, x, ref["b"])
    assert res == pytest.approx(meta(name)["residual"], rel=1e-3, abs=1e-14)


def test_known_answer_cholesky():
    z = arrays("known_answers")
    l2 = orc.chol(z["chol2_a"])
    assert np.allclose(l2, [[2.0, 0.0], [1.0, np.sqrt(2.0)]], atol=1e-15)
    assert np.allclose(l2, z["chol2_l"], atol=1e-15)
    assert np.allclose(orc.chol(z["chol12_a"]), z["chol12_l"], rtol=1e-13, atol=1e-13)
    with pytest.raises(NotPositiveDefiniteError) as exc:
        orc.chol(np.array([[1.0, 2.0], [2.0, 1.0]]), 4, 7)
    assert exc.value.pivot >= 1 and "level 4" in str(exc.value)


def test_known_answer_complete_qr():
    """q_skel and frame are unique under the sign convention (dense_core.py:140-144)."""
    from paper_2502_02395_b200.dense_core import skeleton_selection

    z = arrays("known_answers")
    for pre, w in (("id", None), ("idw", z["idw_w"])):
        ch = skeleton_selection(z["id_s"], tol=1e-6)
        assert np.array_equal(ch.skeleton, z[f"{pre}_skel"])
        zz = ch.t if w is None else w @ ch.t
        qf, fr = orc.complete_qr(zz, ch.rank)
        n, k = zz.shape[0], ch.rank
        assert np.allclose(qf[:, n - k:], z[f"{pre}_qskel"], atol=1e-12)
        assert np.allclose(fr, z[f"{pre}_frame"], atol=1e-12)
        assert np.allclose(qf.T @ qf, np.eye(n), atol=1e-12)


def test_flop_known_answers():
    assert orc._flops("cholesky", (6,)) == 72
    assert orc._flops("multiply", (2, 3, 4)) == 48
    assert orc._flops("tri_solve", (4, 2)) == 32
