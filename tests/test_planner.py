"""CPU checks of planner geometry: Program.gemm's edge carving (program.carve_edges)
covers every output element exactly once with sub-problems of the same operands,
for every transpose combination (numpy stand-in for the grouped GEMM)."""
import numpy as np
import pytest

from paper_2502_02395_b200 import _native as nat
from paper_2502_02395_b200.program import carve_edges

BASE_A, BASE_B, BASE_C = 0, 1 << 24, 2 << 24


def _run(q, A, B, ta, tb, N):
    """Evaluate one problem tuple (pointers relative to the bases) with numpy."""
    a0, b0, c0 = (q[0] - BASE_A) // 8, (q[1] - BASE_B) // 8, (q[2] - BASE_C) // 8
    m, n, k, lda, ldb = q[3], q[4], q[5], q[6], q[7]
    Af, Bf = A.ravel(), B.ravel()
    ia, ka = np.meshgrid(np.arange(m), np.arange(k), indexing="ij")
    As = Af[a0 + (ka * lda + ia if ta else ia * lda + ka)]
    kb, jb = np.meshgrid(np.arange(k), np.arange(n), indexing="ij")
    Bs = Bf[b0 + (jb * ldb + kb if tb else kb * ldb + jb)]
    r0, col0 = divmod(c0, N)
    return r0, col0, As @ Bs


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(457, 300, 70), (100, 96, 10), (200, 200, 33), (64, 97, 5), (130, 64, 8)])
def test_carved_pieces_tile_the_output(ta, tb, M, N, K):
    rng = np.random.default_rng(M + N + K + 2 * ta + tb)
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    p = (BASE_A, BASE_B, BASE_C, M, N, K, A.shape[1], B.shape[1], N, 0, 1.0, 0.0)
    c = carve_edges(p, ta, tb)
    rm, rn = M % 64, N % 64
    if not ((0 < rm <= 32) or (0 < rn <= 32)):
        assert c is None
        return
    interior, edges = c
    assert interior[3] % 64 == 0 or interior[3] == M
    assert interior[4] % 64 == 0 or interior[4] == N
    C = np.zeros((M, N))
    cover = np.zeros((M, N), dtype=int)
    for q in [interior] + edges:
        assert q[6:12] == p[6:12]                  # same leading dimensions, flags, alpha, beta
        r0, col0, blk = _run(q, A, B, ta, tb, N)
        C[r0:r0 + q[3], col0:col0 + q[4]] += blk
        cover[r0:r0 + q[3], col0:col0 + q[4]] += 1
    assert (cover == 1).all()
    np.testing.assert_allclose(C, (A.T if ta else A) @ (B.T if tb else B), rtol=1e-13, atol=1e-12)


def test_lower_and_ext_problems_are_not_carved():
    p = (BASE_A, BASE_B, BASE_C, 457, 457, 10, 10, 457, 457, nat.GEMM_LOWER, 1.0, 0.0)
    assert carve_edges(p, 0, 0) is None
    q = (BASE_A, BASE_B, BASE_C, 457, 300, 10, 10, 300, 300, 0, -1.0, 1.0, (0, 0, 300, -1))
    assert carve_edges(q, 0, 0) is None
