"""Kernel-level GPU checks of the Cholesky panel step and the left-looking row
solve against numpy FP64 (the math of dense_core.cholesky / tri_solve,
dense_core.py:51-81).  Tolerances are relative to the operand scale."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL = 1e-12


@pytest.fixture(scope="module")
def env():
    import torch

    from paper_2502_02395_b200 import _native as nat
    from paper_2502_02395_b200.program import Program

    nat.lib()
    return torch, nat, Program


def _spd(n, seed, shift=None):
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, n))
    return g @ g.T + (shift if shift is not None else n) * np.eye(n)


@pytest.mark.parametrize("n,p,b", [(256, 0, 64), (256, 64, 64), (200, 128, 40), (64, 0, 64), (70, 64, 6)])
def test_chol_panel_step(env, n, p, b):
    """PANEL(q) = previous-panel update of block column q + chol + TRSM of the rows below."""
    torch, nat, Program = env
    a = _spd(n, n + p + b)
    lf = np.linalg.cholesky(a)
    # H after panels < q-1 are complete and their REST updates applied:
    # block column q still lacks the update of panel q-1.
    h = a.copy()
    if p > 0:
        pp = p - 64
        h[:, :p] = np.tril(lf[:, :p], 0) if p else h[:, :p]
        s = lf[:, :pp] @ lf[:, :pp].T if pp > 0 else np.zeros((n, n))
        h[p:, p:] = a[p:, p:] - s[p:, p:]
    hd = torch.from_numpy(h.copy()).cuda()
    linv = torch.zeros(64 * 64, dtype=torch.float64, device="cuda")
    npd = torch.full((1,), 2 ** 31 - 1, dtype=torch.int32, device="cuda")
    prog = Program(torch.device("cuda"))
    prog.chol_panel([(hd.data_ptr(), linv.data_ptr(), n, 64, n, p, b, 0)], npd.data_ptr())
    prog.finalize().run()
    torch.cuda.synchronize()
    out = hd.cpu().numpy()
    assert int(npd.item()) == 2 ** 31 - 1
    scale = np.abs(lf).max()
    np.testing.assert_allclose(np.tril(out[p:p + b, p:p + b]), lf[p:p + b, p:p + b], rtol=0, atol=RTOL * scale * 10)
    if n > p + b:
        np.testing.assert_allclose(out[p + b:, p:p + b], lf[p + b:, p:p + b], rtol=0, atol=RTOL * scale * 10)
    li = linv.cpu().numpy().reshape(64, 64)[:b, :b]
    np.testing.assert_allclose(li @ lf[p:p + b, p:p + b], np.eye(b), rtol=0, atol=1e-12)


def test_chol_panel_reports_first_bad_pivot(env):
    torch, nat, Program = env
    n, bad = 96, 37
    a = _spd(n, 5)
    a[bad, bad] = -1.0e3                       # pivot 37 of the first panel turns negative
    hd = torch.from_numpy(a).cuda()
    linv = torch.zeros(64 * 64, dtype=torch.float64, device="cuda")
    npd = torch.full((1,), 2 ** 31 - 1, dtype=torch.int32, device="cuda")
    prog = Program(torch.device("cuda"))
    prog.chol_panel([(hd.data_ptr(), linv.data_ptr(), n, 64, n, 0, 64, 0)], npd.data_ptr())
    prog.finalize().run()
    torch.cuda.synchronize()
    assert int(npd.item()) == bad


@pytest.mark.parametrize("rows,cols,qb,qe,ident", [(256, 213, 0, 4, False), (100, 64, 0, 1, False),
                                                    (70, 150, 0, 3, False), (300, 300, 0, 5, True),
                                                    (200, 200, 2, 3, True)])
def test_trsm_rows(env, rows, cols, qb, qe, ident):
    """X = B L^-T, block columns [qb, qe) (left-looking, h2g_trsm_rows); B = I when ident."""
    torch, nat, Program = env
    rng = np.random.default_rng(rows + cols + qb)
    L = np.tril(rng.standard_normal((cols, cols))) * 0.1 + 2 * np.eye(cols)
    nq = -(-cols // 64)
    linv = np.zeros((nq, 64, 64))
    for q in range(nq):
        p, b = 64 * q, min(64, cols - 64 * q)
        linv[q, :b, :b] = np.linalg.inv(L[p:p + b, p:p + b])
    B = np.eye(rows, cols) if ident else rng.standard_normal((rows, cols))
    ref = np.linalg.solve(L, B.T).T          # B L^-T
    t = lambda m: torch.from_numpy(np.ascontiguousarray(m)).cuda()
    Ld, Bd, Lid = t(L), t(B), t(linv)
    X = torch.zeros_like(Bd)
    if qb > 0:                               # columns < 64 qb already solved
        X[:, :64 * qb] = t(ref[:, :64 * qb])
    prog = Program(torch.device("cuda"))
    prog.trsm_rows([(Ld.data_ptr(), 0 if ident else Bd.data_ptr(), X.data_ptr(), Lid.data_ptr(), rows, cols, qb, qe,
                     cols, cols)])
    prog.finalize().run()
    torch.cuda.synchronize()
    hi = min(cols, 64 * qe)
    got = X.cpu().numpy()
    np.testing.assert_allclose(got[:, 64 * qb:hi], ref[:, 64 * qb:hi], rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))


@pytest.mark.parametrize("nbox", [100, 200])
def test_chol_panel_many_boxes_rerun(env, nbox):
    """nbox <= h2g_chol_panel_fused_max(): the one-launch ticket/flag variant; above: two kernels.
    The program runs three times to check the sync words are left zeroed between launches."""
    torch, nat, Program = env
    n, p, b = 200, 64, 64
    rng = np.random.default_rng(nbox)
    hs, lfs = [], []
    for _ in range(nbox):
        g = rng.standard_normal((n, n))
        a = g @ g.T + n * np.eye(n)
        lf = np.linalg.cholesky(a)
        h = a.copy()
        h[:, :p] = np.tril(lf[:, :p])
        h[p:, p:] = a[p:, p:]                  # the panel before p is the first one: nothing applied yet
        hs.append(h)
        lfs.append(lf)
    h0 = torch.from_numpy(np.stack(hs)).cuda()
    hd = h0.clone()
    linv = torch.zeros(nbox, 64 * 64, dtype=torch.float64, device="cuda")
    npd = torch.full((nbox,), 2 ** 31 - 1, dtype=torch.int32, device="cuda")
    prog = Program(torch.device("cuda"))
    prog.chol_panel([(hd[i].data_ptr(), linv[i].data_ptr(), n, 64, n, p, b, i) for i in range(nbox)],
                    npd.data_ptr())
    prog = prog.finalize()
    for _ in range(3):
        hd.copy_(h0)
        prog.run()
        torch.cuda.synchronize()
        out = hd.cpu().numpy()
        assert (npd.cpu().numpy() == 2 ** 31 - 1).all()
        for i in range(0, nbox, 17):
            lf = lfs[i]
            tol = RTOL * np.abs(lf).max() * 10
            np.testing.assert_allclose(np.tril(out[i, p:p + b, p:p + b]), lf[p:p + b, p:p + b], rtol=0, atol=tol)
            np.testing.assert_allclose(out[i, p + b:, p:p + b], lf[p + b:, p:p + b], rtol=0, atol=tol)


@pytest.mark.parametrize("cfg", [2, 7, 9])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0)])
def test_gemm_grouped_configs(env, cfg, ta, tb):
    """Grouped C = alpha op(A) op(B) + beta C over ragged problems (h2g_gemm_grouped), every tile
    configuration the planner picks; LOWER problems only write the lower triangle."""
    torch, nat, Program = env
    rng = np.random.default_rng(10 * cfg + 2 * ta + tb)
    shapes = [(85, 85, 64, True), (43, 85, 64, False), (200, 37, 130, False), (96, 96, 21, True), (5, 70, 3, False)]
    hold, probs, refs = [], [], []
    for (m, n, k, lower) in shapes:
        a = rng.standard_normal((k, m) if ta else (m, k))
        b = rng.standard_normal((n, k) if tb else (k, n))
        c = rng.standard_normal((m, n))
        alpha, beta = -1.0, 1.0
        ref = alpha * (a.T if ta else a) @ (b.T if tb else b) + beta * c
        t = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (a, b, c)]
        hold.append(t)
        probs.append((t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(), m, n, k, a.shape[1], b.shape[1], n,
                      nat.GEMM_LOWER if lower else 0, alpha, beta))
        refs.append(ref)
    prog = Program(torch.device("cuda"))
    prog.gemm(ta, tb, probs, tile_cfg=cfg)
    prog.finalize().run()
    torch.cuda.synchronize()
    for t, ref, (m, n, k, lower) in zip(hold, refs, shapes):
        got = t[2].cpu().numpy()
        if lower:   # tiles above the diagonal are left alone; inside diagonal tiles only i >= j is specified
            keep = np.tril(np.ones((m, n), dtype=bool))
            got, ref = np.where(keep, got, 0.0), np.where(keep, ref, 0.0)
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))


@pytest.mark.parametrize("rows,cols", [(1, 1), (45, 70), (64, 64), (130, 97), (200, 200)])
def test_block_copy_modes(env, rows, cols):
    """h2g_block_copy: copy / transpose / symmetric-from-lower / identity into a strided
    destination, bit-exact (the merge of child Schur blocks, ulv_factor.py:115-132)."""
    torch, nat, Program = env
    rng = np.random.default_rng(rows * 1000 + cols)
    src = rng.standard_normal((max(rows, cols) + 3, max(rows, cols) + 5))
    lds = src.shape[1]
    s = torch.from_numpy(src).cuda()
    outs, refs = [], []
    prog = Program(torch.device("cuda"))
    descs = []
    for mode in (0, 1, 2, 3):
        r, c = (rows, rows) if mode == 2 else (rows, cols)
        ldd = c + 7
        d = torch.full((r, ldd), 7.0, dtype=torch.float64, device="cuda")
        ref = np.full((r, ldd), 7.0)
        if mode == 0:
            ref[:, :c] = src[:r, :c]
        elif mode == 1:
            ref[:, :c] = src[:c, :r].T
        elif mode == 2:
            low = np.tril(src[:r, :r])
            ref[:, :c] = low + np.tril(low, -1).T
        else:
            ref[:, :c] = np.eye(r, c)
        descs.append((s.data_ptr(), d.data_ptr(), r, c, lds, ldd, mode))
        outs.append(d)
        refs.append(ref)
    prog.copy(descs)
    prog.finalize().run()
    torch.cuda.synchronize()
    for d, ref in zip(outs, refs):
        np.testing.assert_array_equal(d.cpu().numpy(), ref)


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("alpha,beta", [(1.0, 0.0), (-1.0, 1.0), (0.5, -2.0)])
def test_gemm_split_k(env, ta, tb, alpha, beta):
    """Deterministic split-K (h2g_gemm_grouped_split, picked by Program.gemm(split=True) for
    launches under one wave with long K): every split factor against numpy, the LOWER
    flag, alpha / beta, and bit-identical results on a replay (fixed reduction order)."""
    import paper_2502_02395_b200.program as pm

    torch, nat, Program = env
    rng = np.random.default_rng(7 + 4 * ta + 2 * tb)
    shapes = [(150, 150, 700, True), (70, 130, 517, False), (64, 64, 1000, False), (33, 9, 300, False)]
    for nsplit in (2, 4, 8):
        hold, probs, refs = [], [], []
        for (m, n, k, lower) in shapes:
            a = rng.standard_normal((k, m) if ta else (m, k))
            b = rng.standard_normal((n, k) if tb else (k, n))
            c = rng.standard_normal((m, n))
            ref = alpha * (a.T if ta else a) @ (b.T if tb else b) + beta * c
            t = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (a, b, c)]
            hold.append((t, c.copy()))
            probs.append((t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(), m, n, k, a.shape[1], b.shape[1], n,
                          nat.GEMM_LOWER if lower else 0, alpha, beta))
            refs.append(ref)
        old = pm.choose_split
        pm.choose_split = lambda tiles, ks, sms=148, per_sm=4: nsplit
        try:
            prog = Program(torch.device("cuda"))
            prog.gemm(ta, tb, probs, tile_cfg=2, split=True)
        finally:
            pm.choose_split = old
        assert prog._steps[-1]["arg"] >> 8 == nsplit and prog._steps[-1]["npd"]
        prog.finalize()
        outs = []
        for rep in range(2):
            for (t, c0) in hold:
                t[2].copy_(torch.from_numpy(c0))
            prog.run()
            torch.cuda.synchronize()
            outs.append([t[2].cpu().numpy() for (t, _) in hold])
        for got, again, ref, (m, n, k, lower) in zip(outs[0], outs[1], refs, shapes):
            assert np.array_equal(got, again)
            if lower:
                keep = np.tril(np.ones((m, n), dtype=bool))
                got, ref = np.where(keep, got, 0.0), np.where(keep, ref, 0.0)
            np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))
