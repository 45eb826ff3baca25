"""① Complementary basis on the GPU: batched blocked Householder QR.

For every box of a level, Z_i (n_i x k_i) is factored Z = Q R with the
LAPACK conventions of `np.linalg.qr(z, mode="complete")` (dgeqrf + dorgqr)
that the reference calls in id_basis (dense_core.py:136-144); then the sign
fix s = sign(diag R) (0 -> +1), q_skel = Q[:, :k] s, frame = s R[:k, :],
q_red = Q[:, k:] (dense_core.py:140-144) and q_full = [q_red | q_skel].

Program per level (all boxes in every launch), panels of 32 columns:
  factor:  QR_PANEL(p); W = V_p^T C; W2 = T_p^T W; C -= V_p W2   (C = Z[p:, p+b:])
  form Q:  Q = I; for p = last..0:  W = V_p^T Q_s; W2 = T_p W; Q_s -= V_p W2
           (Q_s = Q[p:, p:], backward accumulation as in dorgqr)
  finish:  BASIS (sign fix, [q_red | q_skel], frame)
"""

import numpy as np
import torch

from . import _native as nat
from .program import Program

F64 = torch.float64
QB = nat.QR_PANEL_WIDTH


class LevelQR:
    """Device buffers + program of the complete QR of one level's Z_i."""

    def __init__(self, device, n, k, z_ptrs=None):
        self.device = device
        self.n = np.asarray(n, dtype=np.int64)
        self.k = np.asarray(k, dtype=np.int64)
        nb = len(self.n)
        self.zoff = np.concatenate([[0], np.cumsum(self.n * self.k)[:-1]]).astype(np.int64)
        self.qoff = np.concatenate([[0], np.cumsum(self.n * self.n)[:-1]]).astype(np.int64)
        self.foff = np.concatenate([[0], np.cumsum(self.k * self.k)[:-1]]).astype(np.int64)
        zs = max(int((self.n * self.k).sum()), 1)
        self.Z = torch.zeros(zs, dtype=F64, device=device)
        self.V = torch.zeros(zs, dtype=F64, device=device)
        self.Q = torch.empty(max(int((self.n * self.n).sum()), 1), dtype=F64, device=device)
        self.qfull = torch.empty_like(self.Q)
        self.frame = torch.empty(max(int((self.k * self.k).sum()), 1), dtype=F64, device=device)
        npan = -(-self.k // QB)
        self.toff = np.concatenate([[0], np.cumsum(npan * QB * QB)[:-1]]).astype(np.int64)
        self.T = torch.zeros(max(int(npan.sum()) * QB * QB, 1), dtype=F64, device=device)
        self.tau = torch.zeros(max(int(self.k.sum()), 1), dtype=F64, device=device)
        self.tauoff = np.concatenate([[0], np.cumsum(self.k)[:-1]]).astype(np.int64)
        wsz = max(int((QB * np.maximum(self.n, 1)).sum()), 1)
        self.woff = np.concatenate([[0], np.cumsum(QB * self.n)[:-1]]).astype(np.int64)
        self.W = torch.empty(wsz, dtype=F64, device=device)
        self.W2 = torch.empty(wsz, dtype=F64, device=device)
        self.nb = nb

    def ptr(self, t, off):
        return t.data_ptr() + 8 * int(off)

    def build(self, prog):
        n, k, nb = self.n, self.k, self.nb
        # identity for boxes with k == 0 (q_red = I) and as the start of dorgqr
        prog.copy([(0, self.ptr(self.Q, self.qoff[i]), int(n[i]), int(n[i]), 0, int(n[i]), 3) for i in range(nb)])
        kmax = int(k.max()) if nb else 0
        panels = list(range(0, kmax, QB))
        for p in panels:
            descs, g1, g2, g3 = [], [], [], []
            for i in range(nb):
                ni, ki = int(n[i]), int(k[i])
                if ki <= p:
                    continue
                b = min(QB, ki - p)
                zi, vi = self.ptr(self.Z, self.zoff[i]), self.ptr(self.V, self.zoff[i])
                ti = self.ptr(self.T, self.toff[i] + (p // QB) * QB * QB)
                descs.append((zi, vi, self.ptr(self.tau, self.tauoff[i]), ti, ni, ki, p, b))
                m = ki - p - b
                if m <= 0:
                    continue
                wi, w2 = self.ptr(self.W, self.woff[i]), self.ptr(self.W2, self.woff[i])
                vp = vi + 8 * (p * ki + p)
                cp = zi + 8 * (p * ki + p + b)
                g1.append((vp, cp, wi, b, m, ni - p, ki, ki, m, 0, 1.0, 0.0))          # W = V^T C
                g2.append((ti, wi, w2, b, m, b, QB, m, m, 0, 1.0, 0.0))                # W2 = T^T W
                g3.append((vp, w2, cp, ni - p, m, b, ki, m, ki, 0, -1.0, 1.0))          # C -= V W2
            prog.qr_panel(descs)
            prog.gemm(1, 0, g1)
            prog.gemm(1, 0, g2)
            prog.gemm(0, 0, g3)
        for p in reversed(panels):
            g1, g2, g3 = [], [], []
            for i in range(nb):
                ni, ki = int(n[i]), int(k[i])
                if ki <= p:
                    continue
                b = min(QB, ki - p)
                m = ni - p
                vi = self.ptr(self.V, self.zoff[i])
                vp = vi + 8 * (p * ki + p)
                ti = self.ptr(self.T, self.toff[i] + (p // QB) * QB * QB)
                wi, w2 = self.ptr(self.W, self.woff[i]), self.ptr(self.W2, self.woff[i])
                qs = self.ptr(self.Q, self.qoff[i]) + 8 * (p * ni + p)
                g1.append((vp, qs, wi, b, m, m, ki, ni, m, 0, 1.0, 0.0))               # W = V^T Q_s
                g2.append((ti, wi, w2, b, m, b, QB, m, m, 0, 1.0, 0.0))                # W2 = T W
                g3.append((vp, w2, qs, m, m, b, ki, m, ni, 0, -1.0, 1.0))              # Q_s -= V W2
            prog.gemm(1, 0, g1)
            prog.gemm(0, 0, g2)
            prog.gemm(0, 0, g3)
        prog.basis([(self.ptr(self.Q, self.qoff[i]), self.ptr(self.Z, self.zoff[i]),
                     self.ptr(self.qfull, self.qoff[i]), self.ptr(self.frame, self.foff[i]),
                     int(n[i]), int(k[i]), int(k[i])) for i in range(nb) if k[i] > 0])
        # k == 0: q_full = I
        prog.copy([(0, self.ptr(self.qfull, self.qoff[i]), int(n[i]), int(n[i]), 0, int(n[i]), 3)
                   for i in range(nb) if k[i] == 0])


def wy_profitable(n, k, ratio=None):
    """Whether the compact-WY diag transform beats the dense one on a level: its
    GEMMs (W = A V~: 2n^2k, the relabelled rank-2k update: ~2n^2k, X and U: 4nk^2)
    against Q^T (A Q) with the lower-only second product (3n^3), summed over the
    boxes.  Every box needs k > 0 (k = 0 means q_full = I)."""
    n = np.asarray(n, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    if not n.size or (k <= 0).any():
        return False
    ratio = WY_RATIO if ratio is None else ratio
    frac = float((4 * n * n * k + 4 * n * k * k).sum()) / float((3 * n ** 3).sum())
    # past half the dense flops the thin WY GEMMs only pay on boxes large enough to keep
    # their tiles busy (M1 levels 9 / 6 / 3, mean n >= 221, gain; C3 level 9, mean n 90, loses)
    return frac < min(ratio, 0.5) or (frac < ratio and float(n.mean()) >= WY_MIN_N)


WY_RATIO = float(__import__("os").environ.get("H2G_WY_RATIO", "0.8"))
WY_MIN_N = float(__import__("os").environ.get("H2G_WY_MIN_N", "128"))


def build_wy(lq, prog):
    """Compact-WY form of every box's Q (Q = I - V T V^T, k reflectors), stored with
    the basis for the diag transform (ulv_factor.FactorPlan): Vt = V T, the operand
    buffers P = [. | V] and Qm = [V | .] (n x 2k; the free halves receive W = A Vt and
    U = W - V (Vt^T W) per factorization), a k x k scratch X and id_basis's column
    signs s = sign(diag R) (0 -> +1; dense_core.py:140-144).  T is never formed:
    with the panel factors T_p of h2g_qr_panel, panel by panel (c = 32 p)
        Vt[:, c:c+b] = V_p T_p - Vt[:, :c] (V[:, :c]^T (V_p T_p))
    (the forward accumulation of the block reflectors, Q_0 ... Q_p = I - [V_a V_p]
    [[T_a, -T_a V_a^T V_p T_p], [0, T_p]] [V_a V_p]^T)."""
    n, k, nb = lq.n, lq.k, lq.nb
    dev = lq.device
    lq.wy_vt = torch.zeros_like(lq.V)
    lq.wy_poff = 2 * lq.zoff
    lq.wy_p = torch.zeros(max(int(2 * (n * k).sum()), 1), dtype=F64, device=dev)
    lq.wy_q = torch.zeros_like(lq.wy_p)
    lq.wy_x = torch.zeros(max(int((k * k).sum()), 1), dtype=F64, device=dev)
    kmax = int(k.max()) if nb else 0
    for c in range(0, kmax, QB):
        g0, g1, g2 = [], [], []
        for i in range(nb):
            ni, ki = int(n[i]), int(k[i])
            if ki <= c:
                continue
            b = min(QB, ki - c)
            v, vt = lq.ptr(lq.V, lq.zoff[i]), lq.ptr(lq.wy_vt, lq.zoff[i])
            tp = lq.ptr(lq.T, lq.toff[i] + (c // QB) * QB * QB)
            g0.append((v + 8 * c, tp, vt + 8 * c, ni, b, b, ki, QB, ki, 0, 1.0, 0.0))          # V_p T_p
            if c:
                w = lq.ptr(lq.W, lq.woff[i])
                g1.append((v, vt + 8 * c, w, c, b, ni, ki, ki, b, 0, 1.0, 0.0))             # X = V_a^T (V_p T_p)
                g2.append((vt, w, vt + 8 * c, ni, b, c, ki, b, ki, 0, -1.0, 1.0))           # -= Vt_a X
        prog.gemm(0, 0, g0)
        prog.gemm(1, 0, g1)
        prog.gemm(0, 0, g2)
    wy_operands(lq, prog)


def wy_operands(lq, prog):
    """The constant halves of the WY operand buffers: Y into P[:, k:] and Qm[:, :k]."""
    cp = []
    for i in range(lq.nb):
        ni, ki = int(lq.n[i]), int(lq.k[i])
        if ki == 0:
            continue
        v = lq.ptr(lq.V, lq.zoff[i])
        cp.append((v, lq.ptr(lq.wy_p, lq.wy_poff[i]) + 8 * ki, ni, ki, ki, 2 * ki, 0))
        cp.append((v, lq.ptr(lq.wy_q, lq.wy_poff[i]), ni, ki, ki, 2 * ki, 0))
    prog.copy(cp)


_IDENT = {}


def _identity(device, n):
    t = _IDENT.get(device)
    if t is None or t.shape[0] < n:
        t = torch.eye(max(n, 1), dtype=F64, device=device)
        _IDENT[device] = t
    return t


def rebuild_qfull(lq, prog, q_ptr):
    """q_full_i = [Q[:, k:] | Q[:, :k] s] from the compact-WY form, Q = I - Yt Y^T: one NT
    GEMM per box (beta term from a shared identity) whose column-relabel store writes the
    [q_red | q_skel s] order with id_basis's signs (dense_core.py:140-148).  Used at
    construct (so the device q_full IS this product) and after a compact upload of a
    pinned-host H2 (DeviceH2.from_host), which therefore rebuilds the same bits."""
    nmax = int(lq.n.max()) if lq.nb else 1
    ident = _identity(lq.device, nmax)
    lq._ident = ident                  # keeps the buffer the program points into alive
    ldi = int(ident.shape[0])          # the shared identity may be larger than this level's n
    prob = []
    for i in range(lq.nb):
        ni, ki = int(lq.n[i]), int(lq.k[i])
        yt, y = lq.ptr(lq.wy_vt, lq.zoff[i]), lq.ptr(lq.V, lq.zoff[i])
        prob.append((yt, y, q_ptr(i), ni, ni, ki, ki, ki, ni, 0, -1.0, 1.0,
                     (ident.data_ptr(), lq.ptr(lq.wy_sgn, lq.tauoff[i]), ldi, -(ki + 2))))
    prog.gemm(0, 1, prob, tile_cfg=2)


class WYLevel:
    """Device buffers of the compact-WY form of one level's bases uploaded from a
    pinned-host H2 (the fields FactorPlan._wy_transform and rebuild_qfull read; the
    construct keeps them on its LevelQR instead)."""

    def __init__(self, device, n, k):
        self.device = device
        self.n = np.asarray(n, dtype=np.int64)
        self.k = np.asarray(k, dtype=np.int64)
        self.nb = len(self.n)
        self.zoff = np.concatenate([[0], np.cumsum(self.n * self.k)[:-1]]).astype(np.int64)
        self.foff = np.concatenate([[0], np.cumsum(self.k * self.k)[:-1]]).astype(np.int64)
        self.tauoff = np.concatenate([[0], np.cumsum(self.k)[:-1]]).astype(np.int64)
        self.wy_poff = 2 * self.zoff
        nk = max(int((self.n * self.k).sum()), 1)
        self.V = torch.zeros(nk, dtype=F64, device=device)
        self.wy_vt = torch.zeros(nk, dtype=F64, device=device)
        self.wy_sgn = torch.ones(max(int(self.k.sum()), 1), dtype=F64, device=device)
        self.wy_p = torch.zeros(2 * nk, dtype=F64, device=device)
        self.wy_q = torch.zeros(2 * nk, dtype=F64, device=device)
        self.wy_x = torch.zeros(max(int((self.k * self.k).sum()), 1), dtype=F64, device=device)

    def ptr(self, t, off):
        return t.data_ptr() + 8 * int(off)

    def sizes(self):
        """(Y, Yt, signs) element counts: the layout of a pinned arena's "w" region."""
        nk = int((self.n * self.k).sum())
        return nk, nk, int(self.k.sum())


def wy_signs(lq):
    """id_basis's signs s_j = sign(R_jj) (0 -> +1) of every box, from the R left in Z
    by the QR (one +-1 double per skeleton column, laid out like tau)."""
    idx = np.concatenate([lq.zoff[i] + np.arange(int(lq.k[i])) * (int(lq.k[i]) + 1) for i in range(lq.nb)]
                         + [np.zeros(0, dtype=np.int64)]).astype(np.int64)
    d = lq.Z[torch.from_numpy(idx).to(lq.device)] if idx.size else lq.Z[:0]
    lq.wy_sgn = torch.where(d < 0, -1.0, 1.0).to(F64)
    if not idx.size:
        lq.wy_sgn = torch.ones(1, dtype=F64, device=lq.device)


def complete_qr_host(zs, device=None):
    """Complete QR of host matrices Z_i on the GPU; returns [(q_full, frame)]."""
    nat.lib()
    device = torch.device(device or "cuda")
    n = [z.shape[0] for z in zs]
    k = [z.shape[1] for z in zs]
    lq = LevelQR(device, n, k)
    host = np.concatenate([np.ascontiguousarray(z, dtype=np.float64).ravel() for z in zs] + [np.zeros(0)])
    if host.size:
        lq.Z[:host.size].copy_(torch.from_numpy(host))
    prog = Program(device)
    lq.build(prog)
    prog.finalize().run()
    out = []
    qf, fr = lq.qfull.cpu().numpy(), lq.frame.cpu().numpy()
    for i in range(len(zs)):
        ni, ki = n[i], k[i]
        out.append((qf[lq.qoff[i]:lq.qoff[i] + ni * ni].reshape(ni, ni).copy(),
                    fr[lq.foff[i]:lq.foff[i] + ki * ki].reshape(ki, ki).copy()))
    return out
