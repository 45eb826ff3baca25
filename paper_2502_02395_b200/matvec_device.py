"""H² matrix-vector product on the GPU — the residual operator of the
reference (`h2ulv.h2_build.h2_matvec`, h2_build.py:232-282; cli.py:199-205
computes ||A x - b|| / ||b|| with it).  SURVEY.md §8(f) "next" #2.

Same four passes as the reference, each ONE grouped GEMV launch per level
over the operands that already live in HBM (DeviceH2):

  upward    xhat_i = q_skel_i^T seg_i          seg = x (leaf) or [xhat_2i; xhat_2i+1]
  coupling  yhat_i = sum_{j far} S_ij xhat_j   S_ij (i > j) or S_ji^T (i < j)
  downward  full_i = q_skel_i yhat_i  ->  yhat of the children / y (leaf)
  near      y_i   += sum_{j near} A_ij x_j     A_ij (i >= j) or A_ji^T

Per level the skeleton vectors are stored back to back in box order, so a
parent's segment [xhat_2i; xhat_2i+1] is contiguous and the reference's
vstack / split cost nothing.  The whole product is one Program (CUDA graph).
"""

import numpy as np
import torch

from . import _native as nat
from .program import Program

F64 = torch.float64


class MatvecPlan:
    """Device buffers + the static GEMV program of y = A x for RHS width w."""

    def __init__(self, dh2, tree, lists, w=1):
        self.dh2 = dh2
        self.w = w
        dev = dh2.device
        self.device = dev
        depth = dh2.depth
        self.count = dh2.count
        self.x = torch.zeros(max(self.count, 1) * w, dtype=F64, device=dev)
        self.y = torch.zeros(max(self.count, 1) * w, dtype=F64, device=dev)
        prog = Program(dev)
        if depth == 0:
            d = self.count
            prog.gemv([(self.y.data_ptr(), 0, 0, d, 0, nat.GEMV_PLUS,
                        [(dh2.root_a.data_ptr(), self.x.data_ptr(), d, 0, d)])], w)
            self.program = prog.finalize()
            self.program.capture()
            return
        p = lambda t, rows: t.data_ptr() + 8 * int(rows) * w
        begins = np.array([b.begin for b in tree.leaves], dtype=np.int64)
        self.xhat, self.yhat, koff = {}, {}, {}
        for l, lay in dh2.levels.items():
            koff[l] = np.concatenate([[0], np.cumsum(lay.k)[:-1]]).astype(np.int64)
            self.xhat[l] = torch.zeros(max(int(lay.k.sum()), 1) * w, dtype=F64, device=dev)
            self.yhat[l] = torch.zeros(max(int(lay.k.sum()), 1) * w, dtype=F64, device=dev)
        # zero the accumulated outputs every run
        self._zero = torch.zeros(max(self.count * w, max(int(t.numel()) for t in self.yhat.values())),
                                 dtype=F64, device=dev)
        prog.memcpy(self.y.data_ptr(), self._zero.data_ptr(), 8 * self.count * w)
        for l in self.yhat:
            prog.memcpy(self.yhat[l].data_ptr(), self._zero.data_ptr(), 8 * int(self.yhat[l].numel()))
        # upward
        for l in range(depth, 0, -1):
            lay = dh2.levels[l]
            q = dh2.q[l]
            outs = []
            for i in range(lay.nb):
                ni, ki, ri = int(lay.n[i]), int(lay.k[i]), int(lay.r[i])
                if ki == 0:
                    continue
                if l == depth:
                    src = p(self.x, begins[i])
                else:
                    src = p(self.xhat[l + 1], dh2_child_off(dh2, l, i, koff))
                outs.append((p(self.xhat[l], koff[l][i]), 0, 0, ki, 0, nat.GEMV_PLUS,
                             [(q.data_ptr() + 8 * int(lay.qoff[i] + ri), src, ni, 1, ni)]))
            prog.gemv(outs, w)
        # coupling
        for l in range(depth, 0, -1):
            lay = dh2.levels[l]
            s = dh2.s[l]
            terms = {}
            for (i, j) in sorted(lists.far[l]):
                ki, kj = int(lay.k[i]), int(lay.k[j])
                if ki == 0 or kj == 0:
                    continue
                if i > j:
                    t = (s.data_ptr() + 8 * int(lay.soff[(i, j)]), p(self.xhat[l], koff[l][j]), kj, 0, kj)
                else:
                    t = (s.data_ptr() + 8 * int(lay.soff[(j, i)]), p(self.xhat[l], koff[l][j]), ki, 1, kj)
                terms.setdefault(i, []).append(t)
            outs = [(p(self.yhat[l], koff[l][i]), 0, 0, int(lay.k[i]), 0, nat.GEMV_PLUS, tl)
                    for i, tl in sorted(terms.items())]
            prog.gemv(outs, w)
        # downward
        for l in range(1, depth + 1):
            lay = dh2.levels[l]
            q = dh2.q[l]
            outs = []
            for i in range(lay.nb):
                ni, ki, ri = int(lay.n[i]), int(lay.k[i]), int(lay.r[i])
                if ki == 0:
                    continue
                dst = p(self.y, begins[i]) if l == depth else p(self.yhat[l + 1], dh2_child_off(dh2, l, i, koff))
                outs.append((dst, 0, dst, ni, 0, nat.GEMV_PLUS,
                             [(q.data_ptr() + 8 * int(lay.qoff[i] + ri), p(self.yhat[l], koff[l][i]), ni, 0, ki)]))
            prog.gemv(outs, w)
        # leaf near blocks
        leaf = dh2.levels[depth]
        terms = {}
        for (i, j) in sorted(lists.near[depth]):
            ni, nj = int(leaf.n[i]), int(leaf.n[j])
            if i >= j:
                t = (dh2.leaf_a.data_ptr() + 8 * int(dh2.aoff[(i, j)]), p(self.x, begins[j]), nj, 0, nj)
            else:
                t = (dh2.leaf_a.data_ptr() + 8 * int(dh2.aoff[(j, i)]), p(self.x, begins[j]), ni, 1, nj)
            terms.setdefault(i, []).append(t)
        outs = [(p(self.y, begins[i]), 0, p(self.y, begins[i]), int(leaf.n[i]), 0, nat.GEMV_PLUS, tl)
                for i, tl in sorted(terms.items())]
        prog.gemv(outs, w)
        self.program = prog.finalize()
        self.program.capture()

    def run(self, x_tree):
        """x_tree: torch (N, w) float64 on the device (tree order) -> y (N, w) tree order."""
        self.x.view(-1, self.w)[:self.count].copy_(x_tree)
        self.program.launch()
        return self.y.view(-1, self.w)[:self.count]


def dh2_child_off(dh2, l, i, koff):
    """Offset (rows) of [xhat_2i; xhat_2i+1] in the level-(l+1) skeleton vector."""
    return int(koff[l + 1][2 * i])


def device_matvec(h2, x):
    """y = A x (tree order).  GPU-built H²: the operands of h2._device, plans
    cached per width.  Host H²: uploaded (DeviceH2.from_host) and planned per
    call — a pure function of the numpy blocks."""
    nat.lib()
    dh2 = getattr(h2, "_device", None)
    xm = np.asarray(x, dtype=np.float64)
    vec = xm.ndim == 1
    xm = xm.reshape(h2.count, -1)
    w = xm.shape[1]
    if dh2 is None:
        from .h2_device import DeviceH2

        dh2 = DeviceH2.from_host(h2)
        plan = MatvecPlan(dh2, h2.tree, h2.lists, w)
    else:
        cache = h2.__dict__.setdefault("_matvec_plans", {})
        if w not in cache:
            cache[w] = MatvecPlan(dh2, h2.tree, h2.lists, w)
        plan = cache[w]
    y = plan.run(torch.from_numpy(np.ascontiguousarray(xm)).to(dh2.device)).cpu().numpy()
    return y[:, 0] if vec else y
