"""Device-resident H² operands of the factorization path.

Layout in HBM (all FP64, row-major, one allocation per level and kind):
  q[l]      the bases q_full_i = [q_red_i | q_skel_i] (n_i x n_i) of every box,
            packed back to back at qoff[l][i] (element offsets);
  leaf_a    the leaf-level near blocks A_ij (i >= j, n_i x n_j) at aoff[(i, j)]
            — upper-level near blocks are never read by the factorization
            (they are rebuilt from child Schur complements by the merge);
  s[l]      far couplings S_ij (i > j, k_i x k_j) at soff[l][(i, j)];
  root_a    the single block when the tree has depth 0.

`DeviceH2.from_host(h2)` uploads a numpy H2Matrix (the reference's, or a
host-materialized one) through one pinned staging buffer per kind;
`h2_build.construct` produces a DeviceH2 directly on the GPU.
"""

import numpy as np
import torch

F64 = torch.float64


def _sorted_pairs(pairs, cond):
    return sorted((i, j) for (i, j) in pairs if cond(i, j))


class LevelLayout:
    """Box dimensions and packing offsets of one level (host metadata)."""

    def __init__(self, l, n, k, near, far):
        self.l = l
        self.nb = len(n)
        self.n = np.asarray(n, dtype=np.int64)
        self.k = np.asarray(k, dtype=np.int64)
        self.r = self.n - self.k
        self.qoff = np.concatenate([[0], np.cumsum(self.n * self.n)[:-1]]).astype(np.int64)
        self.qsize = int((self.n * self.n).sum())
        self.near_pairs = _sorted_pairs(near, lambda i, j: i >= j)     # incl. diagonal
        self.off_pairs = _sorted_pairs(near, lambda i, j: i > j)       # ulv_factor.py:244
        self.far_pairs = _sorted_pairs(far, lambda i, j: i > j)
        self.near_set = set(near)
        self.far_set = set(far)
        soff, acc = {}, 0
        for (i, j) in self.far_pairs:
            soff[(i, j)] = acc
            acc += int(self.k[i] * self.k[j])
        self.soff = soff
        self.ssize = acc


class DeviceH2:
    """Device copy of everything factorize/solve read from an H2Matrix."""

    def __init__(self, device, depth, count, levels, q, s, leaf_a, aoff, root_a=None):
        self.device = device
        self.depth = depth
        self.count = count
        self.levels = levels    # l -> LevelLayout
        self.q = q              # l -> tensor
        self.s = s              # l -> tensor
        self.leaf_a = leaf_a    # tensor (depth >= 1)
        self.aoff = aoff        # (i, j) -> offset in leaf_a
        self.root_a = root_a    # tensor d x d (depth == 0)

    # -------------------------------------------------------------------------------
    @staticmethod
    def layouts_from_host(h2):
        depth = h2.tree.depth
        levels = {}
        for l in range(depth, 0, -1):
            nb = 2 ** l
            n = [h2.bases[(l, i)].n for i in range(nb)]
            k = [h2.bases[(l, i)].rank for i in range(nb)]
            levels[l] = LevelLayout(l, n, k, h2.lists.near[l], h2.lists.far[l])
        return levels

    @classmethod
    def from_host(cls, h2, device=None):
        """Upload the numpy arrays of `h2` (bases, leaf near blocks, couplings)."""
        device = torch.device(device or "cuda")
        depth = h2.tree.depth
        if depth == 0:
            a = np.ascontiguousarray(h2.near_blocks[(0, 0, 0)], dtype=np.float64)
            root_a = torch.from_numpy(a).to(device)
            return cls(device, 0, h2.count, {}, {}, {}, None, {}, root_a=root_a)
        levels = cls.layouts_from_host(h2)
        q, s = {}, {}
        for l, lay in levels.items():
            buf = torch.empty(lay.qsize, dtype=F64, pin_memory=True)
            hv = buf.numpy()
            for i in range(lay.nb):
                b = h2.bases[(l, i)]
                n, k = int(lay.n[i]), int(lay.k[i])
                blk = hv[lay.qoff[i]:lay.qoff[i] + n * n].reshape(n, n)
                blk[:, :n - k] = b.q_red
                blk[:, n - k:] = b.q_skel
            q[l] = buf.to(device, non_blocking=True)
            sbuf = torch.empty(max(lay.ssize, 1), dtype=F64, pin_memory=True)
            sv = sbuf.numpy()
            for (i, j), off in lay.soff.items():
                c = h2.couplings[(l, i, j)]
                sv[off:off + c.size] = c.ravel()
            s[l] = sbuf.to(device, non_blocking=True)
        leaf = levels[depth]
        aoff, acc = {}, 0
        for (i, j) in leaf.near_pairs:
            aoff[(i, j)] = acc
            acc += int(leaf.n[i] * leaf.n[j])
        abuf = torch.empty(max(acc, 1), dtype=F64, pin_memory=True)
        av = abuf.numpy()
        for (i, j), off in aoff.items():
            blk = h2.near_blocks[(depth, i, j)]
            av[off:off + blk.size] = blk.ravel()
        leaf_a = abuf.to(device, non_blocking=True)
        torch.cuda.current_stream(device).synchronize()  # pinned staging buffers die here
        return cls(device, depth, h2.count, levels, q, s, leaf_a, aoff)

    def ptr_q(self, l, i, col=0):
        lay = self.levels[l]
        return self.q[l].data_ptr() + 8 * int(lay.qoff[i] + col)
