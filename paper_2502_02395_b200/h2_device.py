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
host-materialized one) through one reusable pinned staging buffer (bases as
contiguous q_red / q_skel, interleaved into q_full on the device);
`h2_build.construct` produces a DeviceH2 directly on the GPU.
"""

import hashlib
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

F64 = torch.float64
_STAGING = {"buf": None, "done": None}
_POOL = {"pool": None}


def _pool():
    if _POOL["pool"] is None:
        # measured on the B200 box (16 host cores; tools/upload_overlap.py, tools/ab_e2e.sh):
        # 8 gather threads leave the DMA engine enough host memory bandwidth, 16 do not
        n = int(os.environ.get("H2G_UPLOAD_THREADS", "8"))
        _POOL["pool"] = ThreadPoolExecutor(max_workers=max(1, min(n, os.cpu_count() or 1)))
    return _POOL["pool"]


def _staging(n_doubles):
    """Reusable pinned host buffer of at least n doubles: (tensor, numpy view)."""
    buf = _STAGING["buf"]
    if buf is None or buf.numel() < n_doubles:
        buf = torch.empty(int(n_doubles * 1.25) + 1024, dtype=F64, pin_memory=True)
        _STAGING["buf"] = buf
    return buf, buf.numpy()


# doubles per upload chunk (default 16 MB: C2 end to end 31 ms vs 39 ms with 4 MB chunks and 16 threads)
_CHUNK = int(os.environ.get("H2G_UPLOAD_CHUNK", str(1 << 21)))


def _run_tasks(tasks):
    for t in tasks:
        t[0](*t[1:])


def _fill_q(host, off, basis, n, k):
    """q_red then q_skel, each contiguous (fast memcpy); the GPU interleaves
    them into the row-major q_full = [q_red | q_skel] (one block-copy launch)."""
    r = n - k
    host[off:off + n * r].reshape(n, r)[...] = basis.q_red
    host[off + n * r:off + n * n].reshape(n, k)[...] = basis.q_skel


def _fill_flat(host, off, arr):
    a = np.asarray(arr)
    host[off:off + a.size].reshape(a.shape)[...] = a


def _signature(depth, count, levels):
    h = hashlib.sha1(f"{depth}:{count}".encode())
    for l in sorted(levels):
        lay = levels[l]
        h.update(lay.n.tobytes())
        h.update(lay.k.tobytes())
        h.update(np.asarray(lay.near_pairs, dtype=np.int64).tobytes())
        h.update(np.asarray(lay.far_pairs, dtype=np.int64).tobytes())
    return h.hexdigest()


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


def _q_interleave(levels, q, device):
    """Device staging for the bases (q_red, q_skel contiguous per box) and, per
    level, the block-copy program that forms q_full = [q_red | q_skel] row-major
    in q[l]."""
    from .program import Program

    qsplit = {l: torch.empty(max(lay.qsize, 1), dtype=F64, device=device) for l, lay in levels.items()}
    progs = {}
    for l, lay in levels.items():
        prog = Program(device)
        descs = []
        sp, qp = qsplit[l].data_ptr(), q[l].data_ptr()
        for i in range(lay.nb):
            n, k = int(lay.n[i]), int(lay.k[i])
            r, o = n - k, int(lay.qoff[i])
            descs.append((sp + 8 * o, qp + 8 * o, n, r, r, n, 0))
            descs.append((sp + 8 * (o + n * r), qp + 8 * (o + r), n, k, k, n, 0))
        prog.copy(descs)
        progs[l] = prog.finalize()
    return qsplit, progs


_FIX_STREAM = {}


def _fix_stream(device):
    st = _FIX_STREAM.get(device)
    if st is None:
        st = torch.cuda.Stream(device=device, priority=-1)
        _FIX_STREAM[device] = st
    return st


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
        self.wy = {}            # l -> compact-WY form of the level's bases (LevelQR / basis_qr.WYLevel)

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

    def signature(self):
        """Structure key: equal signatures -> identical layouts and programs."""
        sig = self.__dict__.get("_sig")
        if sig is None:
            sig = _signature(self.depth, self.count, self.levels)
            if self.wy:   # compact-WY levels change the staging layout and the program
                sig += ":wy" + ",".join(str(l) for l in sorted(self.wy))
            self._sig = sig
        return sig

    @classmethod
    def allocate_for_host(cls, h2, device=None):
        """Device buffers (and the q interleave programs) for the structure of the
        numpy H2Matrix `h2`, without uploading anything."""
        device = torch.device(device or "cuda")
        depth = h2.tree.depth
        levels = cls.layouts_from_host(h2)
        leaf = levels[depth]
        aoff, asize = {}, 0
        for (i, j) in leaf.near_pairs:
            aoff[(i, j)] = asize
            asize += int(leaf.n[i] * leaf.n[j])
        q = {l: torch.empty(lay.qsize, dtype=F64, device=device) for l, lay in levels.items()}
        s = {l: torch.empty(max(lay.ssize, 1), dtype=F64, device=device) for l, lay in levels.items()}
        leaf_a = torch.empty(max(asize, 1), dtype=F64, device=device)
        out = cls(device, depth, h2.count, levels, q, s, leaf_a, aoff)
        out._qsplit, out._qprog = _q_interleave(levels, q, device)
        # a to_pinned_host matrix whose levels carry the compact-WY form: those levels upload
        # Y, Yt and the signs instead of q_full, and q_full is rebuilt on the device
        arena = getattr(h2, "_arena", None)
        if arena is not None and getattr(arena, "wy_levels", ()) and arena.intact(h2):
            from .basis_qr import WYLevel, rebuild_qfull, wy_operands
            from .program import Program

            out._wyprog = {}
            for l in arena.wy_levels:
                lay = levels[l]
                wyl = WYLevel(device, lay.n, lay.k)
                out.wy[l] = wyl
                pg = Program(device)
                rebuild_qfull(wyl, pg, lambda i, l=l, lay=lay: q[l].data_ptr() + 8 * int(lay.qoff[i]))
                wy_operands(wyl, pg)
                out._wyprog[l] = pg.finalize()
        return out

    @classmethod
    def from_host(cls, h2, device=None, into=None, on_level=None, stream=None):
        """Upload the numpy arrays of `h2` (bases, leaf near blocks, couplings).

        The blocks are gathered in parallel (numpy releases the GIL) into one
        reusable pinned staging buffer and copied to HBM asynchronously, level
        by level from the leaves up (leaf near blocks with the leaf level).
        With `into` (a DeviceH2 of the same structure) its device buffers are
        reused.  With `stream` the copies run there and, once level l is
        complete on that stream, `on_level(l, event)` lets the caller queue the
        compute that needs it (the factorization of level l overlaps the upload
        of the levels above).
        """
        device = torch.device(device or "cuda")
        depth = h2.tree.depth
        if depth == 0:
            a = np.ascontiguousarray(h2.near_blocks[(0, 0, 0)], dtype=np.float64)
            root_a = torch.from_numpy(a).to(device)
            return cls(device, 0, h2.count, {}, {}, {}, None, {}, root_a=root_a)
        if into is None:
            into = cls.allocate_for_host(h2, device)
        levels, leaf, aoff = into.levels, into.levels[depth], into.aoff
        q, s, leaf_a, qsplit, qprog = into.q, into.s, into.leaf_a, into._qsplit, into._qprog
        regions, off = into.staging_regions()
        st = stream if stream is not None else torch.cuda.current_stream(device)
        # the q interleave kernels run on their own high-priority stream: on the copy stream they
        # would hold back the next DMA until they got SMs away from the factorization
        fix = _fix_stream(device)
        st.wait_stream(fix)                   # an earlier upload's interleave still reading qsplit

        def level_done(l):
            ev = torch.cuda.Event()
            ev.record(st)
            fix.wait_event(ev)
            if on_level is not None:
                ev2 = torch.cuda.Event()
                ev2.record(fix)
                on_level(l, ev2)

        def interleave(l):
            ev = torch.cuda.Event()
            ev.record(st)
            fix.wait_event(ev)
            qprog[l].run(fix)

        arena = getattr(h2, "_arena", None)
        if arena is not None and arena.signature == into.signature() and arena.intact(h2):
            # the blocks already sit in one pinned buffer in staging layout (to_pinned_host):
            # one DMA per region back to back, no host gather
            with torch.cuda.stream(st):
                for kind, l, base, size in regions:
                    if kind == "w":
                        # compact-WY level: Y, Yt, signs; q_full is rebuilt from them (its q
                        # region stays in the arena for the numpy views but is not copied)
                        wyl = into.wy[l]
                        o = base
                        for t, m in zip((wyl.V, wyl.wy_vt, wyl.wy_sgn), wyl.sizes()):
                            t[:m].copy_(arena.tensor[o:o + m], non_blocking=True)
                            o += m
                        ev = torch.cuda.Event()
                        ev.record(st)
                        fix.wait_event(ev)
                        into._wyprog[l].run(fix)
                        continue
                    if kind == "q" and l in into.wy:
                        continue
                    dst = qsplit[l] if kind == "q" else s[l] if kind == "s" else leaf_a
                    dst[:size].copy_(arena.tensor[base:base + size], non_blocking=True)
                    if kind == "q":
                        interleave(l)
                    if (kind == "s" and l != depth) or kind == "a":   # level l complete
                        level_done(l)
            st.wait_stream(fix)
            if stream is None:
                st.synchronize()
            return into
        if into.wy:
            raise RuntimeError("a compact-WY device layout uploads only from its intact pinned arena")
        prev = _STAGING.get("done")
        if prev is not None:
            prev.synchronize()                 # the staging buffer is still being read by the last upload
        host_t, host = _staging(off)
        asize = int(into.leaf_a.numel())
        # chunks of ~0.5M doubles inside one region: gathered by the thread pool, each
        # DMA'd to HBM as soon as it is complete (gather and H2D overlap)
        chunks = []
        for kind, l, base, size in regions:
            lay = levels[l]
            dst = qsplit[l] if kind == "q" else s[l] if kind == "s" else leaf_a
            if kind == "q":
                items = [(int(lay.qoff[i]), int(lay.n[i] * lay.n[i]),
                          (_fill_q, host, base + int(lay.qoff[i]), h2.bases[(l, i)], int(lay.n[i]), int(lay.k[i])))
                         for i in range(lay.nb)]
            elif kind == "s":
                items = [(o, int(lay.k[i] * lay.k[j]), (_fill_flat, host, base + o, h2.couplings[(l, i, j)]))
                         for (i, j), o in lay.soff.items()]
            else:
                items = [(o, int(leaf.n[i] * leaf.n[j]), (_fill_flat, host, base + o, h2.near_blocks[(depth, i, j)]))
                         for (i, j), o in aoff.items()]
            cur, c0, c1 = [], 0, 0
            for o, sz, task in items:
                if cur and (o + sz) - c0 > _CHUNK:
                    chunks.append((l, dst, base, c0, c1, cur))
                    cur, c0 = [], o
                cur.append(task)
                c1 = o + sz
            if cur:
                chunks.append((l, dst, base, c0, c1, cur))
        last_of = {}
        for idx, ch in enumerate(chunks):
            last_of[ch[0]] = idx
        futs = [_pool().submit(_run_tasks, ch[5]) for ch in chunks]
        with torch.cuda.stream(st):
            for idx, ((l, dst, base, c0, c1, _), fu) in enumerate(zip(chunks, futs)):
                fu.result()
                dst[c0:c1].copy_(host_t[base + c0:base + c1], non_blocking=True)
                if last_of.get(l) == idx:
                    interleave(l)                # [q_red | q_skel] rows of level l, on the device
                    level_done(l)
        st.wait_stream(fix)
        done = torch.cuda.Event()
        done.record(st)
        _STAGING["done"] = done
        if stream is None:
            done.synchronize()
        return into

    def staging_regions(self):
        """[(kind, level, offset, size)] of the host staging layout, leaves first:
        [q_L][s_L][a][q_L-1][s_L-1] ... [q_1][s_1] (q: q_red then q_skel per box);
        a compact-WY level puts [Y | Yt | signs] ("w") before its q region."""
        regions, off = [], 0
        asize = int(self.leaf_a.numel())
        for l in range(self.depth, 0, -1):
            lay = self.levels[l]
            if l in self.wy:   # [Y | Yt | signs] of a compact-WY level, first
                nk, k = int((lay.n * lay.k).sum()), int(lay.k.sum())
                regions.append(("w", l, off, 2 * nk + k))
                off += 2 * nk + k
            regions.append(("q", l, off, lay.qsize))
            off += lay.qsize
            regions.append(("s", l, off, max(lay.ssize, 1)))
            off += max(lay.ssize, 1)
            if l == self.depth:
                regions.append(("a", self.depth, off, max(asize, 1)))
                off += max(asize, 1)
        return regions, off

    def ptr_q(self, l, i, col=0):
        lay = self.levels[l]
        return self.q[l].data_ptr() + 8 * int(lay.qoff[i] + col)
