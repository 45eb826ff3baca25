"""Static GPU programs: lists of batched steps plus their descriptors.

A factorization (or a basis construction) is known in full from the box
dimensions before any arithmetic runs, so the host builds every descriptor
once, ships all of them to the device in ONE copy, and the native
executor (h2g_run_program) issues the steps back to back — optionally as
a single CUDA graph replay.  This replaces the reference's per-op Python
planner/executor (dense_core.plan_batches / run_plan, dense_core.py:229-284).
"""

import ctypes
import os

import numpy as np
import torch

from . import _native as nat


def gemm_tiles(m, n, flags=0, cfg=2):
    if m <= 0 or n <= 0:
        return 0
    t = nat.GEMM_TILE[cfg]
    if flags & nat.GEMM_LOWER:
        tm = -(-m // t)
        return tm * (tm + 1) // 2
    return (-(-m // t)) * (-(-n // t))


def choose_tile_cfg(ms, ns, flags, sms=148, trans_b=False, ks=None):
    """Tile configuration of a grouped GEMM launch.

    Measured on B200 (tools/gemm_bench.py, profiles/r01_gemm_tile_configs*.jsonl):
    the 64x64 2-stage DMMA.8x8x4 variant at 4 CTAs/SM (cfg 2) is the fastest for
    the NN / TN transforms (30 TFLOP/s on 4096 x 256^3).  The 3-stage
    m16n8k16 variant at 3 CTAs/SM (cfg 6) is 7-13% faster on isolated K = 64
    NT updates but made the whole factorization slower in place (C2 8.52 ->
    8.56 ms, M1 29.1 -> 29.3 ms).  The 2-stage m8n8k4 kernel at 3 CTAs/SM
    (cfg 7, <= 170 registers) is 12-18% faster on the K <= 64 NT trailing
    updates (profiles/r01_gemm_tile_configs_3.jsonl); those launches use it."""
    if trans_b and ks is not None and len(ks) and int(np.max(ks)) <= 64:
        # ragged small updates (REST of the partial Cholesky): 32x32 tiles when 64x64
        # tiles would execute much more padding
        if _TILE32_RATIO > 0:
            ex64 = sum(gemm_tiles(m, n, f, 7) for m, n, f in zip(ms, ns, flags)) * 4
            ex32 = sum(gemm_tiles(m, n, f, 9) for m, n, f in zip(ms, ns, flags))
            if ex64 > _TILE32_RATIO * ex32:
                return 9
        return 7
    # other ragged launches (small upper-level boxes): 32x32 tiles past the same kind of
    # padding threshold (M1 27.94 -> 27.78 ms, C2 unchanged; profiles/r01_tile32_ab.txt)
    if _TILE32_ALL > 0:
        ex64 = sum(gemm_tiles(m, n, f, 2) for m, n, f in zip(ms, ns, flags)) * 4
        ex32 = sum(gemm_tiles(m, n, f, 9) for m, n, f in zip(ms, ns, flags))
        if ex64 > _TILE32_ALL * ex32:
            return 9
    return 2


_TILE32_RATIO = float(os.environ.get("H2G_TILE32_RATIO", "1.5"))
_TILE32_ALL = float(os.environ.get("H2G_TILE32_ALL", "1.5"))
# split a launch whose problems prefer different tile shapes into a 64x64 launch and a 32x32
# launch (each problem goes where its own padding is smaller); 0 disables
_SPLIT_RATIO = float(os.environ.get("H2G_GEMM_SPLIT", "1.5"))


_SPLITK = int(os.environ.get("H2G_SPLITK", "1"))   # largest split-K factor (1: off; measured slower in place)
_SPLITK_OVERHEAD = 48                              # partial write + reduction, in units of K


def choose_split(tiles, ks, sms=148, per_sm=4):
    """Split-K factor of a 64x64-tile launch (h2g_gemm_grouped_split): the S in {1, 2, 4, 8}
    minimising waves(S) x (K_max / S + overhead), waves(S) = ceil(tiles S / (sms x 4 CTAs)).
    Only launches under ~2 waves with long K gain (the few-box upper levels)."""
    if _SPLITK <= 1 or tiles <= 0 or not len(ks):
        return 1
    kmax = int(np.max(ks))
    slots = sms * per_sm
    best, best_cost = 1, -(-tiles // slots) * kmax
    s = 2
    while s <= _SPLITK:
        if kmax // s >= 64:
            cost = -(-tiles * s // slots) * (kmax / s + _SPLITK_OVERHEAD)
            if cost < 0.9 * best_cost:
                best, best_cost = s, cost
        s *= 2
    return best


_CARVE = os.environ.get("H2G_GEMM_CARVE", "1") != "0"
_BIG_CFG = int(os.environ.get("H2G_BIG_CFG", "2"))   # tile config of the large plain launches (A/B: 2 or 11)


def carve_edges(p, trans_a, trans_b):
    """(interior, [edge strips]) of a plain (non-LOWER, no ext) problem whose M or N ends
    in a remainder of 1..32 past a multiple of 64: the interior keeps the 64x64 tiles, the
    bottom / right strips go to the 32x32-tile launch (sub-problems are pointer offsets of
    the same operands, disjoint parts of C).  None when nothing is carved."""
    A, B, C, M, N, K, lda, ldb, ldc, flags, alpha, beta = p[:12]
    if len(p) > 12 or flags & nat.GEMM_LOWER or M < 64 or N < 64:
        return None
    rm, rn = M % 64, N % 64
    mi = M - rm if 0 < rm <= 32 else M
    ni = N - rn if 0 < rn <= 32 else N
    if mi == M and ni == N:
        return None

    def sub(m0, n0, m, n):
        a = A + 8 * (m0 if trans_a else m0 * lda)
        b = B + 8 * (n0 * ldb if trans_b else n0)
        return (a, b, C + 8 * (m0 * ldc + n0), m, n, K, lda, ldb, ldc, flags, alpha, beta)

    edges = []
    if mi < M:
        edges.append(sub(mi, 0, M - mi, N))
    if ni < N:
        edges.append(sub(0, ni, mi, N - ni))
    return sub(0, 0, mi, ni), edges


def split_by_tile(problems):
    """(problems for 64x64 tiles, problems for 32x32 tiles): a problem goes to the 32x32
    launch when its 64x64 tiles would execute more than _SPLIT_RATIO x the 32x32 tiles'
    work (ragged sizes of the upper-level boxes)."""
    big, small = [], []
    for p in problems:
        m, n, f = int(p[3]), int(p[4]), int(p[9])
        (small if 4 * gemm_tiles(m, n, f, 2) > _SPLIT_RATIO * gemm_tiles(m, n, f, 9) else big).append(p)
    return big, small


def copy_tiles(rows, cols):
    if rows <= 0 or cols <= 0:
        return 0
    return (-(-rows // nat.COPY_TILE)) * (-(-cols // nat.COPY_TILE))


def _ablated_lanes():
    """H2G_ABLATE_LANES="3,4" turns every step of those lanes into a NOP (events kept).
    Measurement aid for critical-path analysis only: the results are wrong."""
    v = os.environ.get("H2G_ABLATE_LANES", "")
    return {int(x) for x in v.split(",") if x.strip()}


class Program:
    """Accumulates steps; `finalize()` uploads descriptors and resolves pointers."""

    def __init__(self, device):
        self.device = device
        self._blobs = []      # numpy byte arrays (descriptors and maps)
        self._steps = []      # dicts: kind, count, grid, arg, descs, map, npd, aux, d0, d1
        self.dev_blob = None
        self.steps = None
        self.graph = None
        self.kernel_launches = 0
        self._keep = []       # device buffers the steps point into (CHOL_PANEL sync words)
        self.work = []        # per step: (label, flops, bytes) of useful work, for the roofline
        self.exec_flops = []  # per step: DMMA flops the tiles execute (GEMM: padded to whole tiles)
        self.lane = 0         # lane of the steps added next (0: caller's stream, 1..4: side streams)
        self.role = None      # role tag of the steps added next (write audit: "transform", "factor", ...)
        self.record_writes = False
        self.writes = []      # (step, role, ptr, rows, cols, ld, lower): matrix extents the steps write
        self.n_events = 0
        self.ctx = None

    @property
    def sms(self):
        v = self.__dict__.get("_sms")
        if v is None:
            try:
                v = torch.cuda.get_device_properties(self.device).multi_processor_count
            except (RuntimeError, AssertionError, AttributeError):
                v = 148
            self._sms = v
        return v

    # -- blob bookkeeping -------------------------------------------------------------
    def _blob(self, arr):
        if arr is None:
            return -1
        self._blobs.append(np.ascontiguousarray(arr).view(np.uint8).reshape(-1))
        return len(self._blobs) - 1

    def _writes(self, extents):
        """Record the extents (ptr, rows, cols, ld, lower) the step added next writes."""
        if self.record_writes:
            q = len(self._steps)
            self.writes.extend((q, self.role, int(p), int(r), int(c), int(ld), bool(lo)) for p, r, c, ld, lo in extents)

    def _add(self, kind, count, grid, descs=-1, map_=-1, npd=0, arg=0, aux=0, d0=0.0, d1=0.0, flops=0, nbytes=0,
             wait=-1, rec=-1, exec_flops=None):
        self.work.append((kind, int(flops), int(nbytes)))
        self.exec_flops.append(int(flops if exec_flops is None else exec_flops))
        self._steps.append(dict(kind=kind, count=int(count), grid=int(grid), descs=descs, map=map_, npd=npd,
                                arg=int(arg), aux=aux, d0=float(d0), d1=float(d1), lane=self.lane,
                                wait=int(wait), rec=int(rec)))

    # -- multi-lane scheduling ----------------------------------------------------------
    def event(self):
        self.n_events += 1
        return self.n_events - 1

    def record(self, ev):
        """Record `ev` on the current lane (after the steps added so far)."""
        self._add(nat.STEP["NOP"], 0, 0, rec=ev)

    def wait(self, ev):
        """Make the current lane wait for `ev`."""
        self._add(nat.STEP["NOP"], 0, 0, wait=ev)

    # -- step constructors ------------------------------------------------------------
    def gemm(self, trans_a, trans_b, problems, tile_cfg=None, split=False):
        """problems: iterable of (A, B, C, M, N, K, lda, ldb, ldc, flags, alpha, beta[, ext]) with
        ext = (Cin, sgn, ldcin, remap_k) (h2g_gemm_ext: a separate beta source and / or the
        compact-WY relabel store); a launch with any ext carries the array for all its problems."""
        rows = [p for p in problems if p[3] > 0 and p[4] > 0]
        if not rows:
            return 0
        if tile_cfg is None and _SPLIT_RATIO > 0 and len(rows) > 1:
            big, small = split_by_tile(rows)
            if big and _CARVE:
                carved = []
                for p in big:
                    c = carve_edges(p, trans_a, trans_b)
                    if c is None:
                        carved.append(p)
                    else:
                        carved.append(c[0])
                        small.extend(c[1])
                big = carved
            if big and small:
                return (self.gemm(trans_a, trans_b, big, split=split)
                        + self.gemm(trans_a, trans_b, small, tile_cfg=9))
        arr = np.zeros(len(rows), dtype=nat.GEMM_DT)
        cols = list(zip(*[p[:12] for p in rows]))
        for name, col in zip(("A", "B", "C", "M", "N", "K", "lda", "ldb", "ldc", "flags", "alpha", "beta"), cols):
            arr[name] = col
        aux = 0
        if any(len(p) > 12 for p in rows):
            ext = np.zeros(len(rows), dtype=nat.GEMM_EXT_DT)
            ext["remap_k"] = -1
            for q, p in enumerate(rows):
                if len(p) > 12:
                    ext[q] = p[12]
            aux = ("blob", self._blob(ext))
        cfg = (choose_tile_cfg(arr["M"], arr["N"], arr["flags"], trans_b=bool(trans_b), ks=arr["K"])
               if tile_cfg is None else tile_cfg)
        if tile_cfg is None and cfg == 2 and _BIG_CFG != 2 and not (split and _SPLITK > 1):
            cfg = _BIG_CFG
        tiles = np.array([gemm_tiles(m, n, f, cfg) for m, n, f in zip(arr["M"], arr["N"], arr["flags"])],
                         dtype=np.int64)
        nsplit = choose_split(int(tiles.sum()), arr["K"], self.sms) if (split and cfg == 2 and not aux) else 1
        ctas = tiles * nsplit
        starts = np.concatenate([[0], np.cumsum(ctas)[:-1]])
        arr["tile_start"] = starts
        total = int(ctas.sum())
        tmap = np.repeat(np.arange(len(rows), dtype=np.int32), ctas)
        ws = 0
        if nsplit > 1:
            wsb = int(nat.lib().h2g_gemm_split_workspace(int(tiles.sum()), nsplit))
            wst = torch.zeros((wsb + 7) // 8, dtype=torch.float64, device=self.device)
            self._keep.append(wst)
            ws = wst.data_ptr()
            cfg_arg = cfg | (nsplit << 8)
        # K == 0 problems still need their beta*C epilogue; keep them (tiles > 0)
        kind = nat.STEP["GEMM_NN"] + 2 * int(bool(trans_a)) + int(bool(trans_b))
        self._writes((p[2], p[3], p[4], p[8], p[9] & nat.GEMM_LOWER) for p in rows)
        m64, n64, k64 = arr["M"].astype(np.int64), arr["N"].astype(np.int64), arr["K"].astype(np.int64)
        lower = (arr["flags"] & nat.GEMM_LOWER) != 0
        fl = np.where(lower, m64 * (m64 + 1) * k64, 2 * m64 * n64 * k64).sum()
        t = nat.GEMM_TILE[cfg]
        ex = int((tiles * 2 * t * t * (-(-k64 // 16) * 16)).sum())   # whole t x t tiles, K padded to 16
        self._add(kind, len(rows), total, self._blob(arr), self._blob(tmap), flops=fl,
                  arg=cfg_arg if nsplit > 1 else cfg, exec_flops=ex, aux=aux, npd=ws)
        return total

    def chol_panel(self, descs, npd_ptr):
        """descs: list of (H, Linv, ldh, ldl, n, p, b, npd_slot): one diag CTA per box plus one
        CTA per 64-row chunk below the panel (h2g_chol_panel)."""
        if not descs:
            return 0
        arr = np.zeros(len(descs), dtype=nat.CHOLP_DT)
        for name, col in zip(("H", "Linv", "ldh", "ldl", "n", "p", "b", "npd_slot"), zip(*descs)):
            arr[name] = col
        below = (arr["n"].astype(np.int64) - arr["p"] - arr["b"]).clip(min=0)
        tiles = -(-below // nat.PANEL_WIDTH)
        arr["tile_start"] = np.concatenate([[0], np.cumsum(tiles)[:-1]])
        tmap = np.repeat(np.arange(len(descs), dtype=np.int32), tiles)
        b64 = arr["b"].astype(np.int64)
        # useful flops: previous-panel update of block column p (K = 64) + chol + TRSM of the rows below
        upd = np.where(arr["p"] > 0, (b64 * (b64 + 1) + 2 * below * b64) * nat.PANEL_WIDTH, 0)
        fl = int((upd + b64 ** 3 // 3 + below * b64 * b64).sum())
        # the panel's diagonal block (lower) and the rows below it, columns p .. p+b
        self._writes((d[0] + 8 * (d[5] * d[2] + d[5]), d[4] - d[5], d[6], d[2], False) for d in descs)
        # ticket / flag words of the one-launch variant (h2g_chol_panel_sync), zero between launches
        sync = torch.zeros(2 * len(descs) + 2, dtype=torch.int32, device=self.device)
        self._keep.append(sync)
        self._add(nat.STEP["CHOL_PANEL"], len(descs), int(tiles.sum()), self._blob(arr),
                  self._blob(tmap) if tmap.size else -1, npd=npd_ptr, aux=sync.data_ptr(), flops=fl)
        return int(tiles.sum())

    def chol_box(self, descs, npd_ptr):
        """descs: list of (H, Linv, n, r, ldh, npd_slot[, Q, R]): the fused per-box partial Cholesky
        (h2g_chol_box, one CTA per box); with Q / R also V = q_red L^-T into R."""
        descs = [d for d in descs if d[3] > 0]
        if not descs:
            return 0
        arr = np.zeros(len(descs), dtype=nat.CHOLBOX_DT)
        for name, col in zip(("H", "Linv", "n", "r", "ldh", "npd_slot"), zip(*[d[:6] for d in descs])):
            arr[name] = col
        if len(descs[0]) > 6:
            arr["Q"] = [d[6] for d in descs]
            arr["R"] = [d[7] for d in descs]
            descs = [d if d[6] else d[:6] for d in descs]
        role = self.role
        self.role = "factor"      # RR -> L(r), SR -> L(s) in place
        self._writes((d[0], d[2], d[3], d[4], False) for d in descs)
        self.role = "schur"       # the single SS -= L(s) L(s)^T
        self._writes((d[0] + 8 * (d[3] * d[4] + d[3]), d[2] - d[3], d[2] - d[3], d[4], True) for d in descs if d[2] > d[3])
        self.role = "v"
        self._writes((d[7], d[2], d[3], d[4], False) for d in descs if len(d) > 6)
        self.role = role
        n64, r64 = arr["n"].astype(np.int64), arr["r"].astype(np.int64)
        k64 = n64 - r64
        fl = (r64 ** 3 // 3 + r64 * r64 * k64 + 2 * k64 * k64 * r64).sum()       # chol + trsm of SR + Schur
        fl += np.where(arr["Q"] != 0, n64 * r64 * r64, 0).sum()                     # V = q_red L^-T
        self._add(nat.STEP["CHOL_BOX"], len(descs), len(descs), self._blob(arr), npd=npd_ptr, flops=int(fl))
        return len(descs)

    def trsm_rows(self, descs):
        """descs: list of (Lb, Xin, Xout, Linv, rows, cols, q_begin, q_end, ldlb, ldx): X = B L^-T for
        the block columns [q_begin, q_end) (h2g_trsm_rows), one CTA per 64-row chunk."""
        descs = [d for d in descs if d[4] > 0 and d[5] > 0 and d[7] > d[6]]
        if not descs:
            return 0
        arr = np.zeros(len(descs), dtype=nat.ROWS_DT)
        for name, col in zip(("Lb", "Xin", "Xout", "Linv", "rows", "cols", "q_begin", "q_end", "ldlb", "ldx"),
                             zip(*descs)):
            arr[name] = col
        tiles = -(-arr["rows"].astype(np.int64) // nat.PANEL_WIDTH)
        arr["tile_start"] = np.concatenate([[0], np.cumsum(tiles)[:-1]])
        tmap = np.repeat(np.arange(len(descs), dtype=np.int32), tiles)
        self._writes((d[2] + 8 * nat.PANEL_WIDTH * d[6], d[4], min(d[5], nat.PANEL_WIDTH * d[7]) - nat.PANEL_WIDTH * d[6],
                      d[9], False) for d in descs)
        fl = 0
        W = nat.PANEL_WIDTH
        for d in descs:   # useful flops: rows x b x (2 p + b) per panel (update + triangular solve)
            for q in range(d[6], d[7]):
                p, b = W * q, min(W, d[5] - W * q)
                m = d[4] if d[1] else min(d[4], p + b)
                fl += m * b * (2 * p + b)
        self._add(nat.STEP["TRSM_ROWS"], len(descs), int(tiles.sum()), self._blob(arr), self._blob(tmap), flops=fl)
        return int(tiles.sum())

    def copy(self, descs):
        """descs: list of (src, dst, rows, cols, lds, ldd, mode)."""
        rows = [d for d in descs if d[2] > 0 and d[3] > 0]
        if not rows:
            return 0
        arr = np.zeros(len(rows), dtype=nat.COPY_DT)
        cols = list(zip(*rows))
        for name, col in zip(("src", "dst", "rows", "cols", "lds", "ldd", "mode"), cols):
            arr[name] = col
        self._writes((d[1], d[2], d[3], d[5], False) for d in rows)
        tiles = np.array([copy_tiles(r, c) for r, c in zip(arr["rows"], arr["cols"])], dtype=np.int64)
        arr["tile_start"] = np.concatenate([[0], np.cumsum(tiles)[:-1]])
        tmap = np.repeat(np.arange(len(rows), dtype=np.int32), tiles)
        self._add(nat.STEP["COPY"], len(rows), int(tiles.sum()), self._blob(arr), self._blob(tmap),
                  nbytes=16 * int((arr["rows"].astype(np.int64) * arr["cols"]).sum()))
        return int(tiles.sum())

    def memcpy(self, dst_ptr, src_ptr, nbytes):
        """Device-to-device copy (split into <= 1 GiB steps: the step count is int32)."""
        nbytes = int(nbytes)
        self._writes([(dst_ptr, 1, nbytes // 8, nbytes // 8, False)])
        off = 0
        while off < nbytes:
            sz = min(nbytes - off, 1 << 30)
            self._add(nat.STEP["MEMCPY"], sz, 0, ("raw", dst_ptr + off), ("raw", src_ptr + off), nbytes=2 * sz)
            off += sz

    def qr_panel(self, descs):
        """descs: list of (Z, V, tau, T, n, ldz, p, b)."""
        if not descs:
            return 0
        arr = np.zeros(len(descs), dtype=nat.QRP_DT)
        for name, col in zip(("Z", "V", "tau", "T", "n", "ldz", "p", "b"), zip(*descs)):
            arr[name] = col
        max_rows = int((arr["n"].astype(np.int64) - arr["p"]).max())
        self._add(nat.STEP["QR_PANEL"], len(descs), len(descs), self._blob(arr), arg=max_rows)
        return len(descs)

    def basis(self, descs):
        """descs: list of (Q, Z, qfull, frame, n, k, ldz)."""
        if not descs:
            return 0
        arr = np.zeros(len(descs), dtype=nat.BASIS_DT)
        for name, col in zip(("Q", "Z", "qfull", "frame", "n", "k", "ldz"), zip(*descs)):
            arr[name] = col
        self._add(nat.STEP["BASIS"], len(descs), len(descs), self._blob(arr))
        return len(descs)

    def gemv(self, outs, w, balance=0):
        """outs: list of (y, y2, init, m, split, flags, [terms...]) with terms (A, x, lda, trans, K).

        balance > 0: when the launch has fewer than `balance` 64-row chunks (CTAs), outputs
        with several terms are split into contiguous term groups of about equal bytes, each
        summed into its own partial vector by one launch, and a second launch forms
        y = init -/+ (P_1 + ... + P_p) with identity terms.  The summation order is fixed
        by the structure (term order, then group order), so results stay deterministic."""
        outs = [o for o in outs if o[3] > 0]
        if not outs:
            return 0
        if balance:
            outs, final = self._balance_gemv(outs, w, balance)
            n = self._gemv_step(outs, w)
            if final:
                self._gemv_step(final, w)
            return n
        return self._gemv_step(outs, w)

    def _balance_gemv(self, outs, w, target):
        chunk = nat.GEMV_CHUNK
        nchunks = sum(-(-int(o[3]) // chunk) for o in outs)
        if nchunks >= target:
            return outs, []
        obytes = [8 * int(o[3]) * sum(int(t[4]) for t in o[6]) for o in outs]
        per_cta = max(sum(obytes) / target, 1.0)
        plan = []
        for o, by in zip(outs, obytes):
            m, terms = int(o[3]), o[6]
            ktot = sum(int(t[4]) for t in terms)
            p = min(max(1, ktot // 64), max(1, int(round(by / (per_cta * -(-m // chunk))))))
            if p <= 1:
                plan.append((o, None))
                continue
            if p > len(terms):
                # cut the terms along K (64-multiples) so that p groups can be formed
                kp = -(-ktot // p)
                kp = -(-kp // 64) * 64
                cut = []
                for (a, x, lda, trans, k) in terms:
                    if not a:                    # identity term: K must stay = m
                        cut.append((a, x, lda, trans, k))
                        continue
                    for k0 in range(0, int(k), kp):
                        kk = min(kp, int(k) - k0)
                        step = 8 * k0 * (int(lda) if trans else 1)
                        cut.append((a + step, x + 8 * k0 * w, lda, trans, kk))
                terms = cut
            tb = np.cumsum([8 * m * int(t[4]) for t in terms], dtype=np.float64)
            cuts = sorted({int(np.searchsorted(tb, by * q / p, side="left")) for q in range(1, p)})
            bounds = [0] + [c + 1 for c in cuts if 0 <= c < len(terms) - 1] + [len(terms)]
            groups = [terms[a:b] for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
            plan.append((o, groups) if len(groups) > 1 else (o, None))
        elems = sum(int(o[3]) * w * len(g) for o, g in plan if g)
        if elems == 0:
            return outs, []
        part = torch.empty(elems, dtype=torch.float64, device=self.device)
        self._keep.append(part)
        base = part.data_ptr()
        new, final = [], []
        for o, groups in plan:
            if groups is None:
                new.append(o)
                continue
            y, y2, init, m, split, flags, _ = o
            ids = []
            for g in groups:
                new.append((base, 0, 0, m, 0, nat.GEMV_PLUS, list(g)))
                ids.append((0, base, 0, 0, m))
                base += 8 * int(m) * w
            final.append((y, y2, init, m, split, flags, ids))
        return new, final

    def _gemv_step(self, outs, w):
        oarr = np.zeros(len(outs), dtype=nat.GEMV_OUT_DT)
        tl = []
        chunks = 0
        nbytes = 0
        for q, (y, y2, init, m, split, flags, tms) in enumerate(outs):
            oarr[q] = (y, y2, init, m, split, len(tl), len(tl) + len(tms), flags, chunks)
            chunks += -(-int(m) // nat.GEMV_CHUNK)
            tl.extend(tms)
            nbytes += 8 * int(m) * sum(int(t[4]) for t in tms if t[0])   # matrix bytes (identity terms: none)
        tarr = np.zeros(max(len(tl), 1), dtype=nat.GEMV_TERM_DT)
        for q, (a, x, lda, trans, k) in enumerate(tl):
            tarr[q] = (a, x, lda, trans, k, 0)
        cmap = np.repeat(np.arange(len(outs), dtype=np.int32),
                         [-(-int(o[3]) // nat.GEMV_CHUNK) for o in outs])
        self._add(nat.STEP["GEMV"], len(outs), chunks, self._blob(oarr), self._blob(tarr), arg=w, nbytes=nbytes,
                  aux=("blob", self._blob(cmap)))
        return len(outs)

    def xform_t(self, descs, w):
        """descs: list of (Q, x, y1, y2, n, split, ldq): [y1; y2] = Q^T x (h2g_xform_t)."""
        descs = [d for d in descs if d[4] > 0]
        if not descs:
            return 0
        arr = np.zeros(len(descs), dtype=nat.XFORM_DT)
        for name, col in zip(("Q", "x", "y1", "y2", "n", "split", "ldq"), zip(*descs)):
            arr[name] = col
        tiles = -(-arr["n"].astype(np.int64) // 128)
        arr["tile_start"] = np.concatenate([[0], np.cumsum(tiles)[:-1]])
        tmap = np.repeat(np.arange(len(descs), dtype=np.int32), tiles)
        vec = bool(((arr["Q"] % 16) == 0).all() and ((arr["ldq"] % 2) == 0).all())
        n64 = arr["n"].astype(np.int64)
        nbytes = 8 * int((n64 * n64).sum()) + 16 * int(n64.sum()) * w
        # count < 0 tells the executor every Q row is 16-byte aligned
        self._add(nat.STEP["XFORM_T"], -len(descs) if vec else len(descs), int(tiles.sum()), self._blob(arr),
                  self._blob(tmap), arg=w, nbytes=nbytes)
        return int(tiles.sum())

    def xform_n(self, descs, w):
        """descs: list of (Q, xr, xs, out, n, r, ldq): out = Q [xr; xs] (h2g_xform_n)."""
        descs = [d for d in descs if d[4] > 0]
        if not descs:
            return 0
        if max(d[4] for d in descs) > 4096:
            raise ValueError("h2g_xform_n: box size above 4096")
        arr = np.zeros(len(descs), dtype=nat.XFORMN_DT)
        for name, col in zip(("Q", "xr", "xs", "out", "n", "r", "ldq"), zip(*descs)):
            arr[name] = col
        rows = nat.lib().h2g_xform_n_rows()
        tiles = -(-arr["n"].astype(np.int64) // rows)
        arr["tile_start"] = np.concatenate([[0], np.cumsum(tiles)[:-1]])
        tmap = np.repeat(np.arange(len(descs), dtype=np.int32), tiles)
        vec = bool(((arr["Q"] % 16) == 0).all() and ((arr["ldq"] % 2) == 0).all())
        n64 = arr["n"].astype(np.int64)
        nbytes = 8 * int((n64 * n64).sum()) + 16 * int(n64.sum()) * w
        self._add(nat.STEP["XFORM_N"], -len(descs) if vec else len(descs), int(tiles.sum()), self._blob(arr),
                  self._blob(tmap), arg=w, nbytes=nbytes, d0=float(n64.max()))
        return int(tiles.sum())

    def trsv(self, descs, trans, w):
        """descs: list of (L, Linv, x, n, ldl)."""
        descs = [d for d in descs if d[3] > 0]
        if not descs:
            return 0
        arr = np.zeros(len(descs), dtype=nat.TRSV_DT)
        for q, d in enumerate(descs):
            arr[q] = d
        nbytes = sum(4 * int(d[3]) * (int(d[3]) + 1) for d in descs)
        self._add(nat.STEP["TRSV"], len(descs), w, self._blob(arr), arg=trans, nbytes=nbytes)
        return len(descs)

    def symcheck(self, descs, out_ptr):
        """descs: list of (A, n, lda); out: 2 x len(descs) u64 (max |A - A^T|, max |A|)."""
        if not descs:
            return 0
        arr = np.zeros(len(descs), dtype=nat.SYMCHECK_DT)
        for name, col in zip(("A", "n", "lda"), zip(*descs)):
            arr[name] = col
        nbytes = 8 * int((arr["n"].astype(np.int64) ** 2).sum()) * 2
        self._add(nat.STEP["SYMCHECK"], len(descs), len(descs), self._blob(arr), aux=out_ptr, nbytes=nbytes)
        return len(descs)

    def triinv(self, descs, status_ptr):
        """descs: list of (L, Linv, n, ldl, status_slot): inverses of the 64 x 64 diagonal blocks."""
        descs = [d for d in descs if d[2] > 0]
        if not descs:
            return 0
        arr = np.zeros(len(descs), dtype=nat.TRIINV_DT)
        for name, col in zip(("L", "Linv", "n", "ldl", "status_slot"), zip(*descs)):
            arr[name] = col
        tiles = -(-arr["n"].astype(np.int64) // nat.PANEL_WIDTH)
        arr["tile_start"] = np.concatenate([[0], np.cumsum(tiles)[:-1]])
        tmap = np.repeat(np.arange(len(descs), dtype=np.int32), tiles)
        self._add(nat.STEP["TRIINV"], len(descs), int(tiles.sum()), self._blob(arr), self._blob(tmap),
                  npd=status_ptr)
        return int(tiles.sum())

    def kblock(self, descs, points_ptr, family, shift, decay, flag_ptr):
        """descs: list of (rows_ptr, cols_ptr, out_ptr, m, n, ldo)."""
        descs = [d for d in descs if d[3] > 0 and d[4] > 0]
        if not descs:
            return 0
        arr = np.zeros(len(descs), dtype=nat.KBLOCK_DT)
        for name, col in zip(("rows", "cols", "out", "m", "n", "ldo"), zip(*descs)):
            arr[name] = col
        tiles = (-(-arr["m"].astype(np.int64) // 32)) * (-(-arr["n"].astype(np.int64) // 32))
        arr["tile_start"] = np.concatenate([[0], np.cumsum(tiles)[:-1]])
        tmap = np.repeat(np.arange(len(descs), dtype=np.int32), tiles)
        self._add(nat.STEP["KBLOCK"], len(descs), int(tiles.sum()), self._blob(arr), self._blob(tmap),
                  npd=flag_ptr, arg=family, aux=points_ptr, d0=shift, d1=decay)
        return int(tiles.sum())

    # -- finalize / run ---------------------------------------------------------------
    def finalize(self):
        offs, total = [], 0
        for b in self._blobs:
            offs.append(total)
            total += (b.size + 255) // 256 * 256
        host = torch.zeros(max(total, 256), dtype=torch.uint8, pin_memory=True)
        hv = host.numpy()
        for o, b in zip(offs, self._blobs):
            hv[o:o + b.size] = b
        self.dev_blob = host.to(self.device, non_blocking=True)
        self._host_blob = host  # keep pinned source alive until the copy completes
        base = self.dev_blob.data_ptr()
        steps = np.zeros(len(self._steps), dtype=nat.STEP_DT)

        def resolve(v):
            if isinstance(v, tuple):
                return v[1]
            return base + offs[v] if v >= 0 else 0

        ablate = _ablated_lanes()
        for q, st in enumerate(self._steps):
            steps[q]["kind"] = nat.STEP["NOP"] if st["lane"] in ablate else st["kind"]
            steps[q]["count"] = st["count"]
            steps[q]["grid"] = st["grid"]
            steps[q]["arg"] = st["arg"]
            steps[q]["descs"] = resolve(st["descs"])
            steps[q]["map"] = resolve(st["map"])
            steps[q]["npd"] = st["npd"]
            aux = st["aux"]
            steps[q]["aux"] = base + offs[aux[1]] if isinstance(aux, tuple) else aux
            steps[q]["d0"] = st["d0"]
            steps[q]["d1"] = st["d1"]
            steps[q]["lane"] = st["lane"]
            steps[q]["wait_ev"] = st["wait"]
            steps[q]["rec_ev"] = st["rec"]
        self.steps = steps
        # CHOL_PANEL issues a diag kernel plus, when rows lie below the panel, a row-chunk kernel
        fused_max = nat.lib().h2g_chol_panel_fused_max()
        self.kernel_launches = int(sum((2 if st["kind"] == nat.STEP["CHOL_PANEL"] and st["grid"] > 0
                                        and st["count"] > fused_max else 1)
                                       for st in self._steps
                                       if st["kind"] not in (nat.STEP["MEMCPY"], nat.STEP["NOP"])))
        if any(st["lane"] for st in self._steps):
            ctx = ctypes.c_void_p()
            nat.check(nat.lib().h2g_exec_ctx_create(max(self.n_events, 1), ctypes.byref(ctx)), "h2g_exec_ctx_create")
            self.ctx = ctx
        self.step_kinds = [st["kind"] for st in self._steps]
        self._blobs = []
        return self

    def run(self, stream=None):
        lib = nat.lib()
        rc = lib.h2g_run_program(self.steps.ctypes.data_as(ctypes.c_void_p), len(self.steps), nat.stream_ptr(stream),
                                 self.ctx)
        nat.check(rc, "h2g_run_program")

    def run_timed(self, stream=None):
        """Eager run with an event pair around every step; returns per-step ms."""
        out = np.zeros(len(self.steps), dtype=np.float32)
        rc = nat.lib().h2g_run_program_timed(self.steps.ctypes.data_as(ctypes.c_void_p), len(self.steps),
                                             nat.stream_ptr(stream), out.ctypes.data_as(ctypes.c_void_p))
        nat.check(rc, "h2g_run_program_timed")
        return out

    def capture(self, stream=None):
        """Capture the whole program into one CUDA graph (on a side stream)."""
        lib = nat.lib()
        s = stream if stream is not None else torch.cuda.Stream(device=self.device)
        torch.cuda.current_stream(self.device).synchronize()
        exe = ctypes.c_void_p()
        rc = lib.h2g_graph_capture(self.steps.ctypes.data_as(ctypes.c_void_p), len(self.steps),
                                   nat.stream_ptr(s), self.ctx, ctypes.byref(exe))
        nat.check(rc, "h2g_graph_capture")
        self.graph = exe
        return self

    def launch(self, stream=None):
        if self.graph is None:
            return self.run(stream)
        rc = nat.lib().h2g_graph_launch(self.graph, nat.stream_ptr(stream))
        nat.check(rc, "h2g_graph_launch")

    def __del__(self):
        try:
            if getattr(self, "graph", None) is not None:
                nat.load_library().h2g_graph_destroy(self.graph)
            if getattr(self, "ctx", None) is not None:
                nat.load_library().h2g_exec_ctx_destroy(self.ctx)
        except Exception:
            pass
