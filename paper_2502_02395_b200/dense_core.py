"""Host-side pieces of the dense engine: the basis container, the skeleton
(interpolative-decomposition) selection and the reference flop model.

What stays on the host and why
  * `skeleton_selection` is the column-pivoted QR (dgeqp3) of the sample
    matrix that chooses the skeleton rows and builds the interpolation
    operator T (dense_core.py:114-134).  The north star requires skeleton
    indices BIT-IDENTICAL to the reference, so it runs through the same
    LAPACK routine on identical samples.
  * `flop_count` / `PhaseFlops` restate the reference's flop model and its
    pad-to-level-max accounting (dense_core.py:166-181, 229-248), so
    `factors.flops` equals the reference's dict exactly and GFLOP/s are
    computed with the same numerator.

Everything numerical on the factorization path (the complete QR of ①,
every GEMM, the partial Cholesky, the merge, the substitution) runs on
the GPU through libh2ulv_b200.so.
"""

from dataclasses import dataclass

import numpy as np
import scipy.linalg


@dataclass
class BasisDecomposition:
    """Orthonormal split [q_red | q_skel] of a box's n unknowns (dense_core.py:24-48)."""

    q_skel: np.ndarray
    q_red: np.ndarray
    skeleton: np.ndarray
    rank: int
    frame: np.ndarray

    @property
    def n(self):
        return self.q_skel.shape[0]

    @property
    def q_full(self):
        return np.hstack([self.q_red, self.q_skel])


@dataclass
class SkeletonChoice:
    """Result of the pivoted-QR half of id_basis for one box."""

    skeleton: np.ndarray  # sorted box-local row ids (int64)
    t: np.ndarray         # n x k interpolation operator, columns follow `skeleton`
    rank: int


_GEQP3_LWORK = {}
_TRTRS = {"fn": None, "tried": False}


def _scipy_trtrs():
    """scipy's own LAPACK dtrtrs (the routine scipy.linalg.solve_triangular calls) via
    ctypes, which drops the GIL for the call; None if the library is not found."""
    if not _TRTRS["tried"]:
        _TRTRS["tried"] = True
        import ctypes
        import glob
        import os

        libs = glob.glob(os.path.join(os.path.dirname(os.path.dirname(scipy.__file__)), "scipy.libs",
                                      "libscipy_openblas*.so"))
        for path in libs:
            try:
                fn = ctypes.CDLL(path).scipy_dtrtrs_
            except (OSError, AttributeError):
                continue
            fn.restype = None
            _TRTRS["fn"] = fn
            break
    return _TRTRS["fn"]


def solve_triangular(a, b, lower):
    """scipy.linalg.solve_triangular(a, b, lower=lower) bit for bit (same dtrtrs call on
    the same operands), with the GIL released; falls back to scipy when the library
    symbol is unavailable."""
    fn = _scipy_trtrs()
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if fn is None or a.ndim != 2 or b.ndim not in (1, 2) or a.shape[0] == 0 or b.size == 0:
        return scipy.linalg.solve_triangular(a, b, lower=lower)
    import ctypes

    n = a.shape[0]
    vec = b.ndim == 1
    bf = np.array(b.reshape(n, -1), dtype=np.float64, order="F", copy=True)
    nrhs = bf.shape[1]
    if a.flags.f_contiguous:
        af, uplo, trans = a, (b"L" if lower else b"U"), b"N"
    else:   # the C buffer read as Fortran is a^T: solve a^T^T x = b (scipy's own choice)
        af, uplo, trans = np.ascontiguousarray(a), (b"U" if lower else b"L"), b"T"
    info = ctypes.c_int(0)
    c = lambda v: ctypes.byref(ctypes.c_char(v))
    i = lambda v: ctypes.byref(ctypes.c_int(v))
    fn(c(uplo), c(trans), c(b"N"), i(n), i(nrhs), af.ctypes.data_as(ctypes.c_void_p), i(n),
       bf.ctypes.data_as(ctypes.c_void_p), i(n), ctypes.byref(info))
    if info.value > 0:
        raise np.linalg.LinAlgError(f"singular matrix: resolution failed at diagonal {info.value - 1}")
    if info.value < 0:
        raise ValueError(f"dtrtrs: illegal argument {-info.value}")
    return bf[:, 0] if vec else bf


def _pivoted_qr_r(at):
    """(R, piv) of scipy.linalg.qr(at, pivoting=True, mode="economic"), bit for bit
    (the same dgeqp3 call with the same optimal workspace on the same Fortran-ordered
    operand), through the raw LAPACK wrapper, which releases the GIL — so the
    skeleton pass's thread pool runs the QRs in parallel (scipy.linalg.qr holds it)."""
    at = np.asfortranarray(at, dtype=np.float64)
    m, n = at.shape
    lw = _GEQP3_LWORK.get((m, n))
    if lw is None:
        lw = int(scipy.linalg.lapack.dgeqp3(at, lwork=-1)[3][0])
        _GEQP3_LWORK[(m, n)] = lw
    qr, jpvt, _, _, info = scipy.linalg.lapack.dgeqp3(at, lwork=lw)
    if info < 0:
        raise ValueError(f"dgeqp3: illegal argument {-info}")
    k = min(m, n)
    return np.triu(qr[:k]), jpvt - 1


def skeleton_selection(samples, rank=None, tol=None):
    """Column-pivoted QR of samples^T -> (skeleton, T, k).

    k = rank (capped by the shape) or the first index whose pivot ratio
    |r_kk / r_00| <= tol; exactly-zero pivots are never kept
    (dense_core.py:114-123).  T[skeleton] = I and the other rows are
    (R11^-1 R12)^T (dense_core.py:125-134).
    """
    if (rank is None) == (tol is None):
        raise ValueError("exactly one of rank/tol must be given")
    a = np.asarray(samples, dtype=np.float64)
    n, m = a.shape
    if m < 1:
        raise ValueError("need at least one sample column")
    r, piv = _pivoted_qr_r(a.T)
    diag = np.abs(np.diag(r))
    if diag.size == 0 or diag[0] == 0.0:
        k = 0
    elif rank is not None:
        k = min(rank, n, m)
    else:
        below = np.flatnonzero(diag / diag[0] <= tol)
        k = int(below[0]) if below.size else min(n, m)
    k = min(k, int(np.count_nonzero(diag > 0)))
    if k == 0:
        return SkeletonChoice(skeleton=np.zeros(0, dtype=np.int64), t=np.zeros((n, 0)), rank=0)
    lead = piv[:k]
    order = np.argsort(lead)
    t = np.zeros((n, k))
    t[lead] = np.eye(k)
    if n > k:
        t[piv[k:]] = solve_triangular(r[:k, :k], r[:k, k:], lower=False).T
    return SkeletonChoice(skeleton=lead[order].astype(np.int64), t=t[:, order], rank=k)


def id_basis(samples, rank=None, tol=None, row_weight=None):
    """Drop-in for the reference `id_basis` (dense_core.py:96-150).

    Skeleton selection on the host (bit-exact), complementary basis (①) by
    the batched GPU Householder QR.
    """
    from . import basis_qr

    choice = skeleton_selection(samples, rank=rank, tol=tol)
    n = np.asarray(samples).shape[0]
    if choice.rank == 0:
        return BasisDecomposition(q_skel=np.zeros((n, 0)), q_red=np.eye(n), skeleton=choice.skeleton,
                                  rank=0, frame=np.zeros((0, 0)))
    z = choice.t if row_weight is None else np.asarray(row_weight, dtype=np.float64) @ choice.t
    qfull, frame = basis_qr.complete_qr_host([z])[0]
    k = choice.rank
    return BasisDecomposition(q_skel=qfull[:, n - k:], q_red=qfull[:, :n - k], skeleton=choice.skeleton,
                              rank=k, frame=frame)


# --------------------------------------------------------------------------- flop model

def flop_count(kind, dims):
    """Leading-order flops (dense_core.py:166-181): cholesky n^3/3,
    tri_solve n^2 m, multiply 2 m n k."""
    if kind == "cholesky":
        return dims[0] ** 3 // 3
    if kind == "tri_solve":
        return dims[0] * dims[0] * dims[1]
    if kind == "multiply":
        return 2 * dims[0] * dims[1] * dims[2]
    if kind == "diag_fill":
        return 0
    raise ValueError(f"unknown op kind '{kind}'")


def _pad4(x):
    return 0 if x <= 0 else max(4, -(-x // 4) * 4)


class PhaseFlops:
    """The reference's per-(level, phase) record: true flops, flops of the
    dims padded to the per-kind maximum rounded to 4, and the op count
    (plan_batches + _record, dense_core.py:229-248, ulv_factor.py:135-142)."""

    def __init__(self):
        self.flops = {"levels": {}, "total_true": 0, "total_padded": 0}

    def record(self, level, phase, ops):
        """ops: list of (kind, dims) in the order the reference issues them."""
        by_kind = {}
        for kind, dims in ops:
            by_kind.setdefault(kind, []).append(tuple(int(d) for d in dims))
        true = padded = 0
        for kind, dl in by_kind.items():
            width = len(dl[0])
            mx = tuple(_pad4(max(d[a] for d in dl)) for a in range(width))
            true += sum(flop_count(kind, d) for d in dl)
            padded += flop_count(kind, mx) * len(dl)
        ent = self.flops["levels"].setdefault(level, {}).setdefault(
            phase, {"true": 0, "padded": 0, "count": 0})
        ent["true"] += true
        ent["padded"] += padded
        ent["count"] += len(ops)
        self.flops["total_true"] += true
        self.flops["total_padded"] += padded


# --------------------------------------------------------------------------- single-block API (GPU)
# The reference's dense primitives and batch planner (dense_core.py:51-93,
# 184-284) with the same signatures, errors and results; each call / each
# BatchGroup is one batched launch of the library's kernels (block_engine).

from .block_engine import (BatchGroup, BatchPlan, BlockOp, plan_batches, run_op,  # noqa: E402
                           run_plan, run_sequential)


def cholesky(a, context=None):
    """Lower Cholesky factor on the GPU (dense_core.py:51-66): asymmetry
    beyond 1e-10 relative -> ValueError; a non-positive pivot ->
    NotPositiveDefiniteError(info - 1, *context)."""
    from .block_engine import cholesky_batch

    return cholesky_batch([a], [context])[0]


def tri_solve(l, b, side="left", transposed=False):
    """op(L) X = B (side="left") or X op(L) = B (side="right") on the GPU
    (dense_core.py:69-81); a zero diagonal -> SingularTriangularError."""
    from .block_engine import tri_solve_batch

    return tri_solve_batch([(l, b, side, transposed)])[0]


def multiply(a, b, transpose_a=False, transpose_b=False, accumulate_into=None, scale=1.0):
    """C (+)= scale * op(A) op(B): one grouped DMMA GEMM launch (dense_core.py:84-93)."""
    from .block_engine import multiply_batch

    return multiply_batch([(a, b, transpose_a, transpose_b, accumulate_into, scale)])[0]


def pad_for_cholesky(a, padded_n):
    """Embed a square block top-left in a padded_n square with unit diagonal
    fill (dense_core.py:153-163): the padded factor extends the true one."""
    n = a.shape[0]
    if padded_n < n:
        raise ValueError("padded size smaller than block")
    out = np.zeros((padded_n, padded_n))
    out[:n, :n] = a
    idx = np.arange(n, padded_n)
    out[idx, idx] = 1.0
    return out
