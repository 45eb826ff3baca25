"""Exact-kernel products, residuals and iterative refinement.

The reference measures accuracy against the dense kernel matrix
(`oracle.dense_assemble` + `matvec_error`, oracle.py:34-64), which it caps at
N = 16384 because it forms A.  `exact_matvec` computes the same product
y = A x on the GPU by direct summation (`h2g_direct_matvec`,
csrc/directsum.cu) without forming A, so ‖A_exact x − b‖ is measurable at the
benchmark sizes (1M-8M).  `refine` is classical iterative refinement of the
ULV solve against any operator (the H² matvec or the exact one).

All products are in the cloud's current (tree) order, like
`oracle.dense_assemble`; `exact_operator` / `h2_operator` wrap them for
vectors in the ORIGINAL input order, the order `solve` takes and returns.
"""

import numpy as np
import torch

from . import _native as nat
from . import kernels
from .errors import CoincidentPointsError

F64 = torch.float64


def _coincident_pair(points):
    """The pair gen_block would report (kernels.py:55-57, row-major first):
    the smallest index i with a coincident partner, and its smallest partner j."""
    pts = np.asarray(points, dtype=np.float64)
    order = np.lexsort(pts.T[::-1])
    srt = pts[order]
    same = np.all(srt[1:] == srt[:-1], axis=1)
    if not same.any():
        return -1, -1
    group = np.concatenate([[0], np.cumsum(~same)])
    counts = np.bincount(group)
    members = order[counts[group] > 1]
    i = int(members.min())
    g = group[np.flatnonzero(order == i)[0]]
    j = int(np.sort(order[group == g])[1])
    return i, j


def exact_matvec(kernel, cloud, x, device=None):
    """y = A x with A the EXACT dense kernel matrix of `cloud` in its current
    (tree) order — A_ij = K(|p_i − p_j|), A_ii = diagonal_shift
    (kernels.gen_block, kernels.py:46-64) — by direct summation on the GPU.
    x: (N,) or (N, m); returns numpy of the same shape.  Coincident distinct
    points raise CoincidentPointsError like kernels.py:55-57."""
    lib = nat.lib()
    n = cloud.count
    xm = np.asarray(x, dtype=np.float64)
    vector = xm.ndim == 1
    if xm.shape[0] != n:
        raise ValueError(f"x has {xm.shape[0]} rows, the cloud {n} points")
    xm = np.ascontiguousarray(xm.reshape(n, -1))
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    with torch.cuda.device(dev):
        pts = torch.from_numpy(np.ascontiguousarray(cloud.points, dtype=np.float64)).to(dev)
        xd = torch.from_numpy(xm).to(dev)
        y = torch.empty_like(xd)
        ws = int(lib.h2g_direct_matvec_workspace(n))
        work = torch.empty(max(ws, 1), dtype=F64, device=dev)
        flag = torch.zeros(1, dtype=torch.int64, device=dev)
        st = torch.cuda.current_stream(dev)
        nat.check(lib.h2g_direct_matvec(pts.data_ptr(), xd.data_ptr(), y.data_ptr(), n, xm.shape[1],
                                        kernels.FAMILY_CODE[kernel.family], float(kernel.diagonal_shift),
                                        float(kernel.device_param), work.data_ptr(), ws, flag.data_ptr(),
                                        st.cuda_stream), "h2g_direct_matvec")
        out = y.cpu().numpy()
        if int(flag.item()):
            raise CoincidentPointsError(*_coincident_pair(np.asarray(cloud.points)))
    return out[:, 0] if vector else out


def _in_original_order(perm, tree_op):
    def op(x):
        x = np.asarray(x, dtype=np.float64)
        y = np.empty_like(x)
        y[perm] = tree_op(x[perm])
        return y
    return op


def exact_operator(kernel, cloud, device=None):
    """x -> A_exact x for vectors in the ORIGINAL input order."""
    return _in_original_order(np.asarray(cloud.perm), lambda xt: exact_matvec(kernel, cloud, xt, device))


def h2_operator(h2):
    """x -> A_H2 x (h2_build.h2_matvec) for vectors in the ORIGINAL input order."""
    from .h2_build import h2_matvec

    return _in_original_order(np.asarray(h2.cloud.perm), lambda xt: h2_matvec(h2, xt))


def relative_residual(op, x, b):
    """‖op(x) − b‖ / ‖b‖ (cli.py:199-205's definition, any operator)."""
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(op(x) - b) / np.linalg.norm(b))


def exact_residual(kernel, cloud, x, b, device=None):
    """‖A_exact x − b‖ / ‖b‖ for x, b in the ORIGINAL input order."""
    return relative_residual(exact_operator(kernel, cloud, device), x, b)


def refine(factors, b, op, iters=2, tol=0.0, mode="parallel", x0=None):
    """Iterative refinement of the ULV solve against the operator `op`
    (original order): x_{k+1} = x_k + solve(factors, b − op(x_k)).  Stops after
    `iters` corrections or once the relative residual is ≤ tol.  Returns
    (x, history) with history[k] = ‖b − op(x_k)‖ / ‖b‖ for every iterate."""
    from .ulv_solve import solve

    b = np.asarray(b, dtype=np.float64)
    nb = float(np.linalg.norm(b))
    if nb == 0.0:
        return np.zeros_like(b), [0.0]
    x = solve(factors, b, mode) if x0 is None else np.array(x0, dtype=np.float64)
    history = []
    for k in range(iters + 1):
        r = b - op(x)
        history.append(float(np.linalg.norm(r) / nb))
        if k == iters or history[-1] <= tol:
            break
        x = x + solve(factors, r, mode)
    return x, history
