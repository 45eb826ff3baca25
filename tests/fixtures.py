"""Load the golden fixtures (tests/golden/*.npz|json) into the package's types.

The fixtures were produced by the UNMODIFIED reference (tests/golden/make_golden.py);
an "h2" fixture holds the reference's own H2Matrix, so a factorization of it
can be compared with the reference's factors block by block.
"""
import json
import os

import numpy as np

from paper_2502_02395_b200.dense_core import BasisDecomposition
from paper_2502_02395_b200.geometry import Box, ClusterTree, InteractionLists, PointCloud
from paper_2502_02395_b200.h2_build import BuildConfig, H2Matrix
from paper_2502_02395_b200.kernels import KernelSpec

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def meta(name):
    with open(os.path.join(GOLDEN, name + ".json")) as fh:
        return json.load(fh)


def arrays(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def tree_from(z, leaf_max):
    rng, centers, radii = z["box_ranges"], z["centers"], z["radii"]
    depth = int(rng[:, 0].max())
    boxes = [[] for _ in range(depth + 1)]
    for (l, i, b, e), c, r in zip(rng, centers, radii):
        boxes[int(l)].append(Box(level=int(l), index_in_level=int(i), begin=int(b), end=int(e), center=c,
                                 radius=float(r)))
    return ClusterTree(depth=depth, boxes=boxes, leaf_max=leaf_max)


def lists_from(z, depth):
    near = [set() for _ in range(depth + 1)]
    far = [set() for _ in range(depth + 1)]
    for l, i, j in z["near"]:
        near[int(l)].add((int(i), int(j)))
    for l, i, j in z["far"]:
        far[int(l)].add((int(i), int(j)))
    return InteractionLists(near=near, far=far)


def load_h2(name):
    """The reference's H2Matrix of an h2 fixture, as host numpy blocks."""
    m, z = meta(name), arrays(name)
    cfg = m["config"]
    kw = {key: cfg[key] for key in ("rank", "tol", "s_far", "s_near") if key in cfg}
    tree = tree_from(z, cfg["leaf"])
    depth = tree.depth
    lists = lists_from(z, depth)
    cloud = PointCloud(points=z["points"], perm=z["perm"])
    kernel = KernelSpec(family=cfg["family"], diagonal_shift=cfg["shift"])
    h2 = H2Matrix(tree=tree, lists=lists, kernel=kernel, cloud=cloud,
                  config=BuildConfig(eta=cfg["eta"], leaf_max=cfg["leaf"], **kw))
    bases, near, cpl = {}, {}, {}
    for key in z.files:
        parts = key.split("/")
        if parts[0] == "q_red":
            l, i = int(parts[1]), int(parts[2])
            qs = z[f"q_skel/{l}/{i}"]
            bases[(l, i)] = BasisDecomposition(q_skel=qs, q_red=z[key], skeleton=z[f"skeleton/{l}/{i}"],
                                               rank=qs.shape[1], frame=None)
        elif parts[0] == "near" and len(parts) == 4:
            near[tuple(int(p) for p in parts[1:])] = z[key]
        elif parts[0] == "coupling" and len(parts) == 4:
            cpl[tuple(int(p) for p in parts[1:])] = z[key]
    h2.bases, h2.near_blocks, h2.couplings = bases, near, cpl
    return h2


def reference_factors(name):
    """{'lr_diag': {(l, i): ...}, 'lr_off': {(l, i, j): ...}, 'ls': {...}, 'root': ..., 'x': ...}."""
    z = arrays(name)
    out = {"lr_diag": {}, "lr_off": {}, "ls": {}}
    for key in z.files:
        parts = key.split("/")
        if parts[0] == "f_lr_diag":
            out["lr_diag"][(int(parts[1]), int(parts[2]))] = z[key]
        elif parts[0] == "f_lr_off":
            out["lr_off"][tuple(int(p) for p in parts[1:])] = z[key]
        elif parts[0] == "f_ls":
            out["ls"][tuple(int(p) for p in parts[1:])] = z[key]
    out["root"], out["x"], out["x_naive"], out["b"] = z["root"], z["x"], z["x_naive"], z["b"]
    return out


H2_FIXTURES = ["h2_cube512_rank16", "h2_sphere1024_yukawa_tol", "h2_cube1024_sampled"]


def flops_equal(ours, golden):
    """Compare a flop dict with the JSON-serialised reference one."""
    if ours["total_true"] != golden["total_true"] or ours["total_padded"] != golden["total_padded"]:
        return False
    for l, phases in golden["levels"].items():
        mine = ours["levels"][int(l)]
        for ph, ent in phases.items():
            if {k: int(v) for k, v in mine[ph].items()} != ent:
                return False
    return len(ours["levels"]) == len(golden["levels"])
