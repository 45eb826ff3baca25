"""Generate golden fixtures by running the UNMODIFIED reference `h2ulv`
package (read-only, /root/reference/pkg/src) in this container.

Run:  OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py [names...]

Outputs (committed): tests/golden/<name>.npz and tests/golden/<name>.json.
/root/reference does not exist on the GPU box; the fixtures travel instead.

Three kinds of fixture:
  * "h2" fixtures (small N): the reference's full H2Matrix (bases, leaf
    near blocks, couplings, tree, lists) plus the reference's complete
    ULV factors and solution.  A factorization run on the SAME H2 can be
    compared block by block (tests/test_oracle.py, tests/test_gpu_parity.py).
  * "structure" fixtures (C1 / C2 of BASELINE.md): bit-exact tree, lists
    and skeleton indices (arrays for C1, sha256 for C2), per-level dims,
    the reference flop report, the reference residual and (C1) solution.
  * known-answer vectors for the dense primitives (test_dense_core.py).
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import h2ulv  # noqa: E402
from h2ulv import geometry, kernels, h2_build, ulv_factor, ulv_solve  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def tree_arrays(tree):
    rng = []
    for l in range(tree.depth + 1):
        for b in tree.boxes[l]:
            rng.append((l, b.index_in_level, b.begin, b.end))
    centers = np.array([b.center for l in range(tree.depth + 1) for b in tree.boxes[l]])
    radii = np.array([b.radius for l in range(tree.depth + 1) for b in tree.boxes[l]])
    return np.array(rng, dtype=np.int64), centers, radii


def list_arrays(lists):
    near, far = [], []
    for l in range(len(lists.near)):
        for (i, j) in sorted(lists.near[l]):
            near.append((l, i, j))
        for (i, j) in sorted(lists.far[l]):
            far.append((l, i, j))
    return np.array(near, dtype=np.int64).reshape(-1, 3), np.array(far, dtype=np.int64).reshape(-1, 3)


def skeleton_arrays(h2):
    depth = h2.tree.depth
    keys, ranks, local, glob = [], [], [], []
    for l in range(depth, 0, -1):
        for i in range(2 ** l):
            b = h2.bases[(l, i)]
            keys.append((l, i))
            ranks.append(b.rank)
            local.append(b.skeleton)
            glob.append(h2.skeletons[(l, i)])
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64)
    return (np.array(keys, np.int64).reshape(-1, 2), np.array(ranks, np.int64),
            cat(local).astype(np.int64), cat(glob).astype(np.int64))


def flop_table(f):
    out = {"total_true": int(f["total_true"]), "total_padded": int(f["total_padded"]), "levels": {}}
    for l, phases in f["levels"].items():
        out["levels"][str(l)] = {p: {k: int(v) for k, v in e.items()} for p, e in phases.items()}
    return out


def build(shape, n, leaf, family, shift, cfg_kw, seed=0, eta=1.0):
    gen = geometry.gen_sphere_surface if shape == "sphere" else geometry.gen_uniform_cube
    k = kernels.KernelSpec(family=family, diagonal_shift=shift)
    cloud = gen(n, seed=seed)
    t0 = time.perf_counter()
    tree = geometry.build_tree(cloud, leaf)
    lists = geometry.build_interaction_lists(tree, eta)
    cfg = h2_build.BuildConfig(eta=eta, leaf_max=leaf, seed=0, **cfg_kw)
    h2 = h2_build.construct(k, tree, lists, cfg, cloud)
    return k, cloud, tree, lists, cfg, h2, time.perf_counter() - t0


def residual(h2, x, b):
    perm = h2.cloud.perm
    r = h2_build.h2_matvec(h2, x[perm]) - b[perm]
    return float(np.linalg.norm(r) / np.linalg.norm(b))


def config_echo(shape, n, leaf, family, shift, cfg_kw, eta=1.0):
    return {"shape": shape, "n": n, "leaf": leaf, "family": family, "shift": shift,
            "eta": eta, "seed": 0, **cfg_kw}


def make_h2_fixture(name, shape, n, leaf, family, shift, cfg_kw):
    """Full reference H2 + factors + solution for a small problem."""
    k, cloud, tree, lists, cfg, h2, tbuild = build(shape, n, leaf, family, shift, cfg_kw)
    t0 = time.perf_counter()
    f = ulv_factor.factorize(h2)
    tf = time.perf_counter() - t0
    b = np.random.default_rng(1).standard_normal(n)
    x = ulv_solve.solve(f, b)
    xn = ulv_solve.solve(f, b, mode="naive")
    res = residual(h2, x, b)
    arr = {}
    rng_arr, centers, radii = tree_arrays(tree)
    near, far = list_arrays(lists)
    arr.update(points=cloud.points, perm=cloud.perm, box_ranges=rng_arr, centers=centers,
               radii=radii, near=near, far=far, b=b, x=x, x_naive=xn, root=f.root)
    depth = tree.depth
    for l in range(depth, 0, -1):
        for i in range(2 ** l):
            bs = h2.bases[(l, i)]
            arr[f"q_red/{l}/{i}"] = bs.q_red
            arr[f"q_skel/{l}/{i}"] = bs.q_skel
            arr[f"skeleton/{l}/{i}"] = bs.skeleton
    for (l, i, j), blk in h2.near_blocks.items():
        if l == depth:
            arr[f"near/{l}/{i}/{j}"] = blk
    for (l, i, j), blk in h2.couplings.items():
        arr[f"coupling/{l}/{i}/{j}"] = blk
    for l, lvl in f.levels.items():
        for i, v in lvl.lr_diag.items():
            arr[f"f_lr_diag/{l}/{i}"] = v
        for (i, j), v in lvl.lr_off.items():
            arr[f"f_lr_off/{l}/{i}/{j}"] = v
        for (i, j), v in lvl.ls.items():
            arr[f"f_ls/{l}/{i}/{j}"] = v
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arr)
    meta = {"name": name, "config": config_echo(shape, n, leaf, family, shift, cfg_kw),
            "depth": depth, "flops": flop_table(f.flops), "audit": f.audit,
            "residual": res, "factor_seconds": tf, "construct_seconds": tbuild,
            "dims": {str(l): [list(f.levels[l].dims[i]) for i in range(2 ** l)] for l in f.levels}}
    meta.update(versions())
    with open(os.path.join(HERE, name + ".json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(name, "residual", res, "flops", f.flops["total_true"], "build s", round(tbuild, 2))


def versions():
    import scipy
    return {"numpy": np.__version__, "scipy": scipy.__version__,
            "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
            "reference": "h2ulv " + h2ulv.__version__ + " (/root/reference/pkg)"}


def skeleton_sha_per_level(h2):
    """sha256 of each level's concatenated box-local skeletons (to localise a mismatch)."""
    out = {}
    for l in range(h2.tree.depth, 0, -1):
        sk = [h2.bases[(l, i)].skeleton for i in range(2 ** l)]
        out[str(l)] = sha(np.concatenate(sk).astype(np.int64) if sk else np.zeros(0, np.int64),
                          np.array([len(s) for s in sk], np.int64))
    return out


def make_structure_fixture(name, shape, n, leaf, family, shift, cfg_kw, store_arrays):
    k, cloud, tree, lists, cfg, h2, tbuild = build(shape, n, leaf, family, shift, cfg_kw)
    rng_arr, centers, radii = tree_arrays(tree)
    near, far = list_arrays(lists)
    skel_keys, ranks, skel_local, skel_global = skeleton_arrays(h2)
    t0 = time.perf_counter()
    try:
        f = ulv_factor.factorize(h2)
    except h2ulv.errors.NotPositiveDefiniteError as e:
        # the reference's breakdown contract (dense_core.py:60-63): record where it failed
        meta = {"name": name, "config": config_echo(shape, n, leaf, family, shift, cfg_kw),
                "depth": tree.depth,
                "sha": {"perm": sha(cloud.perm), "box_ranges": sha(rng_arr), "near": sha(near),
                        "far": sha(far), "ranks": sha(ranks), "skeleton_local": sha(skel_local),
                        "skeleton_global": sha(skel_global)},
                "skeleton_sha_per_level": skeleton_sha_per_level(h2),
                "npd": {"pivot": int(e.pivot), "level": int(e.level), "box": int(e.box)},
                "factor_seconds": time.perf_counter() - t0, "construct_seconds": tbuild}
        meta.update(versions())
        with open(os.path.join(HERE, name + ".json"), "w") as fh:
            json.dump(meta, fh, indent=1)
        print(name, "NPD", meta["npd"], "build s", round(tbuild, 2))
        return
    tf = time.perf_counter() - t0
    b = np.random.default_rng(1).standard_normal(n)
    t0 = time.perf_counter()
    x = ulv_solve.solve(f, b)
    ts = time.perf_counter() - t0
    res = residual(h2, x, b)
    meta = {"name": name, "config": config_echo(shape, n, leaf, family, shift, cfg_kw),
            "depth": tree.depth,
            "sha": {"perm": sha(cloud.perm), "points": sha(cloud.points),
                    "box_ranges": sha(rng_arr), "near": sha(near), "far": sha(far),
                    "ranks": sha(ranks), "skeleton_local": sha(skel_local),
                    "skeleton_global": sha(skel_global)},
            "skeleton_sha_per_level": skeleton_sha_per_level(h2),
            "counts": {"near": int(len(near)), "far": int(len(far)), "skeleton": int(len(skel_local))},
            "flops": flop_table(f.flops), "audit": f.audit, "residual": res,
            "factor_seconds": tf, "solve_seconds": ts, "construct_seconds": tbuild,
            "root_dim": int(f.root.shape[0]),
            "root_diag_sha": sha(np.diag(f.root)),
            "x_norm": float(np.linalg.norm(x)),
            "dims": {str(l): [list(f.levels[l].dims[i]) for i in range(2 ** l)] for l in f.levels}}
    meta.update(versions())
    with open(os.path.join(HERE, name + ".json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    if store_arrays:
        np.savez_compressed(os.path.join(HERE, name + ".npz"), perm=cloud.perm, box_ranges=rng_arr,
                            near=near, far=far, skel_keys=skel_keys, ranks=ranks,
                            skel_local=skel_local, skel_global=skel_global, b=b, x=x,
                            root_diag=np.diag(f.root).copy())
    print(name, "residual", res, "flops", f.flops["total_true"], "factor s", round(tf, 2),
          "build s", round(tbuild, 2))


def make_known_answers():
    from h2ulv import dense_core
    rng = np.random.default_rng(0)
    out = {}
    a = np.array([[4.0, 2.0], [2.0, 3.0]])
    out["chol2_a"] = a
    out["chol2_l"] = dense_core.cholesky(a)
    g = rng.standard_normal((12, 12))
    out["chol12_a"] = g @ g.T + 12 * np.eye(12)
    out["chol12_l"] = dense_core.cholesky(out["chol12_a"])
    # id_basis on a random sample matrix, with and without row_weight
    s = rng.standard_normal((40, 60))
    s[:, :] = s @ np.diag(np.logspace(0, -12, 60))
    bd = dense_core.id_basis(s, tol=1e-6)
    out.update(id_s=s, id_skel=bd.skeleton, id_qskel=bd.q_skel, id_frame=bd.frame, id_qred=bd.q_red)
    w = np.linalg.qr(rng.standard_normal((40, 40)))[0] * 3.0
    bw = dense_core.id_basis(s, tol=1e-6, row_weight=w)
    out.update(idw_w=w, idw_skel=bw.skeleton, idw_qskel=bw.q_skel, idw_frame=bw.frame)
    np.savez_compressed(os.path.join(HERE, "known_answers.npz"), **out)
    print("known answers written")


FIXTURES = {
    "known": make_known_answers,
    "h2_cube512_rank16": lambda: make_h2_fixture("h2_cube512_rank16", "cube", 512, 64, "laplace", 1e3, {"rank": 16}),
    "h2_sphere1024_yukawa_tol": lambda: make_h2_fixture("h2_sphere1024_yukawa_tol", "sphere", 1024, 64, "yukawa", 1e3, {"tol": 1e-5}),
    "h2_cube1024_sampled": lambda: make_h2_fixture("h2_cube1024_sampled", "cube", 1024, 32, "laplace", 1e4,
                                                   {"tol": 1e-6, "s_far": 64, "s_near": 64}),
    "c1": lambda: make_structure_fixture("c1", "cube", 4096, 256, "laplace", 1e3, {"tol": 1e-8}, True),
    "c2": lambda: make_structure_fixture("c2", "cube", 65536, 256, "laplace", 1e5,
                                         {"tol": 1e-8, "s_far": 512, "s_near": 512}, False),
    # BASELINE.json configs[2] (C3) and the metric configuration (M1, N = 2^20) + its tolerance sweep (C5, P = 1)
    "c3": lambda: make_structure_fixture("c3", "sphere", 262144, 256, "yukawa", 1e5,
                                         {"tol": 1e-8, "s_far": 512, "s_near": 512}, False),
    "m1": lambda: make_structure_fixture("m1", "cube", 1048576, 256, "laplace", 2e6,
                                         {"tol": 1e-8, "s_far": 512, "s_near": 512}, False),
    "m1_tol6": lambda: make_structure_fixture("m1_tol6", "cube", 1048576, 256, "laplace", 2e6,
                                              {"tol": 1e-6, "s_far": 512, "s_near": 512}, False),
    "m1_tol10": lambda: make_structure_fixture("m1_tol10", "cube", 1048576, 256, "laplace", 2e6,
                                               {"tol": 1e-10, "s_far": 512, "s_near": 512}, False),
    # BASELINE.md §3 breakdown edges: the reference raises NotPositiveDefiniteError(pivot, level, box)
    "c2_npd": lambda: make_structure_fixture("c2_npd", "cube", 65536, 256, "laplace", 1e3,
                                             {"tol": 1e-8, "s_far": 512, "s_near": 512}, False),
    "sphere65k_npd": lambda: make_structure_fixture("sphere65k_npd", "sphere", 65536, 256, "yukawa", 1e3,
                                                    {"tol": 1e-8, "s_far": 512, "s_near": 512}, False),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(FIXTURES)
    for nm in names:
        FIXTURES[nm]()
