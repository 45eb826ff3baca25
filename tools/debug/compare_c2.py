"""Debug: GPU construct/factorize vs CPU oracle on a mid-size sampled problem."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2502_02395_b200 as pkg
from oracle import h2ulv_oracle as orc
import bench

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
c = dict(shape="cube", n=N, leaf=256, family="laplace", shift=1e5, tol=1e-8, s_far=512, s_near=512)
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
hh = bench.host_copy(pkg, h2)
FULL = "--full" in sys.argv
depth = tree.depth
def rel(a, b):
    nb = np.linalg.norm(b); return np.linalg.norm(a - b) / (nb if nb else 1)
if FULL:
    cloud2 = pkg.gen_uniform_cube(N, 0)
    tree2 = pkg.build_tree(cloud2, 256)
    lists2 = pkg.build_interaction_lists(tree2, 1.0)
    ho = orc.construct(kernel, tree2, lists2, cfg, cloud2)
for l in (range(depth, 0, -1) if FULL else []):
    eq = max(rel(hh.bases[(l, i)].q_skel, ho.bases[(l, i)].q_skel) for i in range(2 ** l))
    eqr = max(rel(hh.bases[(l, i)].q_red, ho.bases[(l, i)].q_red) for i in range(2 ** l))
    ef = max(rel(hh.bases[(l, i)].frame, ho.bases[(l, i)].frame) for i in range(2 ** l))
    ec = max([rel(hh.couplings[key], ho.couplings[key]) for key in ho.couplings if key[0] == l] or [0])
    print(f"construct L{l}: q_skel {eq:.2e} q_red {eqr:.2e} frame {ef:.2e} coupling {ec:.2e}")
if FULL:
    en = max(rel(hh.near_blocks[key], ho.near_blocks[key]) for key in ho.near_blocks)
    print("near blocks", en)
b = np.random.default_rng(1).standard_normal(N)
of = orc.factorize(hh)
xo = orc.solve(of, b)
print("oracle on GPU-built H2: residual", orc.residual(hh, xo, b))
if FULL:
    of2 = orc.factorize(ho)
    print("oracle on CPU-built H2: residual", orc.residual(ho, orc.solve(of2, b), b))
from paper_2502_02395_b200.h2_build import h2_matvec
fg = pkg.factorize(h2)
xg = pkg.solve(fg, b)
perm = cloud.perm
print("GPU on device H2: residual(product matvec)", np.linalg.norm(h2_matvec(h2, xg[perm]) - b[perm]) / np.linalg.norm(b),
      "oracle residual", orc.residual(hh, xg, b))
f = pkg.factorize(hh)
x = pkg.solve(f, b)
print("GPU factor on host copy: residual", orc.residual(hh, x, b), "rel err vs oracle x", rel(x, xo))
for l in range(depth, 0, -1):
    lv = f.levels[l]; ol = of.levels[l]
    e1 = max(rel(lv.lr_diag[i], ol["lr_diag"][i]) for i in ol["lr_diag"])
    e2 = max([rel(lv.lr_off[k], ol["lr_off"][k]) for k in ol["lr_off"]] or [0])
    e3 = max(rel(lv.ls[k], ol["ls"][k]) for k in ol["ls"])
    e4 = max(rel(lv.v[i], ol["v"][i]) for i in ol["v"])
    print(f"factor L{l}: lr_diag {e1:.2e} lr_off {e2:.2e} ls {e3:.2e} v {e4:.2e} r={list(lv.dims.values())[:3]}")
print("root", rel(f.root, of.root))
