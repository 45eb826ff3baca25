"""One small factorization + solve run EAGERLY (no CUDA graph) for compute-sanitizer:
  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_factor.py [box]
C1-sized problem (N = 4096, 16 leaves: the one-launch fused panel step with its
ticket / flag synchronisation runs at every level); with `box` the fused per-box
Cholesky (h2g_chol_box) is forced on every level; with `wy` the compact-WY path is
forced on every level (construct's Yt / q_full rebuild, the EXT GEMMs of the transform)
and a pinned-host copy is factorized through the compact upload, plus one split-K launch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200 import ulv_factor
from paper_2502_02395_b200.program import Program
from paper_2502_02395_b200.ulv_solve import SolvePlan

if "box" in sys.argv[1:]:
    ulv_factor.CHOL_BOX_MIN = 1
WY = "wy" in sys.argv[1:]
if WY:
    from paper_2502_02395_b200 import basis_qr, program as pm
    basis_qr.WY_RATIO, basis_qr.WY_MIN_N = 100.0, 0.0
    pm._SPLITK = 8
cloud = pkg.gen_uniform_cube(4096, seed=0)
tree = pkg.build_tree(cloud, 256)
lists = pkg.build_interaction_lists(tree, 1.0)
cfg = pkg.BuildConfig(eta=1.0, leaf_max=256, tol=1e-8, s_far=256, s_near=256)
h2 = pkg.construct(pkg.KernelSpec(family="laplace", diagonal_shift=1e3), tree, lists, cfg, cloud)
if WY:
    assert h2._device.wy, "compact-WY levels expected"
plan = ulv_factor.FactorPlan(h2._device, lists)
for _ in range(2):                       # twice: the sync words must be left clean
    for seg in plan.segments:
        seg.run()
torch.cuda.synchronize()
plan.check_pivots()
f = ulv_factor.factors_from_plan(h2, plan)
sp = SolvePlan(plan, 1, "parallel")
b = np.random.default_rng(1).standard_normal(cloud.count)
sp.xin[:cloud.count].copy_(torch.from_numpy(b[cloud.perm]))
sp.prepare.run()
for seg in sp.fwd_segments + sp.bwd_segments:
    if isinstance(seg, Program):
        seg.run()
torch.cuda.synchronize()
x = np.empty_like(b)
x[cloud.perm] = sp.output[:cloud.count].cpu().numpy()
from oracle import h2ulv_oracle as orc  # noqa: E402  (checker only)
print("residual", orc.residual(h2, x, b))
# the other solve paths: w = 3 (the 4-column GEMV kernel), naive mode, and the exact-kernel direct sum
for w, mode in ((3, "parallel"), (1, "naive")):
    spw = SolvePlan(plan, w, mode)
    bw = np.random.default_rng(2).standard_normal((cloud.count, w))
    spw.xin[:cloud.count * w].copy_(torch.from_numpy(bw[cloud.perm].reshape(-1)))
    spw.prepare.run()
    for seg in spw.fwd_segments + spw.bwd_segments:
        if isinstance(seg, Program):
            seg.run()
    torch.cuda.synchronize()
    xw = np.empty_like(bw)
    xw[cloud.perm] = spw.output[:cloud.count * w].view(-1, w).cpu().numpy()
    print(mode, w, "residual", max(orc.residual(h2, xw[:, j], bw[:, j]) for j in range(w)))
from paper_2502_02395_b200.direct_sum import exact_residual  # noqa: E402
print("exact residual", exact_residual(h2.kernel, cloud, x, b))
if WY:   # the compact upload of a pinned-host copy (q_full rebuilt on the device), eager
    from paper_2502_02395_b200.h2_build import to_pinned_host
    from paper_2502_02395_b200.h2_device import DeviceH2
    hh = to_pinned_host(h2)
    up = DeviceH2.from_host(hh)
    torch.cuda.synchronize()
    print("compact upload q_full equal:", all(bool(torch.equal(up.q[l], h2._device.q[l])) for l in up.wy))
