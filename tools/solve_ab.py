"""A/B of solve variants on one factorization: python tools/solve_ab.py [config]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200 import ulv_solve as us
from paper_2502_02395_b200.program import Program

key = sys.argv[1] if len(sys.argv) > 1 else "m1"
c = bench.CONFIGS[key]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
f = pkg.factorize(h2)
b = np.random.default_rng(1).standard_normal(c["n"])
stream = torch.cuda.current_stream()
xs = {}
for flag in (False, True, False, True):
    us._XFORM_T = flag
    sp = us.SolvePlan(f.device, 1, "parallel")
    for seg in sp.fwd_segments + sp.bwd_segments:
        if isinstance(seg, Program):
            seg.capture()
    sp.xin[:c["n"]].copy_(torch.from_numpy(b))
    for _ in range(3):
        sp.run_forward(stream)
        sp.run_backward(stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(20):
        sp.run_forward(stream)
        sp.run_backward(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    xs[flag] = sp.output[:c["n"]].cpu().numpy()
    print(f"xform_t={flag}: solve {e0.elapsed_time(e1) / 20:.3f} ms", flush=True)
print("rel diff", np.linalg.norm(xs[True] - xs[False]) / np.linalg.norm(xs[False]))
