"""Critical-path ablation in ONE process: build the H2 once, then time the
factorization graph with the steps of some lanes turned into NOPs
(H2G_ABLATE_LANES, read when a Program is finalized).  Results of ablated
runs are numerically invalid; only the time matters.
Usage: python tools/ablate.py [config] [steps]"""
import json
import os
import sys

sys.path.insert(0, ".")
import torch

import bench
import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200.ulv_factor import FactorPlan

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
c = bench.CONFIGS[cfg_name]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
torch.cuda.synchronize()
out = {}
for lanes in ["", "1", "2", "3", "4", "3,4", "2,3,4", "1,2,3,4"]:
    os.environ["H2G_ABLATE_LANES"] = lanes
    plan = FactorPlan(h2._device, lists)
    plan.capture()
    for _ in range(3):
        plan.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        plan.run()
    e1.record()
    torch.cuda.synchronize()
    out[lanes or "none"] = e0.elapsed_time(e1) / steps
    print(f"ablate [{lanes}] {out[lanes or 'none']:.3f} ms", flush=True)
    del plan
print(json.dumps({"config": cfg_name, "ms_by_ablated_lanes": out}))
