"""Lane ablation at one config with ONE construct: for each H2G_ABLATE_LANES set, plan
the factorization again (the ablation is applied when the program is finalized),
capture it and time graph replays with CUDA events.  Results of ablated runs are
wrong by design; only the times matter (critical-path analysis)."""
import os
import sys

sys.path.insert(0, ".")
import torch

import bench
import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200.ulv_factor import FactorPlan

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "m1"
sets = sys.argv[2:] or ["", "4", "2,3", "1", "2,3,4", "1,2,3,4"]
c = bench.CONFIGS[cfg_name]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
torch.cuda.synchronize()
for a in sets:
    os.environ["H2G_ABLATE_LANES"] = a
    plan = FactorPlan(h2._device, lists)
    plan.capture()
    for _ in range(3):
        plan.run()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        plan.run()
    e1.record(st)
    torch.cuda.synchronize()
    print(f"ablate lanes [{a or 'none'}]: {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
    del plan
