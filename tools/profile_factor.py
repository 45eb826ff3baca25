"""Build a config, then run its factorization program N times (for ncu -k/-s/-c capture)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200.ulv_factor import FactorPlan
import bench

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = bench.CONFIGS[cfg_name]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
torch.cuda.synchronize()
plan = FactorPlan(h2._device, lists)
torch.cuda.cudart().cudaProfilerStart()
for _ in range(reps):
    plan.program.run()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", plan.flops["total_true"])
