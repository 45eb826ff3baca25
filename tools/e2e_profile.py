"""Break down the end-to-end factorize(h2 host) + solve time into its host/device phases."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200.h2_device import DeviceH2
from paper_2502_02395_b200.ulv_factor import FactorPlan, factors_from_plan
import bench
c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
hh = bench.host_copy(pkg, h2)
b = np.random.default_rng(1).standard_normal(c["n"])
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    t0 = T(); dh = DeviceH2.from_host(hh); t1 = T()
    plan = FactorPlan(dh, hh.lists); t2 = T()
    plan.run(); t3 = T()
    plan.check_pivots(); t4 = T()
    f = factors_from_plan(hh, plan); x = pkg.solve(f, b); t5 = T()
    x = pkg.solve(f, b); t6 = T()
    print(f"rep {rep}: upload {1e3*(t1-t0):.1f} ms  plan {1e3*(t2-t1):.1f}  run {1e3*(t3-t2):.1f}  check {1e3*(t4-t3):.1f}  solve(1st, incl plan) {1e3*(t5-t4):.1f}  solve(2nd) {1e3*(t6-t5):.1f}", flush=True)
