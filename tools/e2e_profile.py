"""Break the end-to-end factorize(h2 host) + solve(b) time of bench.py into its
host/device phases, with the structure cached as in the bench (second and
later calls)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200 import ulv_factor
from paper_2502_02395_b200.h2_device import DeviceH2

c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
hh = bench.host_copy(pkg, h2)
b = np.random.default_rng(1).standard_normal(c["n"])


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


f = pkg.factorize(hh)
x = pkg.solve(f, b)
del f
for rep in range(4):
    t0 = T()
    levels = DeviceH2.layouts_from_host(hh)
    t1 = T()
    dh2, plan = ulv_factor._cached_plan(hh)
    t2 = T()
    plan.run()
    t3 = T()
    plan.check_pivots()
    t4 = T()
    f = ulv_factor.factors_from_plan(hh, plan)
    x = pkg.solve(f, b)
    t5 = T()
    print(f"rep {rep}: layouts {1e3 * (t1 - t0):.1f} ms  cached_plan(upload) {1e3 * (t2 - t1):.1f}  run {1e3 * (t3 - t2):.1f}"
          f"  check {1e3 * (t4 - t3):.1f}  views+solve {1e3 * (t5 - t4):.1f}  total {1e3 * (t5 - t0):.1f}", flush=True)
    del f
