"""Time the phases of DeviceH2.from_host (the e2e upload) on a config."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200 import h2_device
from paper_2502_02395_b200.h2_device import DeviceH2

c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
hh = bench.host_copy(pkg, h2)
dh = DeviceH2.from_host(hh)
nbytes = sum(t.numel() * 8 for t in dh.q.values()) + sum(t.numel() * 8 for t in dh.s.values()) + dh.leaf_a.numel() * 8
print("bytes", nbytes)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    DeviceH2.from_host(hh, into=dh)
    t1 = time.perf_counter()
    print(f"from_host {1e3 * (t1 - t0):.1f} ms  ({nbytes / (t1 - t0) / 1e9:.1f} GB/s)", flush=True)
# gather only (no H2D): replicate the task list
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
DeviceH2.from_host(hh, into=dh)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
