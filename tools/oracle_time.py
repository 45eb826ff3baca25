"""Time the CPU oracle port's factorize on a GPU-built H2 (host copy) at several BLAS thread counts.
Usage: python tools/oracle_time.py m1 [threads...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from threadpoolctl import threadpool_limits

import bench
import paper_2502_02395_b200 as pkg
from oracle import h2ulv_oracle as orc

key = sys.argv[1] if len(sys.argv) > 1 else "m1"
threads = [int(x) for x in sys.argv[2:]] or [1, 8, os.cpu_count()]
c = bench.CONFIGS[key]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
t0 = time.perf_counter()
h2 = pkg.construct(kernel, tree, lists, cfg, cloud, device=torch.device("cuda", 0))
print("construct s", time.perf_counter() - t0, flush=True)
t0 = time.perf_counter()
hh = bench.host_copy(pkg, h2)
print("host copy s", time.perf_counter() - t0, "cores", os.cpu_count(), flush=True)
for th in threads:
    with threadpool_limits(limits=th):
        t0 = time.perf_counter()
        f = orc.factorize(hh)
        dt = time.perf_counter() - t0
    print(f"threads {th}: factorize {dt:.2f} s  {f.flops['total_true'] / dt / 1e9:.1f} GFLOP/s", flush=True)
    for l in sorted(f.levels)[::-1][:3]:
        pass
