"""Host/device phases of the bench's e2e step (factorize(pinned host H2) + solve(b)) at a config."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200 import ulv_factor
from paper_2502_02395_b200.h2_build import to_pinned_host

c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "m1"]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
hh = to_pinned_host(h2)
b = np.random.default_rng(1).standard_normal(c["n"])


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(4):
    t0 = T()
    ok = hh._arena.intact(hh)
    t1 = time.perf_counter()
    f = pkg.factorize(hh)
    t2 = T()
    x = pkg.solve(f, b)
    t3 = T()
    print(f"rep {rep}: intact {1e3 * (t1 - t0):.1f} ms (={ok})  factorize {1e3 * (t2 - t1):.1f} ms  "
          f"solve {1e3 * (t3 - t2):.1f} ms  total {1e3 * (t3 - t0):.1f}", flush=True)
    del f

# raw H2D rate of the same pinned arena: one copy, and the per-region copies alone
arena = hh._arena
dev = torch.empty(arena.tensor.numel(), dtype=arena.tensor.dtype, device="cuda")
for rep in range(2):
    t0 = T()
    dev.copy_(arena.tensor, non_blocking=True)
    t1 = T()
    print(f"one H2D copy of the arena: {arena.tensor.numel() * 8 / 1e9:.2f} GB in {1e3 * (t1 - t0):.1f} ms "
          f"= {arena.tensor.numel() * 8 / (t1 - t0) / 1e9:.1f} GB/s", flush=True)
f = pkg.factorize(hh)
for rep in range(2):
    t0 = T()
    f = pkg.factorize(hh)
    t1 = T()
    print(f"factorize again: {1e3 * (t1 - t0):.1f} ms", flush=True)

# host-side cost of building the factors object (lazy views) after the pivot check
from paper_2502_02395_b200.ulv_factor import factor_plan_of, factors_from_plan  # noqa: E402
del f
f = pkg.factorize(hh)
fp = factor_plan_of(f)
for rep in range(3):
    t0 = time.perf_counter()
    g = factors_from_plan(hh, fp)
    t1 = time.perf_counter()
    print(f"factors_from_plan: {1e3 * (t1 - t0):.2f} ms", flush=True)
    del g
t0 = time.perf_counter()
fp.check_pivots()
print(f"check_pivots (idle GPU): {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
