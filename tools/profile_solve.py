"""Build a config, factor it, then run ONE solve inside a cudaProfilerStart/Stop
range (for `ncu --profile-from-start off` launch lists of the substitution)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import paper_2502_02395_b200 as pkg

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = bench.CONFIGS[cfg_name]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
f = pkg.factorize(h2)
b = np.random.default_rng(1).standard_normal(c["n"])
x = pkg.solve(f, b)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    x = pkg.solve(f, b)
    torch.cuda.synchronize()
    print(f"solve wall {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
torch.cuda.cudart().cudaProfilerStart()
x = pkg.solve(f, b)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
