"""Per-step device times of the solve's prepare program (once per factorization) at a config."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200 import _native as nat
from paper_2502_02395_b200.ulv_solve import _plan_for

c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "m1"]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
f = pkg.factorize(h2)
sp = _plan_for(f, 1, "parallel")
names = {v: k for k, v in nat.STEP.items()}
for rep in range(3):
    ms = sp.prepare.run_timed()
torch.cuda.synchronize()
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    e0.record(st)
    sp.prepare.launch(st)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"prepare graph: {e0.elapsed_time(e1):.3f} ms", flush=True)
steps = sp.prepare.steps
tot = float(ms.sum())
print(f"serialized steps: {tot:.3f} ms")
order = np.argsort(-ms)
for q in order[:15]:
    print(f"  step {q:3d} {names[int(steps[q]['kind'])]:10s} lane {int(steps[q]['lane'])} grid {int(steps[q]['grid']):6d} {ms[q]:.3f} ms")
