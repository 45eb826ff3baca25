"""Host/device split of solve(f, b) at a config: each step of _solve_on timed with syncs."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200.h2_build import to_pinned_host
from paper_2502_02395_b200.ulv_solve import _plan_for

c = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "m1"]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
hh = to_pinned_host(h2)
del h2
b = np.random.default_rng(1).standard_normal(c["n"])
for rep in range(3):
    f = pkg.factorize(hh)
    x = pkg.solve(f, b)
    del f
f = pkg.factorize(hh)
torch.cuda.synchronize()


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(4):
    t0 = T()
    sp = _plan_for(f, 1, "parallel")
    t1 = T()
    dev = sp.device
    perm = hh.cloud._perm_dev[1]
    b_dev = torch.from_numpy(np.ascontiguousarray(b.reshape(-1, 1))).to(dev)
    t2 = T()
    sp.xin.view(-1, 1)[:hh.count] = b_dev.index_select(0, perm)
    t3 = T()
    sp.run_forward()
    t4 = T()
    sp.run_backward()
    t5 = T()
    x_dev = torch.empty_like(b_dev)
    x_dev[perm] = sp.output.view(-1, 1)[:hh.count]
    t6 = T()
    xx = x_dev.cpu().numpy()
    t7 = T()
    t8 = time.perf_counter()
    pkg.solve(f, b)
    t9 = T()
    print(f"plan {1e3*(t1-t0):.2f}  b H2D {1e3*(t2-t1):.2f}  perm {1e3*(t3-t2):.2f}  fwd {1e3*(t4-t3):.2f}  "
          f"bwd {1e3*(t5-t4):.2f}  scatter {1e3*(t6-t5):.2f}  x D2H {1e3*(t7-t6):.2f}  | solve() {1e3*(t9-t8):.2f} ms",
          flush=True)
