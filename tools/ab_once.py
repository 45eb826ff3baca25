"""A/B of plan-time knobs with ONE construct: argv = config, then variants as
NAME=VALUE[,NAME=VALUE...] (or "base"); each variant sets its environment, plans and
captures the factorization, and times graph replays with CUDA events (10 after 3)."""
import os
import sys

sys.path.insert(0, ".")
import torch

import bench
import paper_2502_02395_b200 as pkg
from paper_2502_02395_b200.ulv_factor import FactorPlan

cfg_name = sys.argv[1]
variants = sys.argv[2:] or ["base"]
c = bench.CONFIGS[cfg_name]
kernel, cloud, tree, lists, cfg = bench.build_problem(pkg, c)
h2 = pkg.construct(kernel, tree, lists, cfg, cloud)
torch.cuda.synchronize()
base_env = dict(os.environ)
for rep in range(2):
    for v in variants:
        os.environ.clear()
        os.environ.update(base_env)
        if v != "base":
            for kv in v.split(";"):
                k_, val = kv.split("=", 1)
                os.environ[k_] = val
        # import-time knobs of the planner follow the variant's environment too
        from paper_2502_02395_b200 import program as pm
        pm._TILE32_RATIO = float(os.environ.get("H2G_TILE32_RATIO", "1.5"))
        pm._TILE32_ALL = float(os.environ.get("H2G_TILE32_ALL", "1.5"))
        pm._SPLIT_RATIO = float(os.environ.get("H2G_GEMM_SPLIT", "1.5"))
        pm._SPLITK = int(os.environ.get("H2G_SPLITK", "1"))
        pm._CARVE = os.environ.get("H2G_GEMM_CARVE", "1") != "0"
        pm._BIG_CFG = int(os.environ.get("H2G_BIG_CFG", "2"))
        from paper_2502_02395_b200 import ulv_factor as uf
        uf.CHOL_BOX_MIN = int(os.environ.get("H2G_CHOL_BOX_MIN", "4096"))
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
        print(f"[{v}] {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
        del plan
