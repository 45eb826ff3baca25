"""H²-ULV factorization benchmark (BASELINE.json metric) — one JSON line.

A "step" is one complete H²-ULV factorization (all levels + root) of the
configuration named by `--config` (default C2 = BASELINE.json configs[1]:
Laplace-3D, N = 65536 uniform-cube points, leaf 256, tol 1e-8, shift 1e5,
512/512 sampling).  The H² matrix is built once (untimed; construction is
not part of the reference metric).

  value         factorization GFLOP/s = reference flop model total_true
                (dense_core.flop_count) / device time, operands resident in
                HBM, whole program replayed as one CUDA graph
  e2e           the same metric through the public API with HOST buffers:
                factorize(h2 of numpy blocks) + solve(b) -> x on the host,
                all host<->device copies inside the timed region (the upload
                streams level by level and overlaps the factorization)
  roofline      dominant kernel = grouped FP64 DMMA GEMM; achieved flops over
                its CUDA-event time inside an instrumented pass of K steps
  cpu_baseline  the CPU oracle port (oracle/h2ulv_oracle.py) on the host cores

Multi-GPU (`torchrun ... bench.py --gpus N`): ONE factorization sharded over
the ranks (distributed.py: boxes of the levels >= log2 N split by contiguous
leaf ranges, NCCL all_gather of halo / boundary blocks, top levels replicated);
strong scaling, time = max over ranks.
`--impl reference` times the CPU oracle port (the reference is pure Python and
does not travel to the GPU box) on rank 0 only.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H²-ULV factorization time (s) and GFLOP/s at N=1M, 1/2/4/8 B200; solve residual"
FP64_PEAK_TFLOPS = 37.1   # measured DMMA issue peak, profiles/r01_fp64_peak.txt (no FP64 entry in MEASURED_PEAKS.json)

CONFIGS = {
    "c1": dict(shape="cube", n=4096, leaf=256, family="laplace", shift=1e3, tol=1e-8, s_far=0, s_near=0),
    "c2": dict(shape="cube", n=65536, leaf=256, family="laplace", shift=1e5, tol=1e-8, s_far=512, s_near=512),
    "c3": dict(shape="sphere", n=262144, leaf=256, family="yukawa", shift=1e5, tol=1e-8, s_far=512, s_near=512),
    "m1": dict(shape="cube", n=1048576, leaf=256, family="laplace", shift=2e6, tol=1e-8, s_far=512, s_near=512),
}


def workload_name(key, c):
    return (f"{key.upper()}: {c['family']} {c['shape']} N={c['n']} leaf={c['leaf']} tol={c['tol']:g} "
            f"shift={c['shift']:g} s_far/s_near={c['s_far']}/{c['s_near']}")


def build_problem(pkg, c, on_gpu=True):
    gen = pkg.gen_uniform_cube if c["shape"] == "cube" else pkg.gen_sphere_surface
    cloud = gen(c["n"], seed=0)
    tree = pkg.build_tree(cloud, c["leaf"])
    lists = pkg.build_interaction_lists(tree, 1.0)
    cfg = pkg.BuildConfig(eta=1.0, leaf_max=c["leaf"], tol=c["tol"], s_far=c["s_far"], s_near=c["s_near"], seed=0)
    kernel = pkg.KernelSpec(family=c["family"], diagonal_shift=c["shift"])
    return kernel, cloud, tree, lists, cfg


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def host_copy(pkg, h2):
    """numpy-only H2Matrix (the reference's data model) of a GPU-built one."""
    from paper_2502_02395_b200.h2_build import H2Matrix

    hh = H2Matrix(tree=h2.tree, lists=h2.lists, kernel=h2.kernel, cloud=h2.cloud, config=h2.config)
    hh.bases = {key: h2.bases[key] for key in h2.bases}
    depth = h2.tree.depth
    hh.near_blocks = {key: h2.near_blocks[key] for key in h2.near_blocks if key[0] == depth}
    hh.couplings = {key: h2.couplings[key] for key in h2.couplings}
    hh.skeletons, hh.eff_points = h2.skeletons, h2.eff_points
    return hh


def h2d_bytes(h2):
    depth = h2.tree.depth
    nb = sum(b.q_red.nbytes + b.q_skel.nbytes for b in h2.bases.values())
    nb += sum(v.nbytes for k, v in h2.near_blocks.items() if k[0] == depth)
    nb += sum(v.nbytes for v in h2.couplings.values())
    return nb


def cpu_oracle_time(h2_host, threads):
    from threadpoolctl import threadpool_limits

    from oracle import h2ulv_oracle as orc

    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        f = orc.factorize(h2_host)
        dt = time.perf_counter() - t0
    return dt, f.flops["total_true"]


def run_reference(args, c, key):
    """--impl reference: the CPU oracle port on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2502_02395_b200 as pkg
    from threadpoolctl import threadpool_limits

    from oracle import h2ulv_oracle as orc

    kernel, cloud, tree, lists, cfg = build_problem(pkg, c)
    h2 = orc.construct(kernel, tree, lists, cfg, cloud)
    cores = os.cpu_count()
    threads = sorted({1, min(8, cores), cores})
    best = None
    for th in threads:  # nproc and 1 BLAS thread (and 8), keep the fastest
        with threadpool_limits(limits=th):
            t0 = time.perf_counter()
            orc.factorize(h2)
            dt = time.perf_counter() - t0
        if best is None or dt < best[0]:
            best = (dt, th)
    th = best[1]
    times = []
    with threadpool_limits(limits=th):
        for s in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            f = orc.factorize(h2)
            dt = time.perf_counter() - t0
            if s >= args.warmup:
                times.append(dt)
    flops = f.flops["total_true"]
    ms = 1e3 * float(np.mean(times))
    val = flops / (ms * 1e-3) / 1e9
    b = np.random.default_rng(1).standard_normal(c["n"])
    res = orc.residual(h2, orc.solve(f, b), b)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (uniform cube, seed 0)",
            "config": {"workload": workload_name(key, c), "flops_per_step": flops, "residual": res},
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": th, "kind": "port",
                             "sample": f"full factorization of {key.upper()} per step (oracle/h2ulv_oracle.py, "
                                       f"OpenBLAS threads={th}, host has {cores} cores)"},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    c = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, c, args.config)

    import torch
    import torch.distributed as dist

    import paper_2502_02395_b200 as pkg
    from paper_2502_02395_b200 import _native as nat
    from paper_2502_02395_b200.h2_build import h2_matvec
    from paper_2502_02395_b200.ulv_factor import FactorPlan, factors_from_plan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("BENCH_SHARE_GPU"):   # test mode: all ranks on GPU 0 (gloo)
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    backend = os.environ.get("BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    kernel, cloud, tree, lists, cfg = build_problem(pkg, c)
    t0 = time.perf_counter()
    h2 = pkg.construct(kernel, tree, lists, cfg, cloud, device=dev)
    construct_s = time.perf_counter() - t0

    comm = part = None
    if world > 1:
        from paper_2502_02395_b200.distributed import Comm, Partition

        comm = Comm.from_env()
        part = Partition(world, tree.depth)
    plan = FactorPlan(h2._device, lists, part=part, comm=comm)
    plan.capture()
    progs = [sg for sg in plan.segments if not isinstance(sg, tuple)]
    flops = plan.flops["total_true"]
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        plan.run(stream)
    torch.cuda.synchronize(dev)
    ablating = bool(os.environ.get("H2G_ABLATE_LANES"))   # critical-path analysis: results invalid
    if not ablating:
        plan.check_pivots()

    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        plan.run(stream)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    if ablating:
        print(json.dumps({"ablated_lanes": os.environ["H2G_ABLATE_LANES"], "ms_per_step": ms}), flush=True)
        return
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # one matrix per step: replicas would multiply by world; the sharded factorization
    # splits ONE factorization over the ranks (strong scaling)
    value = flops / (ms * 1e-3) / 1e9

    # ---- roofline: per-step CUDA events over K instrumented (eager) factorizations
    per_kind = {}
    work = [w for pg in progs for w in pg.work]
    exec_fl = [x for pg in progs for x in pg.exec_flops]
    steps_arr = np.concatenate([pg.steps for pg in progs])
    step_ms = np.zeros(len(steps_arr))
    for _ in range(args.steps):
        parts = []
        for sg in plan.segments:
            if isinstance(sg, tuple):
                from paper_2502_02395_b200.distributed import run_exchange

                run_exchange(plan, sg)
            else:
                parts.append(sg.run_timed(stream))
        step_ms += np.concatenate(parts)
    step_ms /= args.steps
    gemm_kinds = {nat.STEP[k] for k in ("GEMM_NN", "GEMM_NT", "GEMM_TN", "GEMM_TT")}
    names = {v: k for k, v in nat.STEP.items()}
    g_fl = g_ms = 0.0
    for (kind, fl, by), t in zip(work, step_ms):
        nm = "GEMM" if kind in gemm_kinds else names[kind]
        d = per_kind.setdefault(nm, {"ms": 0.0, "launches": 0, "flops": 0, "bytes": 0})
        d["ms"] += float(t)
        d["launches"] += 1
        d["flops"] += int(fl)
        d["bytes"] += int(by)
        if kind in gemm_kinds:
            g_fl += fl
            g_ms += t
    eager_ms = float(step_ms.sum())
    if os.environ.get("BENCH_DUMP"):
        with open(os.environ["BENCH_DUMP"], "w") as fh:
            json.dump([{"kind": names[int(kd)], "flops": int(fl), "exec_flops": int(ex), "bytes": int(by),
                        "ms": float(t), "count": int(st["count"]), "grid": int(st["grid"]), "lane": int(st["lane"])}
                       for (kd, fl, by), ex, t, st in zip(work, exec_fl, step_ms, steps_arr)], fh)
    achieved = g_fl / (g_ms * 1e-3) / 1e12 if g_ms > 0 else 0.0
    traffic = traffic_note = None
    tfile = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tfile):
        with open(tfile) as fh:
            tr = json.load(fh).get(args.config)
        if tr:
            traffic = tr["bytes"]
            traffic_note = (f"{tr['launch']}; algorithmic bytes of that launch {tr['algorithmic_bytes']} "
                            f"({tr['source']})")
    roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic, "traffic_note": traffic_note,
                "kernel": "gemm_grouped_kernel (FP64 DMMA.8x8x4)",
                "peak_source": "measured FP64 DMMA issue peak (profiles/r01_fp64_peak.txt); "
                               "cuBLAS DGEMM 8192^3 = 35.5 TFLOP/s",
                "gemm_share_of_step": g_ms / eager_ms if eager_ms else None,
                "per_kind": {k: {"ms": round(v["ms"], 4), "launches": v["launches"],
                                 "tflops": (v["flops"] / (v["ms"] * 1e-3) / 1e12) if v["flops"] and v["ms"] else None,
                                 "gbs": (v["bytes"] / (v["ms"] * 1e-3) / 1e9) if v["bytes"] and v["ms"] else None}
                             for k, v in per_kind.items()}}

    # ---- solve + residual (device factors)
    f = factors_from_plan(h2, plan)
    if world > 1:
        from paper_2502_02395_b200.distributed import factorize_distributed, solve_distributed

        f.partition, f.comm = part, comm
        solve_fn, factor_fn = solve_distributed, factorize_distributed
    else:
        solve_fn, factor_fn = pkg.solve, pkg.factorize
    b = np.random.default_rng(1).standard_normal(c["n"])
    x = solve_fn(f, b)
    torch.cuda.synchronize(dev)
    ts0 = time.perf_counter()
    for _ in range(3):
        x = solve_fn(f, b)
    solve_ms = (time.perf_counter() - ts0) / 3 * 1e3
    perm = cloud.perm
    res = float(np.linalg.norm(h2_matvec(h2, x[perm]) - b[perm]) / np.linalg.norm(b))

    # ---- e2e through the public API with host buffers
    h2_host = host_copy(pkg, h2)
    hb = h2d_bytes(h2_host) + b.nbytes
    e2e_times = []
    for s in range(1 + args.e2e_steps):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        fe = factor_fn(h2_host)
        xe = solve_fn(fe, b)
        torch.cuda.synchronize(dev)
        if s:
            e2e_times.append(time.perf_counter() - t0)
        del fe
    e2e_s = float(np.mean(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": flops / e2e_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(hb),
           "d2h_bytes_per_step": int(xe.nbytes + plan.npd.numel() * 4), "seconds_per_step": e2e_s,
           "includes": "factorize(h2 of host numpy blocks): parallel pinned gather + H2D of bases / leaf near "
                       "blocks / couplings level by level on a copy stream, each level's factorization graph "
                       "queued behind its level's copies (upload and factorization overlap), pivot-status D2H; "
                       "solve(b): H2D b, forward/backward graphs, D2H x. The symbolic part (layout, descriptors, "
                       "CUDA graphs) is cached per structure, the numeric upload is redone every step"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        best = None
        for th in sorted({1, min(8, cores), cores}):   # same thread candidates as --impl reference
            dt, fl = cpu_oracle_time(h2_host, th)
            if best is None or dt < best[0]:
                best = (dt, fl, th)
        dt, fl, th = best
        cpu = {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": th, "kind": "port",
               "sample": f"one full {args.config.upper()} factorization (oracle/h2ulv_oracle.py), fastest of "
                         f"{sorted({1, min(8, cores), cores})} BLAS threads: {th} threads, {dt:.2f} s"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (uniform cube, seed 0)",
                "config": {"workload": workload_name(args.config, c),
                           "parallelism": (f"sharded{world}: boxes of levels >= log2 P split by contiguous leaf "
                                           f"ranges, top levels + root replicated, {backend} exchanges")
                           if world > 1 else "single GPU",
                           "flops_per_step": flops, "padded_flops": plan.flops["total_padded"],
                           "factor_seconds": ms * 1e-3, "solve_ms": solve_ms, "residual": res,
                           "construct_seconds": construct_s, "eager_ms_per_step": eager_ms,
                           "l2": "inputs > L2 (leaf near blocks + bases ~0.4 GB per step)",
                           "depth": tree.depth, "root_dim": plan.root_dim},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
                "gpu_launches": sum(pg.kernel_launches for pg in progs) * args.steps}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
