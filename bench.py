"""H²-ULV factorization benchmark (BASELINE.json metric) — one JSON line.

A "step" is one complete H²-ULV factorization (all levels + root) of the
configuration named by `--config` (default M1 = the metric's configuration:
Laplace-3D, N = 1 048 576 uniform-cube points, leaf 256, tol 1e-8, shift
2e6 (1e5 breaks down at the root), 512/512 sampling; it
fits one B200).  The H² matrix is built once (untimed; construction is not
part of the reference metric).

  value         factorization GFLOP/s = reference flop model total_true
                (dense_core.flop_count) / device time, operands resident in
                HBM, whole program replayed as one CUDA graph
  e2e           the same metric through the public API with HOST buffers:
                factorize(h2 of numpy blocks in pinned host memory) +
                solve(b) -> x on the host, all host<->device copies inside the
                timed region (the upload streams level by level and overlaps
                the factorization)
  roofline      dominant kernel = grouped FP64 DMMA GEMM; achieved flops over
                its CUDA-event time inside an instrumented pass of K steps
  solve         device-timed forward + backward sweeps, GB/s of the SURVEY
                §8(d) algorithmic solve bytes
  cpu_baseline  the CPU oracle port (oracle/h2ulv_oracle.py) on the host cores,
                on a bounded sample: the diagonal sub-hierarchy under one box of
                level L0 = max(0, depth - 9) (1/8 of the leaves at N = 1M)

Multi-GPU (`torchrun ... bench.py --gpus N`): ONE factorization sharded over
the ranks (distributed.py: boxes of the levels >= log2 N split by contiguous
leaf ranges, the levels above computed by subtree process groups, NCCL
all_gather of the V halo and one AllReduce per parent near block at the
merges — comm_sim.simulate_factor's events); strong scaling, time = max over
ranks.
`--impl reference` times the CPU oracle port (the reference is pure Python and
does not travel to the GPU box) on rank 0 only; each step factors one sampled
sub-hierarchy (the sample rotates over the 2^L0 subtrees), the warm-up steps
choose the BLAS thread count.
"""

import argparse
import gc
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


def _measured_hbm():
    """MEASURED_PEAKS.json hbm_gbs (driver-written, this pool's B200s); 6547.2 = its round-2 value."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6547.2


HBM_PEAK_GBS = _measured_hbm()
FP64_PEAK_TFLOPS = 37.1   # measured DMMA issue peak, profiles/r01_fp64_peak.txt (no FP64 entry in MEASURED_PEAKS.json)

CONFIGS = {
    "c1": dict(shape="cube", n=4096, leaf=256, family="laplace", shift=1e3, tol=1e-8, s_far=0, s_near=0),
    "c2": dict(shape="cube", n=65536, leaf=256, family="laplace", shift=1e5, tol=1e-8, s_far=512, s_near=512),
    "c3": dict(shape="sphere", n=262144, leaf=256, family="yukawa", shift=1e5, tol=1e-8, s_far=512, s_near=512),
    "m1": dict(shape="cube", n=1048576, leaf=256, family="laplace", shift=2e6, tol=1e-8, s_far=512, s_near=512),
    # BASELINE configs[3]: Gaussian covariance exp(-(r/l)^2), l = 0.1 (no reference family: opt-in
    # GaussianKernelSpec; shift ~ 2x the kernel row sum N pi^1.5 l^3, SURVEY §8(d) C4 probes)
    "c4": dict(shape="cube", n=1048576, leaf=256, family="gaussian", length_scale=0.1, shift=2e4, tol=1e-8,
               s_far=512, s_near=512),
    # BASELINE configs[4] points on one GPU: the metric config at the tolerance sweep ends
    "m1_tol6": dict(shape="cube", n=1048576, leaf=256, family="laplace", shift=2e6, tol=1e-6, s_far=512, s_near=512),
    "m1_tol10": dict(shape="cube", n=1048576, leaf=256, family="laplace", shift=2e6, tol=1e-10, s_far=512,
                     s_near=512),
    "m2": dict(shape="cube", n=2097152, leaf=256, family="laplace", shift=4e6, tol=1e-8, s_far=512, s_near=512),
    "m4": dict(shape="cube", n=4194304, leaf=256, family="laplace", shift=8e6, tol=1e-8, s_far=512, s_near=512),
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
    if c["family"] == "gaussian":
        kernel = pkg.GaussianKernelSpec(length_scale=c["length_scale"], diagonal_shift=c["shift"])
    else:
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
    """Bytes one factorize(h2) copies host -> device: bases (q_red / q_skel, or for the
    levels a pinned arena ships in compact-WY form Y, Yt and the signs), leaf near blocks,
    couplings."""
    depth = h2.tree.depth
    arena = getattr(h2, "_arena", None)
    wy = set(arena.wy_levels) if arena is not None and arena.intact(h2) else set()
    nb = 0
    for (l, i), b in h2.bases.items():
        if l in wy:
            nb += 8 * (2 * b.q_skel.shape[0] * b.rank + b.rank)
        else:
            nb += b.q_red.nbytes + b.q_skel.nbytes
    nb += sum(v.nbytes for k, v in h2.near_blocks.items() if k[0] == depth)
    nb += sum(v.nbytes for v in h2.couplings.values())
    return nb


def sample_level(depth):
    """Level whose boxes root the CPU samples: one sample = 2^-(L0) of the leaves."""
    return max(0, depth - 9)


def sub_hierarchy(hh, L0, g):
    """The diagonal sub-hierarchy of a host H² under box g of level L0, as a
    standalone H² of depth D - L0 (box i of level l -> box i - g 2^(l-L0) of
    level l - L0): its leaf near blocks, bases and couplings, with the near /
    far pairs whose both boxes lie in the subtree.  Its factorization is the
    share of the full factorization's work that this subtree does (cross-
    subtree near pairs and the levels above L0 excluded); the flop report of
    the oracle counts exactly that work."""
    from types import SimpleNamespace

    D = hh.tree.depth
    d = D - L0
    near, far = [set() for _ in range(d + 1)], [set() for _ in range(d + 1)]
    bases, nblk, cpl = {}, {}, {}
    for s_ in range(d, -1, -1):
        l = s_ + L0
        lo, hi = g << s_, (g + 1) << s_
        near[s_] = {(i - lo, j - lo) for (i, j) in hh.lists.near[l] if lo <= i < hi and lo <= j < hi}
        far[s_] = {(i - lo, j - lo) for (i, j) in hh.lists.far[l] if lo <= i < hi and lo <= j < hi}
        if s_ == 0:
            near[0], far[0] = {(0, 0)}, set()
            continue
        for i in range(lo, hi):
            bases[(s_, i - lo)] = hh.bases[(l, i)]
        for (i, j) in far[s_]:
            if i > j:
                cpl[(s_, i, j)] = hh.couplings[(l, i + lo, j + lo)]
    lo = g << d
    for (i, j) in near[d]:
        if i >= j:
            nblk[(d, i, j)] = hh.near_blocks[(D, i + lo, j + lo)]
    tree = SimpleNamespace(depth=d)
    lists = SimpleNamespace(near=near, far=far)
    return SimpleNamespace(tree=tree, lists=lists, bases=bases, near_blocks=nblk, couplings=cpl)


class OracleSampler:
    """Times the CPU oracle port's factorize on the sub-hierarchies of a host H²."""

    def __init__(self, hh):
        self.hh = hh
        self.L0 = sample_level(hh.tree.depth)
        self.count = 2 ** self.L0
        self.subs = {}

    def sub(self, g):
        g %= self.count
        if g not in self.subs:
            self.subs[g] = sub_hierarchy(self.hh, self.L0, g) if self.L0 else self.hh
        return self.subs[g]

    def run(self, g, threads):
        from threadpoolctl import threadpool_limits

        from oracle import h2ulv_oracle as orc

        sub = self.sub(g)
        with threadpool_limits(limits=threads):
            t0 = time.perf_counter()
            f = orc.factorize(sub)
            dt = time.perf_counter() - t0
        return dt, int(f.flops["total_true"])

    def describe(self, key):
        if self.L0 == 0:
            return f"one full {key.upper()} factorization per step"
        return (f"{key.upper()}: per step the diagonal sub-hierarchy under one level-{self.L0} box "
                f"(1/{self.count} of the leaves, levels {self.hh.tree.depth}..{self.L0 + 1} + its Cholesky at "
                f"level {self.L0}; cross-subtree near pairs excluded), rotating over the {self.count} boxes")


def thread_candidates():
    cores = os.cpu_count() or 1
    return sorted({1, min(8, cores), cores})


def reference_h2(pkg, c):
    """Host (numpy) H² for the CPU arm: the GPU construct (skeletons bit-exact vs the
    reference, tests/test_gpu_fullsize.py) when a GPU is present, else the oracle's own."""
    import torch

    kernel, cloud, tree, lists, cfg = build_problem(pkg, c)
    if torch.cuda.is_available():
        h2 = pkg.construct(kernel, tree, lists, cfg, cloud, device=torch.device("cuda", 0))
        hh = host_copy(pkg, h2)
        del h2
        from paper_2502_02395_b200.ulv_factor import clear_cache

        clear_cache()
        torch.cuda.empty_cache()
        return hh, "paper_2502_02395_b200.construct (GPU), downloaded to numpy"
    from oracle import h2ulv_oracle as orc

    return orc.construct(kernel, tree, lists, cfg, cloud), "oracle construct (CPU)"


def run_reference(args, c, key):
    """--impl reference: the CPU oracle port on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2502_02395_b200 as pkg

    hh, src = reference_h2(pkg, c)
    smp = OracleSampler(hh)
    cands = thread_candidates()
    # warm-up steps double as the BLAS thread sweep (1, 8 and nproc threads)
    rates = {}
    for w in range(args.warmup):
        th = cands[w % len(cands)]
        dt, fl = smp.run(w, th)
        rates.setdefault(th, []).append(fl / dt)
    for th in cands:
        if th not in rates:
            dt, fl = smp.run(0, th)
            rates[th] = [fl / dt]
    th = max(rates, key=lambda t: max(rates[t]))
    tot_t = tot_f = 0.0
    for st in range(args.steps):
        dt, fl = smp.run(args.warmup + st, th)
        tot_t += dt
        tot_f += fl
    val = tot_f / tot_t / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (uniform cube, seed 0)" if c["shape"] == "cube" else "synthetic (sphere, seed 0)",
            "config": {"workload": workload_name(key, c), "flops_per_step": tot_f / args.steps,
                       "sample": smp.describe(key), "h2_source": src},
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": th, "kind": "port",
                             "sample": smp.describe(key) + f"; oracle/h2ulv_oracle.py, OpenBLAS threads={th} "
                                       f"(best of {cands} over the warm-up steps), host has {os.cpu_count()} cores"},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def solve_bytes(plan):
    """SURVEY §8(d) algorithmic bytes of one solve (w = 1; every basis / factor
    block read once per sweep): 2*8*[sum n^2 + sum r(r+1)/2 + sum_{near i>j} r_i r_j
    + sum_{near (a,b)} k_a r_b] + 2*8*d(d+1)/2."""
    tot = 0
    for l, B in plan.bufs.items():
        lay = B.lay
        n, k, r = lay.n.astype(np.int64), lay.k.astype(np.int64), lay.r.astype(np.int64)
        tot += int((n * n).sum() + (r * (r + 1) // 2).sum() + (k * r).sum())
        for (i, j) in lay.off_pairs:
            tot += int(r[i] * r[j] + k[i] * r[j] + k[j] * r[i])
    d = plan.root_dim
    return 16 * tot + 16 * (d * (d + 1) // 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="m1", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-exact-residual", action="store_true",
                    help="skip the direct-sum ||A_exact x - b|| (N^2 kernel evaluations, ~1 s at N = 1M)")
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
    # every rank builds the (replicated) H²: share the host cores among the ranks of this node
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    workers = max(1, min(32, (os.cpu_count() or 1) // max(local_world, 1)))
    h2 = pkg.construct(kernel, tree, lists, cfg, cloud, device=dev, workers=workers)
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
                "note": ("achieved = useful flops of ALL grouped-GEMM launches / their CUDA-event time. Levels "
                         "whose bases carry the compact-WY form (the N = 1M leaf) replace the 3n^3 of Q^T (A Q) "
                         "by thin K <= 2k GEMMs (4n^2k + 4nk^2 flops): fewer flops at a lower DMMA rate, so this "
                         "fraction is lower than with the dense transform while the step is faster"),
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
    solve_ms = (time.perf_counter() - ts0) / 3 * 1e3     # host wall, incl. b / x transfers
    perm = cloud.perm
    res = float(np.linalg.norm(h2_matvec(h2, x[perm]) - b[perm]) / np.linalg.norm(b))
    exact = None
    if rank == 0 and not args.no_exact_residual:
        # ||A_exact x - b|| / ||b|| by the GPU direct sum (no N^2 matrix): the true accuracy
        from paper_2502_02395_b200.direct_sum import exact_residual

        torch.cuda.synchronize(dev)
        tx0 = time.perf_counter()
        exact = {"residual": exact_residual(kernel, cloud, x, b, device=dev)}
        exact["seconds"] = time.perf_counter() - tx0
        exact["pairs_per_s"] = float(c["n"]) ** 2 / exact["seconds"]
    solve = None
    if world == 1:
        # device-timed forward + backward sweeps (graph replays), operands in HBM
        from paper_2502_02395_b200.ulv_solve import _plan_for

        sp = _plan_for(f, 1, "parallel")
        for _ in range(3):
            sp.run_forward(stream)
            sp.run_backward(stream)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(args.steps):
            sp.run_forward(stream)
            sp.run_backward(stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        s_ms = e0.elapsed_time(e1) / args.steps
        # the per-factorization prepare step of the solve (inverses, [V | q_skel~], M blocks:
        # derived from the stored factor blocks once per factorization, before the first solve;
        # inside e2e, outside both device-timed regions — reported here)
        e0.record(stream)
        for _ in range(args.steps):
            sp.prepare.launch(stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        prep_ms = e0.elapsed_time(e1) / args.steps
        sb = solve_bytes(plan)
        # bytes the steps of THIS path move (basis / factor blocks as the programs count them):
        # below the formula on neighbour-free levels (V replaces q_red, no L read), above it
        # where explicit inverses are read whole
        pb = sum(int(wk[2]) for pg in (sp.fwd, sp.bwd) if pg is not None for wk in pg.work)
        solve = {"ms": s_ms, "algorithmic_bytes": sb, "gbs": sb / (s_ms * 1e-3) / 1e9,
                 "hbm_peak_gbs": HBM_PEAK_GBS, "frac": sb / (s_ms * 1e-3) / 1e9 / HBM_PEAK_GBS,
                 "prepare_ms": prep_ms,
                 "path_bytes": pb, "path_gbs": pb / (s_ms * 1e-3) / 1e9,
                 "path_frac": pb / (s_ms * 1e-3) / 1e9 / HBM_PEAK_GBS,
                 "note": "SURVEY §8(d) bytes (w = 1): every basis / factor block read once per sweep; "
                         "forward + backward CUDA graphs replayed back to back, CUDA events"}

    cpu = None
    # the CPU baseline runs AFTER the e2e leg (its BLAS threads and multi-GB host copies would
    # otherwise still compete for the host while the e2e upload runs); its input is copied now
    smp = OracleSampler(host_copy(pkg, h2)) if rank == 0 and world == 1 and not args.no_cpu_baseline else None

    def cpu_baseline():
        best = None
        for th in thread_candidates():   # same candidates as --impl reference
            dt, fl = smp.run(0, th)
            if best is None or fl / dt > best[1] / best[0]:
                best = (dt, fl, th)
        dt, fl, th = best
        return {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": th, "kind": "port",
                "sample": smp.describe(args.config) + f" (box 0 here); oracle/h2ulv_oracle.py, fastest of "
                          f"{thread_candidates()} BLAS threads: {th} threads, {dt:.2f} s for {fl:.3e} flops"}

    # ---- e2e through the public API with host buffers (the H² blocks in pinned host memory)
    from paper_2502_02395_b200.h2_build import to_pinned_host

    padded, root_dim, npd_n = plan.flops["total_padded"], plan.root_dim, plan.npd.numel()
    launches = sum(pg.kernel_launches for pg in progs) * args.steps
    # the e2e leg builds its own (streamed) plan: release the device-resident one first
    # so the largest configs hold one factorization in HBM at a time
    sp = f = plan = progs = work = None
    gc.collect()
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    e2e = None
    h2_host = to_pinned_host(h2)
    hb = h2d_bytes(h2_host) + b.nbytes
    l2_note = (f"inputs > L2 (leaf near blocks + bases {h2d_bytes(h2_host) / 1e9:.2f} GB per step "
               f"vs 126 MB L2)")
    if args.e2e_steps > 0:     # the device-built H² is not needed any more: free its HBM too
        h2 = None
        gc.collect()
        torch.cuda.empty_cache()
    e2e_times = []
    for s_ in range(1 + args.e2e_steps if args.e2e_steps > 0 else 0):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        fe = factor_fn(h2_host)
        xe = solve_fn(fe, b)
        torch.cuda.synchronize(dev)
        if s_:
            e2e_times.append(time.perf_counter() - t0)
        del fe
    if e2e_times:
        e2e_s = float(np.mean(e2e_times))
        if world > 1:
            t = torch.tensor([e2e_s], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": flops / e2e_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(hb),
           "d2h_bytes_per_step": int(xe.nbytes + npd_n * 4), "seconds_per_step": e2e_s,
           "includes": "factorize(h2): the reference's numpy H2Matrix data model, its blocks in one pinned host "
                       "buffer (to_pinned_host); H2D of bases / leaf near blocks / couplings level by level on a "
                       "copy stream, each level's factorization graph queued behind its level's copies (upload "
                       "and factorization overlap); bases of compact-WY levels travel as their Householder form "
                       "(Y, Yt, signs) and q_full is rebuilt on the device; pivot-status D2H; solve(b): H2D b, "
                       "the per-factorization solve prepare, forward/backward graphs, D2H x. The symbolic part "
                       "(layout, descriptors, CUDA graphs) is cached per structure, the numeric upload is redone "
                       "every step"}

    if smp is not None:
        cpu = cpu_baseline()
        smp = None

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (uniform cube, seed 0)" if c["shape"] == "cube" else "synthetic (sphere, seed 0)",
                "config": {"workload": workload_name(args.config, c),
                           "parallelism": (f"sharded{world}: boxes of levels >= log2 P split by contiguous leaf "
                                           f"ranges, levels < log2 P by subtree process groups (merge AllReduces per parent near block), {backend} exchanges")
                           if world > 1 else "single GPU",
                           "flops_per_step": flops, "padded_flops": padded,
                           "factor_seconds": ms * 1e-3, "solve_ms_host": solve_ms, "residual": res,
                           "exact_residual": exact,
                           "construct_seconds": construct_s, "eager_ms_per_step": eager_ms,
                           "l2": l2_note,
                           "depth": tree.depth, "root_dim": root_dim},
                "roofline": roofline, "solve": solve, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
                "gpu_launches": launches}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
