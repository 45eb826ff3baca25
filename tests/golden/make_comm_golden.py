"""Golden communication traces from the UNMODIFIED reference simulator
(h2ulv.comm_sim.simulate_factor / simulate_solve, comm_sim.py:92-148) for the
fixture structures at p = 2, 4, 8 ranks.

Run (this container, /root/reference present):  python tests/golden/make_comm_golden.py
Output (committed): tests/golden/comm_sim.json
"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
from h2ulv import comm_sim, geometry  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
NAMES = ["h2_cube512_rank16", "h2_sphere1024_yukawa_tol", "h2_cube1024_sampled", "c2"]


def main():
    out = {}
    for name in NAMES:
        meta = json.load(open(os.path.join(HERE, f"{name}.json")))
        cfg = meta["config"]
        gen = geometry.gen_uniform_cube if cfg["shape"] == "cube" else geometry.gen_sphere_surface
        cloud = gen(cfg["n"], seed=cfg.get("seed", 0))
        tree = geometry.build_tree(cloud, cfg["leaf"])
        lists = geometry.build_interaction_lists(tree, cfg.get("eta", 1.0))
        ranks = {(int(l), i): int(rk[1]) for l, boxes in meta["dims"].items() for i, rk in enumerate(boxes)}
        ent = {}
        for p in (2, 4, 8):
            if p > 2 ** tree.depth:
                continue
            a = comm_sim.assign(tree, p)
            ev = lambda tr: [[e.phase, e.level, e.kind, list(e.participants), e.bytes] for e in tr.events]
            ent[str(p)] = {"factor": ev(comm_sim.simulate_factor(tree, lists, ranks, a)),
                           "solve": ev(comm_sim.simulate_solve(tree, lists, ranks, a))}
        out[name] = ent
    with open(os.path.join(HERE, "comm_sim.json"), "w") as fh:
        json.dump(out, fh)
    print({k: {p: len(v["factor"]) for p, v in e.items()} for k, e in out.items()})


if __name__ == "__main__":
    main()
