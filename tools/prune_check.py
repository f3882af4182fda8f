"""Pruned vs exhaustive causal order on one config (analysis tool, GPU box).

    python tools/prune_check.py --config c3 [--tileseg]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    import bench
    import paper_2403_03772_b200 as plg

    X = np.asfortranarray(bench.make_input(args.config))
    eng = plg.Engine(0)
    eng.set_detail_timing(True)
    res = {}
    for mode in ("prune", "full"):
        eng.set_prune(mode == "prune")
        for _ in range(args.reps):
            t = time.time()
            order = eng.causal_order(X)
            wall = time.time() - t
        res[mode] = (order, wall, eng.stats())
    same = res["prune"][0] == res["full"][0]
    out = {"config": args.config, "same_order": same,
           "first_diff": None if same else next(i for i, (a, b) in enumerate(zip(res["prune"][0], res["full"][0])) if a != b)}
    for mode in res:
        s = res[mode][2]
        out[mode] = {"wall_s": res[mode][1], "device_s": s["total_ms"] / 1e3, "pair_s": s["pair_ms"] / 1e3,
                     "pairs_evaluated": s["pairs_evaluated"], "pair_evals": s["pair_evals"],
                     "frac_unordered": s["pairs_evaluated"] / (s["pair_evals"] / 2), "launches": s["launches"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
