"""Profiling driver (run under ncu on the GPU box, never for bench numbers).

    python tools/profile_round.py --config c5 --mode search   # one search round, u = d
    python tools/profile_round.py --config c2 --mode order    # one full causal order
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2403_03772_b200 as plg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5", choices=sorted(bench.CONFIGS))
    ap.add_argument("--mode", default="search", choices=["search", "order"])
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    X = bench.make_input(args.config)
    eng = plg.Engine(0)
    for _ in range(args.reps):
        if args.mode == "search":
            eng.search(X, list(range(X.shape[1])))
        else:
            eng.causal_order(X)
        print(eng.stats(), flush=True)


if __name__ == "__main__":
    main()
