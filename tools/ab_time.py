"""A/B timing helper (analysis): median device time of a causal order under the current
environment's engine knobs, plus the order's hash (to compare variants).

    PLG_LIST_VAR=8 python tools/ab_time.py --config c5 --reps 3
"""
import argparse
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tag", default="")
    ap.add_argument("--peer", action="store_true", help="one-rank peer-memory context (every exchange through its arena)")
    ap.add_argument("--pkg", default="", help="directory holding an A/B snapshot of the package (tools/ab_snapshot.sh)")
    ap.add_argument("--detail", action="store_true", help="per-launch timing: pair_ms / resid_ms (adds event overhead)")
    args = ap.parse_args()
    if args.pkg:
        sys.path.insert(0, os.path.join(ROOT, args.pkg))
    import paper_2403_03772_b200 as plg
    import bench
    X = bench.make_input(args.config)
    eng = plg.Engine.peer(0, 0, 1, X.shape[1]) if args.peer else plg.Engine(0)
    if args.detail:
        eng.set_detail_timing(True)
    order = eng.causal_order(X)
    ms = []
    for _ in range(args.reps):
        order = eng.causal_order(X)
        ms.append(eng.stats()["total_ms"])
    k = eng.round_k()
    st = eng.stats()
    print(json.dumps({"tag": args.tag, "pkg": os.path.dirname(plg.__file__), "config": args.config, "median_ms": float(np.median(ms)), "ms": ms,
                      "pairs": st["pairs_evaluated"], "launches": st["launches"],
                      "pair_ms": st["pair_ms"], "resid_ms": st["resid_ms"],
                      "order_sha": hashlib.sha1(str(order).encode()).hexdigest()[:12],
                      "k_sha": hashlib.sha1(np.asarray(k).tobytes()).hexdigest()[:12]}), flush=True)


if __name__ == "__main__":
    main()
