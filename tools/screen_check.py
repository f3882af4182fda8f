"""An engine variant against the goldens (analysis): for each config, the causal order with
the engine knobs of the environment (or an experimental build, e.g. the screening patch in
profiles/r2_screening_experiment.patch with PLG_SCREEN=1), checked against
tests/golden/<config>_order_full.json (order; every round's winning k within 1e-9 rel.),
with the median device time and the pair counts.

    python tools/screen_check.py --configs c3,c5 --reps 3
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c3,c5")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    import bench
    import paper_2403_03772_b200 as plg

    for cfg in args.configs.split(","):
        X = bench.make_input(cfg)
        eng = plg.Engine(0)
        order = eng.causal_order(X)
        ms = []
        for _ in range(args.reps):
            o2 = eng.causal_order(X)
            assert o2 == order
            ms.append(eng.stats()["total_ms"])
        st = eng.stats()
        rec = {"tag": args.tag, "config": cfg, "median_ms": float(np.median(ms)), "ms": ms,
               "pairs": st["pairs_evaluated"], "screened": st.get("pairs_screened"),
               "near_ties": st["near_ties"], "min_gap": st["min_gap"]}
        gp = os.path.join(ROOT, "tests", "golden", f"{cfg}_order_full.json")
        if os.path.exists(gp):
            g = json.load(open(gp))
            k = np.asarray(eng.round_k())
            kr = np.array([float.fromhex(v) for v in g["winner_k"]])
            rec["order_ok"] = order == g["order"]
            rec["k_ok"] = bool(np.all(np.abs(k - kr) <= 1e-9 * np.abs(kr) + 1e-15))
            rec["golden_pairs"] = g.get("pairs_evaluated")
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
