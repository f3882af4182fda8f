"""Sweep PLG_PRUNE settings on one config (analysis tool, GPU box).

    python tools/prune_sweep.py --config c5 --specs "8:3:0.05,0.15" "4:3:0.05,0.15"
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, json
sys.path.insert(0, %r)
import numpy as np, bench, paper_2403_03772_b200 as plg
X = np.asfortranarray(bench.make_input(%r))
eng = plg.Engine(0)
eng.set_detail_timing(True)
o1 = eng.causal_order(X)
o2 = eng.causal_order(X)
s = eng.stats()
print(json.dumps({"order_hash": hash(tuple(o2)), "same": o1 == o2, "device_s": s["total_ms"] / 1e3,
                  "pair_s": s["pair_ms"] / 1e3, "pairs": s["pairs_evaluated"]}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--specs", nargs="+", required=True)
    args = ap.parse_args()
    for spec in args.specs:
        env = dict(os.environ, PLG_PRUNE=spec, PLG_PRUNE_DEBUG="1")
        r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, args.config)], env=env, capture_output=True, text=True)
        dbg = [l for l in r.stderr.splitlines() if l.startswith("[plg prune]")]
        out = r.stdout.strip().splitlines()
        print(spec, out[-1] if out else r.stderr[-500:], dbg[-1] if dbg else "", flush=True)


if __name__ == "__main__":
    main()
