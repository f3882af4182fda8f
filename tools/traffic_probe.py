"""Child process of bench.py's in-job traffic measurement: one causal order of a bench
config on cuda:0, run under ncu (which profiles a single pair-kernel launch of it).

    python tools/traffic_probe.py <config> <prune 0|1>
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2403_03772_b200 as plg  # noqa: E402

if __name__ == "__main__":
    cfg, prune = sys.argv[1], sys.argv[2] == "1"
    X = bench.make_input(cfg)
    eng = plg.Engine(0)
    eng.set_prune(prune)
    eng.causal_order(X)
