"""Per-stage cost of the multi-rank schedule on one GPU (analysis tool): the same causal order
through a one-rank NCCL communicator (PLG_NCCL_SELFTEST=1: a host synchronisation and an
all-gather per pruned stage) against a local context."""
import os, sys, time
os.environ["PLG_NCCL_SELFTEST"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2403_03772_b200 as plg

X = np.asfortranarray(bench.make_input(sys.argv[1] if len(sys.argv) > 1 else "c5"))
for mode in ("local", "nccl"):
    eng = plg.Engine.distributed(0, 0, 1, plg.nccl_unique_id()) if mode == "nccl" else plg.Engine(0)
    eng.causal_order(X)
    t = time.time(); o = eng.causal_order(X); w = time.time() - t
    print(mode, {"wall_s": round(w, 3), "device_s": round(eng.stats()["total_ms"] / 1e3, 3), "launches": eng.stats()["launches"]})
