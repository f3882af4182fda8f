"""Multi-rank peer-memory run at a BASELINE config, every rank checked against the golden.

    torchrun --nproc-per-node W tools/p2p_scale_check.py --config c5 [--shared-gpu]

Each rank builds a peer-memory context (handles exchanged through a gloo group), runs the
causal order (pruned rounds, slices of every stage list exchanged through the IPC-mapped
arenas) and compares the order and every round's winning k with tests/golden/<config>_
order_full.json (k within the goldens' score bar). --shared-gpu puts every rank on cuda:0
(a one-GPU box: the ranks time-slice, so the run says nothing about speed)."""
import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2403_03772_b200 as plg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--shared-gpu", action="store_true")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = 0 if args.shared_gpu else int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    X = np.asfortranarray(bench.make_input(args.config))
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", f"{args.config}_order_full.json")))
    assert hashlib.sha256(X.tobytes(order="F")).hexdigest() == golden["sha256"]
    eng = plg.Engine.peer(local, rank, world, X.shape[1])
    handles = [None] * world
    dist.all_gather_object(handles, eng.p2p_handle())
    eng.p2p_connect(handles)
    dist.barrier()
    t0 = time.time()
    order = eng.causal_order(X)
    el = time.time() - t0
    k = np.asarray(eng.round_k())
    k_ref = np.array([float.fromhex(v) for v in golden["winner_k"]])
    ok_order = order == golden["order"]
    ok_k = bool(np.all(np.abs(k - k_ref) <= 1e-9 * np.abs(k_ref) + 1e-15))
    res = [None] * world
    dist.all_gather_object(res, {"rank": rank, "order_ok": ok_order, "k_ok": ok_k,
                                 "k_sha": hashlib.sha1(k.tobytes()).hexdigest()[:12], "seconds": round(el, 2),
                                 "pairs": eng.stats()["pairs_evaluated"]})
    if rank == 0:
        print(json.dumps({"config": args.config, "world": world, "shared_gpu": args.shared_gpu, "ranks": res,
                          "all_ok": all(r["order_ok"] and r["k_ok"] for r in res),
                          "k_bits_equal_across_ranks": len({r["k_sha"] for r in res}) == 1}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
