"""Measured multi-GPU projection on one B200 (analysis; run on the GPU box).

    python tools/scale_projection.py [--config c5] [--worlds 1,2,4,8] [--out gpurun_out/scale]

Only one GPU is reachable from this build, so the W-rank run cannot be timed directly. This
tool times the W-rank *schedule* on the GPU instead: PLG_EMULATE_WORLD=W makes one context
run exactly what each rank runs — every replicated launch (predictions, selection, scans,
bounds, Gram update, residualisation, commit) plus the pair lists split into the W
contiguous rank slices, one launch per slice — with per-launch CUDA events (detail timing)
and the per-(round, stage) stage log (each stage's slice-launch times). The slowest rank's
device time is the production single-GPU time (graph-replayed, no per-launch events: those
events inflate the replicated launches) with each stage's pair-list time replaced by its
slowest slice's:

    T_W = T_1 - sum_stages pair(W = 1) + sum_stages max_slice pair(W)
              - round 0 (exhaustive tiles, split W ways) * (1 - 1/W)  +  exchange

every term measured on the GPU except the exchange: per pruned stage one signal + wait
through peer memory, measured on this GPU through a one-rank peer context (the extra device
time of the peer context over the local one, `peer_overhead_ms_1rank`), plus a per-barrier
NVLink latency allowance (`--nvlink-us`, default 3 us). Rounds with u <= 128 run replicated
on every rank (no exchange) and are counted whole. Output: one JSON
line per W with T_W, the speed-up over W = 1 and the parts.
"""

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child_graph(config):
    """The production single-GPU device time: graph-replayed calls, no per-launch events (the
    engine reads PLG_STAGE_LOG once per process, so this runs in a process of its own)."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2403_03772_b200 as plg

    X = bench.make_input(config)
    eng = plg.Engine(0)
    ms = []
    for _ in range(5):
        eng.causal_order(X)
        ms.append(eng.stats()["total_ms"])
    print(json.dumps({"graph_ms": min(ms[3:]), "ms": ms}), flush=True)


def child(config, world, out, peer):
    """One timed causal order (after a warm-up) under PLG_EMULATE_WORLD=world."""
    sys.path.insert(0, ROOT)
    os.environ["PLG_EMULATE_WORLD"] = str(world)
    slog = os.path.join(out, f"{config}_w{world}{'_peer' if peer else ''}_stages.txt")
    rlog = os.path.join(out, f"{config}_w{world}{'_peer' if peer else ''}_rounds.txt")
    os.environ["PLG_STAGE_LOG"] = slog
    os.environ["PLG_ROUND_TIMES"] = rlog
    import bench
    import paper_2403_03772_b200 as plg

    X = bench.make_input(config)
    eng = plg.Engine.peer(0, 0, 1, X.shape[1]) if peer else plg.Engine(0)
    eng.causal_order(X)
    eng.set_detail_timing(True)
    order = eng.causal_order(X)
    st = eng.stats()
    stage_sum = stage_max = 0.0
    stages = 0
    emu_ms = 0.0
    for line in open(slog):
        if line.startswith("#"):
            emu_ms = float(line.split()[4])
            continue
        f = line.split()
        if float(f[4]) >= 0.0:
            stage_sum += float(f[4])
            stage_max += float(f[5])
            stages += 1
    r0 = float(open(rlog).readline().split()[2])
    print(json.dumps({"world": world, "peer": peer, "total_ms": st["total_ms"], "pair_ms": st["pair_ms"],
                      "stage_sum_ms": stage_sum, "stage_max_ms": stage_max, "stages": stages,
                      "emu_ms": emu_ms, "round0_ms": r0, "pairs": st["pairs_evaluated"],
                      "order_head": list(order[:8])}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "scale"))
    ap.add_argument("--nvlink-us", type=float, default=3.0)
    ap.add_argument("--child", type=int, default=0)
    ap.add_argument("--peer", action="store_true")
    ap.add_argument("--graph", action="store_true")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    if args.graph:
        child_graph(args.config)
        return
    if args.child:
        child(args.config, args.child, args.out, args.peer)
        return

    def run(world, peer=False, graph=False):
        cmd = [sys.executable, __file__, "--config", args.config, "--out", args.out, "--child", str(world)]
        if peer:
            cmd.append("--peer")
        if graph:
            cmd.append("--graph")
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            sys.stderr.write(p.stdout + p.stderr)
            raise SystemExit(f"child failed: {cmd}")
        return json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])

    # the single-GPU base and the exchange cost use the default engine; PLG_PRUNE_SEGLEN and
    # PLG_PRUNE (the refinement ladder), if set, apply to the emulated W-rank runs only
    emu_env = {k: os.environ.pop(k) for k in ("PLG_PRUNE_SEGLEN", "PLG_PRUNE") if k in os.environ}
    seg = emu_env or None
    base = run(1)
    base["graph_ms"] = run(1, graph=True)["graph_ms"]
    peer = run(1, peer=True)
    os.environ.update(emu_env)
    peer_overhead = max(0.0, peer["total_ms"] - base["total_ms"])
    per_stage_xchg = peer_overhead / max(1, base["stages"])
    # Base: the production single-GPU device time (graph-replayed, no per-launch events).
    # Per-launch events inflate the replicated launches' time (~0.17 s on C5), so the W-rank
    # time is that base with the measured pair-list stage times swapped for the slowest
    # slice's: T_W = T_1 - sum_stages(W=1) + sum_stages max_slice(W) - round 0 (1 - 1/W) + exchange.
    t1 = base["graph_ms"]
    for w in [int(x) for x in args.worlds.split(",")]:
        r = base if (w == 1 and seg is None) else run(w)
        assert r["order_head"] == base["order_head"], "emulated schedule changed the order"
        xchg = 0.0 if w == 1 else r["stages"] * (per_stage_xchg + args.nvlink_us * 1e-3)
        # (per-stage exchange cost measured with the default ladder, charged per stage of this one)
        t = t1 - base["stage_sum_ms"] + r["stage_max_ms"] - base["round0_ms"] * (1.0 - 1.0 / w) + xchg
        t_detail = (r["total_ms"] - (r["stage_sum_ms"] - r["stage_max_ms"]) - r["emu_ms"]
                    - r["round0_ms"] * (1.0 - 1.0 / w) + xchg)
        print(json.dumps({"config": args.config, "world": w, "seg_len": os.environ.get("PLG_PRUNE_SEGLEN", "128"),
                          "ladder": os.environ.get("PLG_PRUNE", "default"),
                          "projected_ms": round(t, 2), "speedup_vs_1": round(t1 / t, 3),
                          "base_graph_ms": round(t1, 2), "projected_ms_detail_basis": round(t_detail, 2),
                          "total_ms_emulated": round(r["total_ms"], 2),
                          "pair_stage_sum_ms": round(r["stage_sum_ms"], 2),
                          "pair_stage_max_ms": round(r["stage_max_ms"], 2), "emulation_ms": round(r["emu_ms"], 2),
                          "round0_ms": round(r["round0_ms"], 2), "exchange_ms": round(xchg, 2),
                          "peer_overhead_ms_1rank": round(peer_overhead, 2), "stages": r["stages"],
                          "pairs": r["pairs"], "basis": "detail timing (per-launch events)"}), flush=True)


if __name__ == "__main__":
    main()
