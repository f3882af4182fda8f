"""Per-stage anatomy of the pruned rounds (analysis; run on the GPU box).

    python tools/stage_profile.py [--config c5] [--out gpurun_out/stages]

One causal order with per-launch CUDA events (detail timing), PLG_STAGE_LOG (list length
and pair-list launch time of every (round, stage)) and PLG_ROUND_TIMES (device time of
every round). Prints, per u-bucket: rounds, device ms, pair-list ms by stage, pairs by
stage, the pair-list rate (ns per pair-eval) and the non-pair remainder.
"""

import argparse
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "stages"))
    ap.add_argument("--buckets", default="2000,1500,1000,700,500,300,200,129")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    slog = os.path.join(args.out, f"{args.config}_stage_log.txt")
    rlog = os.path.join(args.out, f"{args.config}_round_times.txt")
    os.environ["PLG_STAGE_LOG"] = slog
    os.environ["PLG_ROUND_TIMES"] = rlog
    import bench
    import paper_2403_03772_b200 as plg

    X = bench.make_input(args.config)
    eng = plg.Engine(0)
    eng.causal_order(X)  # warm-up
    eng.set_detail_timing(True)
    eng.causal_order(X)
    st = eng.stats()
    print({k: st[k] for k in ("total_ms", "pair_ms", "resid_ms", "pairs_evaluated", "launches")})
    rounds = {}
    for line in open(rlog):
        r, u, ms = line.split()
        rounds[int(r)] = (int(u), float(ms))
    stages = defaultdict(dict)
    for line in open(slog):
        if line.startswith("#"):
            continue
        r, u, s, n, ms = line.split()[:5]
        stages[int(r)][int(s)] = (int(n), float(ms))
    edges = [int(x) for x in args.buckets.split(",")]
    print(f"{'u range':>12} {'rounds':>6} {'dev ms':>9} {'pair ms':>9} {'other ms':>9} "
          + " ".join(f"{'s%d pairs' % s:>11} {'s%d ms' % s:>8}" for s in range(4)) + f" {'ns/pair':>8}")
    for hi, lo in zip(edges[:-1], edges[1:]):
        rs = [r for r, (u, _) in rounds.items() if lo < u <= hi]
        if not rs:
            continue
        dev = sum(rounds[r][1] for r in rs)
        per = [[0, 0.0] for _ in range(4)]
        for r in rs:
            for s, (n, ms) in stages.get(r, {}).items():
                if s < 4:
                    per[s][0] += n
                    per[s][1] += max(ms, 0.0)
        pair_ms = sum(p[1] for p in per)
        npairs = sum(p[0] for p in per)
        line = f"{lo + 1:>5}-{hi:<6} {len(rs):>6} {dev:>9.1f} {pair_ms:>9.1f} {dev - pair_ms:>9.1f} "
        line += " ".join(f"{p[0]:>11d} {p[1]:>8.1f}" for p in per)
        line += f" {pair_ms * 1e6 / max(1, 2 * npairs):>8.2f}"
        print(line)
    r0 = rounds.get(0)
    print(f"round 0 (exhaustive): {r0}")


if __name__ == "__main__":
    main()
