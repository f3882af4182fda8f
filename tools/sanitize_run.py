"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Small config (d = 300, n = 2 000, sparse Laplace DAG) through every hot-path kernel family:
pruned causal order (cooperative pair-list kernels incl. the short-list one, atomic work
fetch, last-finisher finalisation, selection/scan/bound kernels), the same through a one-rank
peer-memory context, exhaustive causal order (mbarrier ring pair
kernel, small-round kernels), one search round, the fused residualisation, the weights
step and the VAR front-end. Run under a sanitizer as

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

and compare nothing but the sanitizer's error summary: the orders are checked against
each other (pruned == exhaustive) so a silently corrupted run still fails.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2403_03772_b200 as plg  # noqa: E402


def main() -> None:
    d, n = int(os.environ.get("SAN_D", 300)), int(os.environ.get("SAN_N", 2000))
    dag = plg.gen_sparse_dag(d, avg_parents=2.0, seed=5)
    X = np.asfortranarray(plg.sample_lingam(dag, n, seed=5, kind="laplace"))
    eng = plg.Engine(0)
    eng.set_prune(True)
    print("pruned order", flush=True)
    o_pruned = eng.causal_order(X)
    st = eng.stats()
    eng.set_prune(False)
    print("exhaustive order", flush=True)
    o_exh = eng.causal_order(X)
    assert o_pruned == o_exh, "pruned and exhaustive orders differ"
    if os.environ.get("SAN_PEER", "1") == "1":
        peer = plg.Engine.peer(0, 0, 1, d)  # every exchange through the peer-memory arena (signal/wait, scatter)
        assert peer.causal_order(X) == o_exh, "peer-memory and local orders differ"
    print("orders ok", flush=True)
    chosen, scores = eng.search(X, list(range(d)))
    assert chosen == o_exh[0]
    B, pinv = eng.fit_weights(X, o_exh)
    assert np.isfinite(B).all()
    rng = np.random.default_rng(3)
    ts = np.zeros((400, 60))
    for t in range(1, 400):
        ts[t] = 0.5 * ts[t - 1] + rng.laplace(size=60)
    plg.estimate_var(np.asfortranarray(ts), 1)
    print(f"sanitize workload ok: d={d} n={n} pairs_evaluated={st['pairs_evaluated']} of "
          f"{st['pair_evals'] // 2}; pinv={pinv}")


if __name__ == "__main__":
    main()
