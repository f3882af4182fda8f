"""Generate the committed golden orders under tests/golden/ (run here, on CPU).

Inputs are produced by the package's seeded generators (C++ mt19937_64, deterministic
across machines of this image); the expected outputs come from the CPU oracle
(oracle/plingam_oracle.c, the restated reference). Each fixture stores the SHA-256 of
the input matrix so a GPU test can prove it fed the oracle's exact input.

    python tests/golden/make_golden.py [c1 c2 c4]
    python tests/golden/make_golden.py --full c3 c5   # full orders by the oracle's exact pruned rounds
"""

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle_lib  # noqa: E402
import paper_2403_03772_b200 as plg  # noqa: E402

WORKERS = int(os.environ.get("GOLDEN_WORKERS", os.cpu_count() or 1))


def digest(X: np.ndarray) -> str:
    return hashlib.sha256(np.asfortranarray(X).tobytes(order="F")).hexdigest()


def config_input(name: str) -> np.ndarray:
    """The synthetic inputs of BASELINE.json configs."""
    if name == "c2":  # sparse DAG d=100, n=10000, Laplace noise, seed 1
        dag = plg.gen_sparse_dag(100, avg_parents=2.0, seed=1)
        return plg.sample_lingam(dag, 10000, seed=1, noise=(0.0, 1.0), kind="laplace")
    if name == "c3":  # Perturb-seq-shaped d=1000, n=10000, heavy-tailed noise, seed 1
        dag = plg.gen_sparse_dag(1000, avg_parents=2.0, seed=1)
        return plg.sample_lingam(dag, 10000, seed=1, noise=(0.0, 1.0), kind="t3")
    if name == "c4":  # VarLiNGAM lag 1: d=500, T=2500 SVAR, Laplace noise; the path sees the residuals
        return c4_residuals()
    if name == "c5":  # large synthetic d=2000, n=10000, Laplace noise, seed 1
        dag = plg.gen_sparse_dag(2000, avg_parents=2.0, seed=1)
        return plg.sample_lingam(dag, 10000, seed=1, noise=(0.0, 1.0), kind="laplace")
    raise ValueError(name)


def c4_series():
    """SVAR d=500, T=2500, burn-in 500: sparse acyclic B0 (|w| in [0.1, 0.5]) and a diagonal
    lag-1 matrix with entries U(0.2, 0.5), so M1 = (I - B0)^-1 B1 has spectral radius <= 0.5."""
    d = 500
    b0 = plg.gen_sparse_dag(d, avg_parents=2.0, seed=1, wmin=0.1, wmax=0.5)
    b1 = np.diag(plg.uniform_vector(d, 1, 0.2, 0.5))
    return b0, plg.sample_svar(b0, [np.asfortranarray(b1)], T=2500, burn_in=500, seed=1, noise=(0.0, 1.0),
                               kind="laplace")


def c4_residuals():
    _, X = c4_series()
    return plg._estimate_var_qr(X, 1)[1]  # the reference's QR (CPU); the device path is tested against it


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1", "c2"], help="c1 c2 c4 (c3: hours on 8 cores)")
    ap.add_argument("--full", action="store_true",
                    help="whole order + winning k per round via orc_causal_order_pruned (C3: ~15 min, "
                         "C5: ~1.5 h on 8 cores)")
    args = ap.parse_args()
    if args.full:
        for name in args.configs:
            make_full(name)
        return
    if "c1" in args.configs:
        make_c1()
    for name in [c for c in args.configs if c != "c1"]:
        make_config(name)


def make_c1():
    # C1: acceptance AC1 seeds (acceptance.cpp:39-69), two-level DAG d=10, m=10000, U(0,1) noise
    c1 = []
    for s in range(50):
        seed = 42000 + s
        dag = plg.gen_two_level_dag(10, seed=seed)
        X = plg.sample_lingam(dag, 10000, seed=seed)
        order = oracle_lib.causal_order(X, parallel=True, workers=WORKERS, fast=True)
        B, pinv = oracle_lib.fit_weights(X, order)
        c1.append({"seed": seed, "sha256": digest(X), "order": order, "B": B.tolist(), "used_pinv": pinv})
    with open(os.path.join(HERE, "c1_two_level.json"), "w") as f:
        json.dump({"config": "two-level DAG d=10 n=10000 U(0,1) noise, seeds 42000..42049",
                   "generator": "gen_two_level_dag + sample_lingam", "cases": c1}, f)
    print("c1 done", flush=True)


def make_config(name):
    if True:
        X = config_input(name)
        t0 = time.time()
        order, scores = oracle_lib.causal_order(X, parallel=True, workers=WORKERS, fast=True, return_scores=True)
        el = time.time() - t0
        B, pinv = oracle_lib.fit_weights(X, order)
        # per-round best-vs-second gap of k (the margin the GPU must respect)
        gaps = []
        for r in range(scores.shape[0]):
            s = np.sort(-scores[r][np.isfinite(scores[r])])
            gaps.append(float(s[1] - s[0]) if s.size > 1 else None)
        with open(os.path.join(HERE, f"{name}_order.json"), "w") as f:
            json.dump({"config": name, "n": int(X.shape[0]), "d": int(X.shape[1]), "sha256": digest(X),
                       "order": order, "round0_scores": scores[0].tolist(), "round_gaps": gaps,
                       "B": B.tolist() if X.shape[1] <= 100 else None,
                       # larger d: 40 target rows spread over the order (full B is d^2 doubles)
                       "B_rows": {int(order[p]): B[order[p]].tolist()
                                  for p in np.linspace(1, X.shape[1] - 1, 40).astype(int)}
                       if X.shape[1] > 100 else None,
                       "used_pinv": pinv,
                       "oracle_seconds": el, "oracle_workers": WORKERS}, f)
        print(name, "done", el, flush=True)


def make_full(name):
    """The oracle's exact pruned rounds (bit-identical order and winning k to its faithful
    mode, tests/test_oracle_kats.py) over the whole order of a large config."""
    X = config_input(name)
    t0 = time.time()
    order, wk, pairs, sk = oracle_lib.causal_order_pruned(X, workers=WORKERS, return_second=True)
    el = time.time() - t0
    n, d = X.shape
    with open(os.path.join(HERE, f"{name}_order_full.json"), "w") as f:
        json.dump({"config": name, "n": int(n), "d": int(d), "sha256": digest(X), "order": order,
                   "winner_k": [float(v).hex() for v in wk],
                   # lower bound of each round's runner-up k (exact when that row was fully
                   # evaluated): second_k - winner_k bounds the best-vs-second gap from below
                   "second_k": [float(v).hex() for v in sk],
                   "oracle": "orc_causal_order_pruned (exact branch and bound over the faithful "
                             "pair statistics; same order and winning k as orc_causal_order)",
                   "pairs_evaluated": int(pairs), "pairs_exhaustive": int(d * (d - 1) * (d + 1) // 6),
                   "oracle_seconds": el, "oracle_workers": WORKERS}, f)
    print(name, "full done", el, pairs, flush=True)


if __name__ == "__main__":
    main()
