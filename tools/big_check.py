"""Large-d robustness check (analysis tool, GPU box): pruned causal order at d=4000, n=5000 —
runs, returns a permutation, repeats bit-identically."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2403_03772_b200 as plg

d, n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000, int(sys.argv[2]) if len(sys.argv) > 2 else 5000
dag = plg.gen_sparse_dag(d, avg_parents=2.0, seed=7)
X = np.asfortranarray(plg.sample_lingam(dag, n, seed=7, kind="laplace"))
eng = plg.Engine(0)
t = time.time(); o1 = eng.causal_order(X); t1 = time.time() - t
k1 = eng.round_k(); s = eng.stats()
t = time.time(); o2 = eng.causal_order(X); t2 = time.time() - t
k2 = eng.round_k()
print({"d": d, "n": n, "perm": sorted(o1) == list(range(d)), "repeat_same": o1 == o2 and k1 == k2,
       "s_first": round(t1, 2), "s_second": round(t2, 2), "pairs_frac": s["pairs_evaluated"] / (s["pair_evals"] / 2)})
