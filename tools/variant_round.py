"""Time one C5 search round with a package variant directory first on sys.path.
    python tools/variant_round.py <variant_dir> [reps]"""
import os
import sys

variant = os.path.abspath(sys.argv[1])
sys.path.insert(0, variant)
import paper_2403_03772_b200 as plg  # noqa: E402

assert plg.__file__.startswith(variant), plg.__file__
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

X = bench.make_input("c5")
eng = plg.Engine(0)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    eng.search(X, list(range(X.shape[1])))
    print(variant, eng.stats()["pair_ms"], flush=True)
