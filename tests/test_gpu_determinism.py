"""Determinism contracts of the engine (the reference's seq == par bit identity,
test_ordering.cpp:148-179, restated for the GPU): every k bit is a pure function of the data
and (u, n), independent of the pair-kernel thread geometry and tile schedule, of repeated
runs, and of host vs device entry points."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_2403_03772_b200 as plg
dag = plg.gen_sparse_dag(150, avg_parents=2.0, seed=12)
X = plg.sample_lingam(dag, 3000, seed=12, kind="laplace")
eng = plg.Engine(0)
order = eng.causal_order(X)
c, s = eng.search(X, list(range(150)))
print(json.dumps({"order": order, "scores": [float(v).hex() for v in s]}))
"""


def _run(geom):
    env = dict(os.environ, PLG_PAIR_GEOM=geom)
    out = subprocess.run([sys.executable, "-c", _CHILD % ROOT], env=env, capture_output=True, text=True,
                         check=True, timeout=600)
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_bits_independent_of_thread_geometry():
    a = _run("22d")
    b = _run("12")
    assert a["order"] == b["order"]
    assert a["scores"] == b["scores"]  # bit-identical k for every candidate


def test_repeat_runs_bit_identical(engine, plg):
    dag = plg.gen_sparse_dag(80, avg_parents=2.0, seed=4)
    X = plg.sample_lingam(dag, 5000, seed=4, kind="laplace")
    c1, s1 = engine.search(X, list(range(80)))
    c2, s2 = engine.search(X, list(range(80)))
    assert c1 == c2 and np.asarray(s1).tobytes() == np.asarray(s2).tobytes()
    assert engine.causal_order(X) == engine.causal_order(X)


_GRAPH_CHILD = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
import paper_2403_03772_b200 as plg
eng = plg.Engine(0)
out = []
for seed in (21, 22, 23, 24, 25, 26):  # one shape: calls 1-2 run directly, 3 captures, 4-6 replay
    dag = plg.gen_sparse_dag(220, avg_parents=2.0, seed=seed)
    X = plg.sample_lingam(dag, 2500, seed=seed, kind="laplace")
    order = eng.causal_order(X)
    out.append({"order": order, "k": [float(v).hex() for v in eng.round_k()],
                "launches": eng.stats()["launches"], "pairs": eng.stats()["pairs_evaluated"]})
print(json.dumps(out))
"""


def test_graph_replay_matches_direct_launches():
    # The round loop is captured into a CUDA graph on the second call of a shape and replayed
    # afterwards (engine.cu run_rounds_graph): every call, on different data of one shape,
    # must give the bits of the directly launched loop (PLG_GRAPHS=0), and the same stats.
    runs = {}
    for g in ("0", "1"):
        env = dict(os.environ, PLG_GRAPHS=g)
        out = subprocess.run([sys.executable, "-c", _GRAPH_CHILD % ROOT], env=env, capture_output=True, text=True,
                             check=True, timeout=900)
        runs[g] = json.loads(out.stdout.strip().splitlines()[-1])
    assert runs["0"] == runs["1"]
