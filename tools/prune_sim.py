"""Feasibility study for an exact pruned round (analysis tool, runs on a GPU box).

Runs the engine's causal order with the round hook (plg_debug_set_round_hook), which hands
every round's full entropy table to this script, and simulates, on the true E of every
round, how many unordered pairs an exact branch-and-bound round would evaluate:

  1. full rows of the R candidates with the lowest predicted k  -> k* = min of their k
  2. each other candidate's T top predicted contributors (pairs)
  3. prune p when its partial k (evaluated pairs only) > k*
  4. surviving candidates: their top fraction f of predicted contributors, prune again
  5. survivors: full rows (exact k), argmin

Predictions use only what the device would know: the last evaluated contribution
min(0, M_pq)^2 of every pair (a d x d matrix updated with the pairs each round
evaluates; never-evaluated pairs predict 0).

    python tools/prune_sim.py --config c5 --out gpurun_out/prune_c5.json
"""

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HOOK = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                        ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_double),
                        ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double))


class Status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("row", ctypes.c_int64), ("col", ctypes.c_int64),
                ("msg", ctypes.c_char * 256)]


def topm(a, rows, m):
    """column indices of the m largest entries of a[rows] (unordered within the top m)."""
    m = min(m, a.shape[1])
    return np.argpartition(-a[rows], m - 1, axis=1)[:, :m]


class Strategy:
    def __init__(self, d, R, T, fracs):
        self.R, self.T, self.fracs = R, T, fracs
        self.known = np.zeros((d, d))  # last evaluated contribution of every pair (by variable)
        self.pairs = 0.0
        self.full = 0.0
        self.bad = 0

    def round(self, u, act, C, k, best):
        K = self.known[np.ix_(act, act)]
        pk = K.sum(1)
        ev = np.zeros((u, u), dtype=bool)
        top = np.argsort(pk, kind="stable")[: self.R]
        ev[top, :] = True
        ev[:, top] = True
        kstar = k[top].min()
        stg = [np.triu(ev, 1).sum()]
        rows = np.arange(u)
        sus = topm(K, rows, self.T)
        rr = np.repeat(rows, sus.shape[1])
        ev[rr, sus.ravel()] = True
        ev[sus.ravel(), rr] = True
        np.fill_diagonal(ev, False)
        margin = kstar * (1 + 1e-12)
        alive = np.where(ev, C, 0.0).sum(1) <= margin
        alive[top] = False
        na = [int(alive.sum())]
        stg.append(np.triu(ev, 1).sum())
        for f in self.fracs:
            rows = np.nonzero(alive)[0]
            if rows.size:
                cols = topm(K, rows, max(1, int(f * u)))
                rr = np.repeat(rows, cols.shape[1])
                ev[rr, cols.ravel()] = True
                ev[cols.ravel(), rr] = True
                np.fill_diagonal(ev, False)
                alive &= np.where(ev, C, 0.0).sum(1) <= margin
            stg.append(np.triu(ev, 1).sum())
            na.append(int(alive.sum()))
        rows = np.nonzero(alive)[0]
        ev[rows, :] = True
        ev[:, rows] = True
        np.fill_diagonal(ev, False)
        tot = np.triu(ev, 1).sum()
        stg.append(tot)
        if not (alive[best] or best in set(top.tolist())):
            self.bad += 1
        self.pairs += tot
        self.full += u * (u - 1) / 2
        # knowledge update: evaluated pairs only
        sub = self.known[np.ix_(act, act)]
        sub[ev] = C[ev]
        self.known[np.ix_(act, act)] = sub
        return {"frac": float(tot / (u * (u - 1) / 2)), "alive": na, "stages": [int(s) for s in stg],
                "kstar_over_kmin": float(kstar / k[best])}


class Sim:
    def __init__(self, d, strategies, every_log):
        self.d = d
        self.strategies = strategies
        self.every_log = every_log
        self.log = []

    def __call__(self, _user, rnd, u, act_p, E_p, H_p, k_p):
        if u <= 128:
            return
        act = np.ctypeslib.as_array(act_p, (u,)).copy()
        E = np.ctypeslib.as_array(E_p, (u * u,)).reshape(u, u)
        H = np.ctypeslib.as_array(H_p, (u,))
        k = np.ctypeslib.as_array(k_p, (u,)).copy()
        M = (H[None, :] + E) - (H[:, None] + E.T)
        np.fill_diagonal(M, 0.0)
        C = np.minimum(M, 0.0) ** 2
        best = int(np.argmin(k))
        res = [s.round(u, act, C, k, best) for s in self.strategies]
        if rnd % self.every_log == 0:
            self.log.append({"round": rnd, "u": u, "res": res})
            print(json.dumps(self.log[-1]), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--strategies", default="32:3:0.05,0.15;8:3:0.05,0.15;8:3:0.02,0.05,0.15;4:2:0.03,0.1")
    ap.add_argument("--every-log", type=int, default=100)
    ap.add_argument("--out", default="gpurun_out/prune_sim.json")
    args = ap.parse_args()
    import bench

    X = np.asfortranarray(bench.make_input(args.config))
    n, d = X.shape
    strategies = []
    for spec in args.strategies.split(";"):
        R, T, fr = spec.split(":")
        strategies.append(Strategy(d, int(R), int(T), [float(x) for x in fr.split(",")]))
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2403_03772_b200", "libplingam_b200.so"))
    st = Status()
    ctx = ctypes.c_void_p()
    assert lib.plg_ctx_create(0, ctypes.byref(ctx), ctypes.byref(st)) == 0, st.msg
    sim = Sim(d, strategies, args.every_log)
    cb = HOOK(sim)
    lib.plg_debug_set_round_hook(ctx, cb, None)
    order = (ctypes.c_int32 * d)()
    t0 = time.time()
    rc = lib.plg_causal_order(ctx, X.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.c_int64(n),
                              ctypes.c_int32(d), ctypes.c_int64(n), order, ctypes.byref(st))
    assert rc == 0, st.msg
    out = {"config": args.config, "d": d, "n": n, "seconds": time.time() - t0,
           "strategies": [{"spec": spec, "weighted_frac_pairs": s.pairs / s.full, "winner_lost": s.bad}
                          for spec, s in zip(args.strategies.split(";"), strategies)],
           "log": sim.log}
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["strategies"]))


if __name__ == "__main__":
    main()
