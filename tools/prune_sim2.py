"""Pruning-policy simulator on the true per-round tables (analysis tool, runs on a GPU box).

Like prune_sim.py (the engine's round hook hands every round's full entropy table to this
script), but it simulates the product's policy and finer "stepwise" policies side by side:

  ladder  the product's round: R top rows' full rows (k* = min of their exact k), each
          other row's T strongest predicted partners, then refinement stages at cumulative
          fractions of the row, each taking min(deficit cut, fraction step) partners
          (deficit cut: strongest predicted partners until their predicted sum reaches
          beta x (k* - L_p); all remaining partners if the prediction falls short), then
          full rows for the survivors
  screen  the ladder's probe (exact), then refinement stages whose pairs are screened: a
          screened pair gives row p only min(0, M_pq + W)^2 (W: the screening kernel's error
          bound, constant here), then optionally a screened full stage (every remaining
          partner of the alive rows), then the exact full stage (rows still alive: every
          partner not yet exact). Spec screen:R:T:fracs:beta:W:sfull
  step    after the same probe, every alive row takes its strongest unevaluated predicted
          partners in steps of at most S (deficit cut, at least s_min; S when the predictions
          fall short of the deficit) and is re-tested after each step, until it is pruned or
          complete

Reports the fraction of the exhaustive rounds' pairs each policy evaluates and how many
sequential steps (stages) it needs per round.

    python tools/prune_sim2.py --config c5 --out gpurun_out/prune_sim2_c5.json
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
sys.path.insert(0, os.path.join(ROOT, "tools"))

from prune_sim import HOOK, Status  # noqa: E402

SLACK = 1e-9


class Policy:
    def __init__(self, d, spec):
        self.spec = spec
        kind, rest = spec.split(":", 1)
        self.kind = kind
        vals = rest.split(":")
        self.R, self.T = int(vals[0]), int(vals[1])
        if kind in ("ladder", "screen"):
            self.fracs = [float(x) for x in vals[2].split(",")]
            self.beta = float(vals[3]) if len(vals) > 3 else 1.1
            self.W = float(vals[4]) if len(vals) > 4 else 0.0
            self.sfull = int(vals[5]) if len(vals) > 5 else 0
        else:
            self.S, self.smin = int(vals[2]), int(vals[3])
            self.beta = float(vals[4]) if len(vals) > 4 else 1.1
        self.known = np.zeros((d, d))
        self.pairs = 0.0
        self.full = 0.0
        self.stages = 0
        self.rounds = 0
        self.bad = 0
        self.scr = 0.0  # screened pairs (screen policy)

    def _take(self, order_row, K_row, ev_row, need, cap):
        """strongest unevaluated partners (order_row: partner indices by prediction, strongest
        first) until their predicted sum reaches need, at most cap; all if it falls short."""
        cand = order_row[~ev_row[order_row]]
        if cand.size == 0:
            return cand
        cs = np.cumsum(K_row[cand])
        if cs[-1] < need:  # predictions fall short of the deficit: the step's cap
            return cand[:cap]
        c = int(np.searchsorted(cs, need)) + 1
        return cand[: min(c, cap)]

    def round(self, u, act, C, k, best):
        K = self.known[np.ix_(act, act)].copy()
        np.fill_diagonal(K, 0.0)
        pk = K.sum(1)
        ev = np.zeros((u, u), dtype=bool)
        top = np.argsort(pk, kind="stable")[: self.R]
        ev[top, :] = True
        ev[:, top] = True
        np.fill_diagonal(ev, False)
        kstar = k[top].min()
        thr = kstar * (1 + SLACK)
        rows = np.setdiff1d(np.arange(u), top)
        Kt = K.copy()
        Kt[:, top] = -1.0
        sus = np.argsort(-Kt[rows], axis=1, kind="stable")[:, : self.T]
        rr = np.repeat(rows, sus.shape[1])
        ev[rr, sus.ravel()] = True
        ev[sus.ravel(), rr] = True
        np.fill_diagonal(ev, False)
        L = np.where(ev, C, 0.0).sum(1)
        alive = L <= thr
        alive[top] = False
        stages = 1
        if self.kind == "screen":
            Mrow = self.M  # row p's M_pq
            Cs = np.minimum(Mrow + self.W, 0.0) ** 2  # lower bound of row p's contribution from a screened pair
            sc = np.zeros((u, u), dtype=bool)

            def lower():
                return np.where(ev, C, np.where(sc, Cs, 0.0)).sum(1)

            prev = 0.0
            for f in self.fracs:
                idx = np.nonzero(alive)[0]
                if idx.size:
                    cap = max(1, int((f - prev) * u))
                    orders = np.argsort(-K[idx], axis=1, kind="stable")
                    done = ev | sc
                    for i, pp in enumerate(idx):
                        sel = self._take(orders[i], K[pp], done[pp], self.beta * (thr - L[pp]), cap)
                        sel = sel[sel != pp]
                        sc[pp, sel] = True
                        sc[sel, pp] = True
                    np.fill_diagonal(sc, False)
                    L = lower()
                    alive &= L <= thr
                stages += 1
                prev = f
            if self.sfull:
                idx = np.nonzero(alive)[0]
                sc[idx, :] = True
                sc[:, idx] = True
                np.fill_diagonal(sc, False)
                L = lower()
                alive &= L <= thr
                stages += 1
            idx = np.nonzero(alive)[0]
            ev[idx, :] = True
            ev[:, idx] = True
            np.fill_diagonal(ev, False)
            stages += 1
            self.scr += np.triu(sc & ~ev, 1).sum() + np.triu(sc & ev, 1).sum()
            ev_all = ev | sc
        elif self.kind == "ladder":
            prev = 0.0
            for f in self.fracs:
                idx = np.nonzero(alive)[0]
                if idx.size:
                    cap = max(1, int((f - prev) * u))
                    orders = np.argsort(-K[idx], axis=1, kind="stable")
                    for i, p in enumerate(idx):
                        sel = self._take(orders[i], K[p], ev[p], self.beta * (thr - L[p]), cap)
                        ev[p, sel] = True
                        ev[sel, p] = True
                    np.fill_diagonal(ev, False)
                    L = np.where(ev, C, 0.0).sum(1)
                    alive &= L <= thr
                stages += 1
                prev = f
            idx = np.nonzero(alive)[0]
            ev[idx, :] = True
            ev[:, idx] = True
            np.fill_diagonal(ev, False)
            stages += 1
        else:
            idx = np.nonzero(alive)[0]
            orders = {int(p): o for p, o in zip(idx, np.argsort(-K[idx], axis=1, kind="stable"))} if idx.size else {}
            while True:
                idx = np.nonzero(alive & ~ev.all(1, where=~np.eye(u, dtype=bool)))[0]
                if not idx.size:
                    break
                for p in idx:
                    sel = self._take(orders[int(p)], K[p], ev[p], self.beta * (thr - L[p]), self.S)
                    if sel.size < self.smin:
                        cand = orders[int(p)][~ev[p, orders[int(p)]]]
                        cand = cand[cand != p]
                        sel = cand[: self.smin]
                    ev[p, sel] = True
                    ev[sel, p] = True
                np.fill_diagonal(ev, False)
                L = np.where(ev, C, 0.0).sum(1)
                alive &= L <= thr
                stages += 1
                if stages > 10000:
                    break
        if self.kind != "screen":
            ev_all = ev
        tot = np.triu(ev, 1).sum()
        full_rows = ev.sum(1) == u - 1
        if not (full_rows[best] or best in set(top.tolist())):
            self.bad += 1
        self.pairs += tot
        self.full += u * (u - 1) / 2
        self.stages += stages
        self.rounds += 1
        sub = self.known[np.ix_(act, act)]
        sub[ev_all] = C[ev_all]
        self.known[np.ix_(act, act)] = sub
        return {"frac": float(tot / (u * (u - 1) / 2)), "stages": stages}


class Sim:
    def __init__(self, d, policies, every_log):
        self.policies = policies
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
        for p in self.policies:
            p.M = M
        res = [p.round(u, act, C, k, best) for p in self.policies] if rnd > 0 else []
        if rnd == 0:  # round 0 is exhaustive in the product: every pair becomes known
            for p in self.policies:
                sub = p.known[np.ix_(act, act)]
                sub[:] = C
                p.known[np.ix_(act, act)] = sub
        if rnd % self.every_log == 0:
            self.log.append({"round": rnd, "u": u, "res": res})
            print(json.dumps(self.log[-1]), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--policies", default="ladder:3:1:0.05,0.25;step:3:1:64:8;step:3:1:32:4;step:3:1:16:2")
    ap.add_argument("--every-log", type=int, default=100)
    ap.add_argument("--max-rounds", type=int, default=-1)
    ap.add_argument("--out", default="gpurun_out/prune_sim2.json")
    args = ap.parse_args()
    import bench

    X = np.asfortranarray(bench.make_input(args.config))
    n, d = X.shape
    policies = [Policy(d, s) for s in args.policies.split(";")]
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2403_03772_b200", "libplingam_b200.so"))
    st = Status()
    ctx = ctypes.c_void_p()
    assert lib.plg_ctx_create(0, ctypes.byref(ctx), ctypes.byref(st)) == 0, st.msg
    sim = Sim(d, policies, args.every_log)
    cb = HOOK(sim)
    lib.plg_debug_set_round_hook(ctx, cb, None)
    t0 = time.time()
    if args.max_rounds > 0:  # the first rounds only (the large-u rounds hold most of the work)
        act = np.zeros(d, dtype=np.int32)
        na = ctypes.c_int32(0)
        cols = np.zeros((n, d), order="F")
        pref = np.zeros(d, dtype=np.int32)
        I = ctypes.POINTER(ctypes.c_int32)
        rc = lib.plg_round_state(ctx, X.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.c_int64(n),
                                 ctypes.c_int32(d), ctypes.c_int64(n), ctypes.c_int32(args.max_rounds),
                                 act.ctypes.data_as(I), ctypes.byref(na),
                                 cols.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), pref.ctypes.data_as(I),
                                 ctypes.byref(st))
    else:
        order = (ctypes.c_int32 * d)()
        rc = lib.plg_causal_order(ctx, X.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.c_int64(n),
                                  ctypes.c_int32(d), ctypes.c_int64(n), order, ctypes.byref(st))
    assert rc == 0, st.msg
    out = {"config": args.config, "d": d, "n": n, "seconds": time.time() - t0,
           "policies": [{"spec": p.spec, "weighted_frac_pairs": p.pairs / max(p.full, 1),
                         "exact_pairs": float(p.pairs), "screened_pairs": float(p.scr),
                         "stages_per_round": p.stages / max(p.rounds, 1), "winner_lost": p.bad}
                        for p in policies],
           "log": sim.log}
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["policies"]))


if __name__ == "__main__":
    main()
