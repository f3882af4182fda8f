"""Oracle lower bound of the pairs an exact row-pruning round must evaluate (analysis tool).

With perfect knowledge of the round's contributions C_pq = min(0, M_pq)^2 and of k* = min k,
row p != winner needs its m_p largest contributions to exceed k*; the winner needs its full
row. The bound counts the distinct unordered pairs of those sets per round.

    python tools/prune_bound.py --config c5 --every 20
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from prune_sim import HOOK, Status  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--every", type=int, default=20)
    args = ap.parse_args()
    import bench

    X = np.asfortranarray(bench.make_input(args.config))
    n, d = X.shape
    tot = {"bound": 0.0, "full": 0.0}
    rows = []

    def cb(_u, rnd, u, act_p, E_p, H_p, k_p):
        if rnd % args.every or u <= 128:
            return
        E = np.ctypeslib.as_array(E_p, (u * u,)).reshape(u, u)
        H = np.ctypeslib.as_array(H_p, (u,))
        k = np.ctypeslib.as_array(k_p, (u,)).copy()
        M = (H[None, :] + E) - (H[:, None] + E.T)
        np.fill_diagonal(M, 0.0)
        C = np.minimum(M, 0.0) ** 2
        w = int(np.argmin(k))
        kstar = k[w]
        Cs = -np.sort(-C, axis=1)
        cs = np.cumsum(Cs, axis=1)
        need = (cs > kstar * (1 + 1e-9)).argmax(axis=1) + 1  # rows whose full sum never exceeds: argmax 0
        order = np.argsort(-C, axis=1, kind="stable")
        ev = np.zeros((u, u), dtype=bool)
        for p in range(u):
            if p == w or cs[p, -1] <= kstar * (1 + 1e-9):
                ev[p, :] = True
            else:
                ev[p, order[p, : need[p]]] = True
        ev |= ev.T
        np.fill_diagonal(ev, False)
        b = np.triu(ev, 1).sum()
        full = u * (u - 1) / 2
        tot["bound"] += b
        tot["full"] += full
        rows.append({"round": rnd, "u": u, "frac": b / full, "median_need": float(np.median(need))})

    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2403_03772_b200", "libplingam_b200.so"))
    st = Status()
    ctx = ctypes.c_void_p()
    assert lib.plg_ctx_create(0, ctypes.byref(ctx), ctypes.byref(st)) == 0
    f = HOOK(cb)
    lib.plg_debug_set_round_hook(ctx, f, None)
    order = (ctypes.c_int32 * d)()
    assert lib.plg_causal_order(ctx, X.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.c_int64(n),
                                ctypes.c_int32(d), ctypes.c_int64(n), order, ctypes.byref(st)) == 0
    print(json.dumps({"config": args.config, "bound_frac": tot["bound"] / tot["full"], "rounds": rows[::10]}))


if __name__ == "__main__":
    main()
