"""Golden adjacency weights B for the large configs C3 and C5 (run here, on CPU).

B is d x d and dense below the causal order (every predecessor gets an OLS coefficient,
direct_lingam.cpp:46-70), so the fixture stores, for the committed golden order:
  * full B rows of a few targets spread over the order, computed by the FAITHFUL route —
    one column-pivoted Householder QR per target (orc_fit_weights_targets, the restatement
    of Eigen::ColPivHouseholderQR + CompleteOrthogonalDecomposition);
  * the L2 norm of every B row from the prefix-QR oracle (orc_fit_weights_prefix: one QR of
    the order-permuted centred design, the O(n d^2) reference for large d), after checking
    the prefix oracle against the faithful rows here (max relative difference recorded).
The GPU test compares the device B with the live prefix oracle (every entry) and with these
rows and norms.

    python tests/golden/make_weights_golden.py c3 c5
"""

import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import make_golden as MG  # noqa: E402
import oracle_lib  # noqa: E402

POSITIONS = {"c3": [1, 2, 10, 100, 333, 500, 750, 999], "c5": [1, 2, 10, 100, 500, 1000, 1500, 1999]}


def make(name: str, workers: int) -> None:
    X = np.asfortranarray(MG.config_input(name))
    g = json.load(open(os.path.join(HERE, f"{name}_order_full.json")))
    assert MG.digest(X) == g["sha256"], "input differs from the golden order's input"
    order = g["order"]
    d = X.shape[1]
    t0 = time.time()
    B_pre, pinv_pre, ndep = oracle_lib.fit_weights_prefix(X, order, workers=workers)
    t_pre = time.time() - t0
    pos = POSITIONS[name]
    t0 = time.time()
    with ThreadPoolExecutor(workers) as ex:  # ctypes releases the GIL: one target per thread
        parts = list(ex.map(lambda p: oracle_lib.fit_weights_targets(X, order, [p]), pos))
    t_faith = time.time() - t0
    rows, worst = {}, 0.0
    for p, (Bp, _) in zip(pos, parts):
        t = order[p]
        rows[str(p)] = {"target": int(t), "row": [float(v).hex() for v in Bp[t]]}
        scale = np.maximum(1.0, np.abs(Bp[t]))
        worst = max(worst, float(np.max(np.abs(B_pre[t] - Bp[t]) / scale)))
    assert worst < 1e-9, f"prefix-QR oracle vs per-target QR: {worst}"
    out = {
        "config": name, "n": int(X.shape[0]), "d": int(d), "sha256": g["sha256"],
        "order_from": f"{name}_order_full.json",
        "faithful_rows": rows,
        "prefix_row_norms": [float(v).hex() for v in np.linalg.norm(B_pre, axis=1)],
        "prefix_used_pinv": bool(pinv_pre), "prefix_dependent_columns": int(ndep),
        "prefix_vs_faithful_max_rel": worst,
        "seconds": {"prefix": t_pre, "faithful_rows": t_faith}, "workers": workers,
    }
    with open(os.path.join(HERE, f"{name}_weights.json"), "w") as f:
        json.dump(out, f)
    print(name, "weights golden done", out["seconds"], "max rel", worst, flush=True)


if __name__ == "__main__":
    w = int(os.environ.get("GOLDEN_WORKERS", os.cpu_count() or 1))
    for name in sys.argv[1:] or ["c3", "c5"]:
        make(name, w)
