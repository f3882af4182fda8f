"""H2D upload time of the host-buffer entry point (analysis): C5 from pinned and pageable memory."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2403_03772_b200 as plg  # noqa: E402

X = bench.make_input("c5")
n, d = X.shape
eng = plg.Engine(0)
pinned = torch.empty((d, n), dtype=torch.float64, pin_memory=True)
pinned.copy_(torch.from_numpy(np.ascontiguousarray(X.T)))
for name, A in (("pinned", pinned.numpy().T), ("pageable", np.asfortranarray(X))):
    for _ in range(3):
        eng.causal_order(A)
        st = eng.stats()
        print(name, "h2d_ms", round(st["h2d_ms"], 3), "GB/s", round(st["h2d_bytes"] / st["h2d_ms"] / 1e6, 1),
              "total_ms", round(st["total_ms"], 1), flush=True)
