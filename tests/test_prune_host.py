"""Host-side checks of the exact pruned rounds (no device needed).

1. The branch-and-bound logic of prune_kernels.cu restated in numpy: stages (probe with R
   full rows + T predicted suspects, refinement ladder, full rows for the survivors), the
   prune test L_p > k* (1 + 1e-9) and the lowest-position argmin over the rows with exact
   k. On random, tied and adversarial contribution tables the pruned argmin must equal the
   exhaustive argmin, whatever the predictions are (exactness does not depend on them).
2. The multi-rank schedule of a pruned stage on gloo (world 2 and 3): the product's slice
   plan (plg_plan_list_shard), one all-gather of equal slots and the scatter by list index
   rebuild the single-process table bit for bit.
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2403_03772_b200", "libplingam_b200.so")
SLACK = 1e-9  # prune_kernels.cu kPruneSlack


def k_exact(M, p):
    """kreduce_kernel's value (order is irrelevant here: float sums of the same terms)."""
    c = np.minimum(M[p], 0.0)
    c[p] = 0.0
    return float(np.sum(c * c))


def pruned_argmin(M, pred, R=3, T=1, fracs=(0.03, 0.1, 0.3)):
    """numpy restatement of search_round_pruned (engine.cu) on a full M table.

    pred[p, q] >= 0 plays KN (the predictions). Returns (winner, evaluated mask)."""
    u = M.shape[0]
    ev = np.zeros((u, u), dtype=bool)

    def evaluate(p, qs):
        for q in qs:
            if q != p:
                ev[p, q] = ev[q, p] = True

    def partial(p):
        c = np.where(ev[p], np.minimum(M[p], 0.0), 0.0)
        return float(np.sum(c * c))

    def strongest(p, cand, m):
        cand = [q for q in cand if q != p and not ev[p, q]]
        cand.sort(key=lambda q: (-pred[p, q], q))
        return cand[:m]

    pk = np.array([sum(pred[p, q] for q in range(u) if q != p) for p in range(u)])
    top = sorted(range(u), key=lambda p: (pk[p], p))[: min(R, u)]
    state = np.ones(u, dtype=int)
    state[top] = 2
    for p in range(u):  # probe
        if state[p] == 2:
            evaluate(p, range(u))
        else:
            evaluate(p, strongest(p, [q for q in range(u) if state[q] != 2], T))
    kstar = min(k_exact(M, p) for p in top)
    thr = kstar * (1 + SLACK)
    prev = 0.0
    for f in fracs:  # refinement (count mode)
        m = max(1, int((f - prev) * u))
        prev = f
        for p in range(u):
            if state[p] == 1:
                if partial(p) > thr:
                    state[p] = 0
                else:
                    evaluate(p, strongest(p, range(u), m))
    for p in range(u):  # full
        if state[p] == 1:
            if partial(p) > thr:
                state[p] = 0
            else:
                evaluate(p, range(u))
    k = np.array([k_exact(M, p) if state[p] >= 1 else np.inf for p in range(u)])
    for p in range(u):
        if state[p] >= 1:
            assert ev[p].sum() == u - 1  # an exact k needs the full row
        else:
            assert k_exact(M, p) > kstar  # a pruned row cannot win or tie
    return int(np.argmin(k)), ev


def exhaustive_argmin(M):
    return int(np.argmin([k_exact(M, p) for p in range(M.shape[0])]))


def antisym(rng, u, scale):
    A = rng.normal(scale=scale, size=(u, u))
    M = np.triu(A, 1)
    return M - M.T


@pytest.mark.parametrize("seed", range(12))
def test_pruned_argmin_equals_exhaustive_random(seed):
    rng = np.random.default_rng(seed)
    u = int(rng.integers(8, 40))
    M = antisym(rng, u, 1e-3)
    # a few "roots": rows with no negative entries against most others
    for r in rng.choice(u, size=max(1, u // 5), replace=False):
        M[r] = np.abs(M[r]) * rng.uniform(0.0, 0.2)
        M[:, r] = -M[r]
    np.fill_diagonal(M, 0.0)
    C = np.minimum(M, 0.0) ** 2
    for pred in (C, C[rng.permutation(u)][:, rng.permutation(u)], np.zeros_like(C), rng.uniform(size=C.shape)):
        w, ev = pruned_argmin(M, pred)
        assert w == exhaustive_argmin(M)


def test_pruned_argmin_ties_pick_lowest_position():
    u = 12
    M = np.zeros((u, u))  # every k = 0: the lowest position must win
    assert pruned_argmin(M, np.zeros((u, u)))[0] == 0
    rng = np.random.default_rng(5)
    M = antisym(rng, u, 1e-2)
    # rows 3 and 7 get identical k (mirror images), both better than everyone else
    for r in (3, 7):
        M[r] = np.abs(M[r])
        M[:, r] = -M[r]
    M[3, 7] = M[7, 3] = 0.0
    np.fill_diagonal(M, 0.0)
    assert k_exact(M, 3) == k_exact(M, 7) == 0.0
    C = np.minimum(M, 0.0) ** 2
    assert pruned_argmin(M, C)[0] == exhaustive_argmin(M) == 3


def test_pruning_near_tie_is_not_pruned():
    # a row whose k exceeds k* by far less than the slack must survive to its exact k
    rng = np.random.default_rng(9)
    u = 10
    M = antisym(rng, u, 1e-3)
    np.fill_diagonal(M, 0.0)
    ks = [k_exact(M, p) for p in range(u)]
    w = int(np.argmin(ks))
    w, ev = pruned_argmin(M, np.minimum(M, 0.0) ** 2, R=1)
    assert w == exhaustive_argmin(M)


def test_pruning_saves_pairs_with_good_predictions():
    rng = np.random.default_rng(2)
    u = 60
    M = antisym(rng, u, 1e-2)
    np.fill_diagonal(M, 0.0)
    C = np.minimum(M, 0.0) ** 2
    w, ev = pruned_argmin(M, C)
    assert w == exhaustive_argmin(M)
    assert np.triu(ev, 1).sum() < 0.6 * u * (u - 1) / 2


# ---------------------------------------------------------------- multi-rank schedule (gloo)

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard(total, rank, world):
    lib = ctypes.CDLL(LIB)
    b, e, slot = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    assert lib.plg_plan_list_shard(total, rank, world, ctypes.byref(b), ctypes.byref(e), ctypes.byref(slot)) == 0
    return b.value, e.value, slot.value


def _stage_worker(rank, world, port, total, u, out, bound=None):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(123)  # every rank builds the same list (deterministic selection)
        pairs = [(int(p), int(q)) for p, q in rng.integers(0, u, size=(total, 2)) if p != q][:total]
        total_eff = len(pairs)
        if bound is None:  # host-planned slice (the full stage): plg_plan_list_shard
            b, e, slot = _shard(total_eff, rank, world)
            base = b
        else:  # device-planned slice, fixed slot of ceil(bound / world) (probe / refinement)
            cnt = (total_eff + world - 1) // world
            b, e = min(total_eff, rank * cnt), min(total_eff, (rank + 1) * cnt)
            slot = (bound + world - 1) // world
            base = rank * slot
        res = torch.zeros(slot * world, dtype=torch.float64)
        for k in range(b, e):  # this rank's slice: "evaluate" entry k into its slot
            p, q = pairs[k]
            res[base + (k - b)] = np.sin(1.0 + p * 0.37 + q * 0.011)  # any deterministic function
        mine = res[rank * slot:(rank + 1) * slot].clone()
        gathered = [torch.zeros(slot, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, mine)
        full = torch.cat(gathered).numpy()
        cnt = max(1, (total_eff + world - 1) // world)
        Md = np.full((u, u), np.nan)
        for k, (p, q) in enumerate(pairs):  # prune_scatter_kernel: entry k at (k / cnt) slot + k % cnt
            v = full[(k // cnt) * slot + k % cnt]
            Md[p, q], Md[q, p] = v, -v
        if rank == 0:
            np.save(out, Md)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,total,bound", [(2, 1000, None), (3, 1001, None), (3, 2, None), (2, 0, None),
                                               (2, 700, 1200), (3, 1001, 1001), (3, 5, 64)])
def test_pruned_stage_shard_gather_scatter(tmp_path, world, total, bound):
    u = 50
    out = str(tmp_path / "md.npy")
    mp.spawn(_stage_worker, args=(world, _free_port(), total, u, out, bound), nprocs=world, join=True)
    rng = np.random.default_rng(123)
    pairs = [(int(p), int(q)) for p, q in rng.integers(0, u, size=(total, 2)) if p != q][:total]
    ref = np.full((u, u), np.nan)
    for p, q in pairs:
        v = np.sin(1.0 + p * 0.37 + q * 0.011)
        ref[p, q], ref[q, p] = v, -v
    got = np.load(out)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    assert np.array_equal(got[~np.isnan(ref)], ref[~np.isnan(ref)])
    # the slices tile [0, total) exactly
    spans = [_shard(len(pairs), r, world)[:2] for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == len(pairs)
    assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
