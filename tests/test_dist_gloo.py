"""World-size 2 and 3 check of the multi-GPU exchange on CPU (gloo), no device needed.

The engine shards each round's pair tiles over ranks (plg_plan_round, the product's own
host schedule), every rank evaluates both residual entropies of its tiles into the packed
layout [tile][2][32][32] (epack[t][0][x][y] = E(a_x|b_y), epack[t][1][y][x] = E(b_y|a_x)),
and one all-gather of equal per-rank slots rebuilds the full table on every rank, which
then forms k and the lowest-index argmin locally. Here the per-pair
entropies come from the CPU oracle; the schedule, the slot placement of the all-gather and
the k/argmin assembly must reproduce the oracle's single-process search bit for bit, for
every world size.
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
BT = 32


class RoundPlan(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in
                ("nb", "ntiles", "tiles_per_rank", "tile_begin", "tile_count", "nseg", "seg_len", "replicated")]


def tile_index(bi, bj, nb):
    return bi * nb - (bi * (bi - 1)) // 2 + (bj - bi)


def pair_entropies(oracle, Z, ci, cj):
    """E(i|j), E(j|i) of standardised columns (ordering.cpp:86-92)."""
    e_ij = oracle.entropy_of_normalized(oracle.residual(Z[:, ci], Z[:, cj]))
    e_ji = oracle.entropy_of_normalized(oracle.residual(Z[:, cj], Z[:, ci]))
    return e_ij, e_ji


def kreduce(epack, H, u, nb):
    """k_p = sum_{q != p, ascending} min(0, M_pq)^2 read through the packed layout."""
    k = np.zeros(u)
    for p in range(u):
        bp, xp = divmod(p, BT)
        acc = 0.0
        for q in range(u):
            if q == p:
                continue
            bq, xq = divmod(q, BT)
            if bp < bq or (bp == bq and xp < xq):
                t = epack[tile_index(bp, bq, nb)]
                e_pq, e_qp = t[0, xp, xq], t[1, xq, xp]
            else:
                t = epack[tile_index(bq, bp, nb)]
                e_pq, e_qp = t[1, xp, xq], t[0, xq, xp]
            mi = (H[q] + e_pq) - (H[p] + e_qp)
            c = mi if mi < 0.0 else 0.0
            acc += c * c
        k[p] = acc
    return k


def _worker(rank, world, port, X, result_q):
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        lib = ctypes.CDLL(LIB)
        n, u = X.shape
        plan = RoundPlan()
        assert lib.plg_plan_round(u, n, rank, world, ctypes.byref(plan)) == 0
        Z = np.asfortranarray(np.stack([oracle.standardize(X[:, j]) for j in range(u)], axis=1))
        H = np.array([oracle.entropy_approx(Z[:, j]) for j in range(u)])
        slot = np.zeros((plan.tiles_per_rank, 2, BT, BT))
        for tl in range(plan.tile_count):
            bi, bj = ctypes.c_int32(), ctypes.c_int32()
            lib.plg_tile_decode(plan.tile_begin + tl, plan.nb, ctypes.byref(bi), ctypes.byref(bj))
            for x in range(BT):
                for y in range(BT):
                    i, j = bi.value * BT + x, bj.value * BT + y
                    if i >= u or j >= u or (bi.value == bj.value and x >= y):
                        continue
                    e_ij, e_ji = pair_entropies(oracle, Z, i, j)
                    slot[tl, 0, x, y] = e_ij
                    slot[tl, 1, y, x] = e_ji
        if plan.replicated:  # small round: every rank holds every tile, no exchange
            assert plan.tile_count == plan.ntiles
            epack = slot
        else:
            send = torch.from_numpy(slot.reshape(-1).copy())
            recv = [torch.zeros_like(send) for _ in range(world)]
            dist.all_gather(recv, send)  # the engine's in-place ncclAllGather of rank slots
            epack = torch.cat(recv).numpy().reshape(-1, 2, BT, BT)
        k = kreduce(epack, H, u, plan.nb)
        chosen = int(np.argmin(k))  # np.argmin returns the lowest index on ties
        result_q.put((rank, chosen, k.tobytes()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,d", [(2, 150), (3, 150), (2, 70)])
def test_sharded_round_matches_single_process(world, d, oracle):
    # d = 150: 5 position blocks -> 15 tiles, uneven over 2 ranks; d = 70 is a replicated
    # small round (u <= 128)
    rng = np.random.default_rng(11)
    n = 300
    X = np.asfortranarray(rng.uniform(-1, 1, size=(n, d)) + 0.5 * rng.laplace(size=(n, d)))
    chosen_ref, scores_ref = oracle.search_causal_order(X, list(range(d)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ks = {r: kb for r, _, kb in results}
    assert len(set(ks.values())) == 1  # every rank holds the identical k bits
    for _, chosen, kb in results:
        assert chosen == chosen_ref
        k = np.frombuffer(kb)
        assert (-k).tobytes() == scores_ref.tobytes()


def _peer_setup_worker(rank, world, port, q):
    # cli._setup_gpus' peer-memory path on CPU: the engine's init_peer is replaced by a stand-in
    # that hands its 64-byte "IPC handle" to the CLI's allgather and records what comes back
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys

    sys.path.insert(0, ROOT)
    from paper_2403_03772_b200 import cli

    got = {}

    def fake_init_peer(device, rnk, wld, max_dims, allgather):
        got.update(device=device, rank=rnk, world=wld, max_dims=max_dims,
                   handles=allgather(bytes([rnk]) * 64))

    cli._core.init_peer = fake_init_peer
    try:
        cli._setup_gpus(world, 37, "p2p")
        q.put((rank, got["device"], got["rank"], got["world"], got["max_dims"], [h[0] for h in got["handles"]],
               [len(h) for h in got["handles"]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_cli_peer_handle_exchange(world):
    # every rank must receive every rank's handle, in rank order, through the host channel
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_setup_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, device, rnk, wld, max_dims, firsts, lens in results:
        assert (device, rnk, wld, max_dims) == (rank, rank, world, 37)
        assert firsts == list(range(world)) and lens == [64] * world
