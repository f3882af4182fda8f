"""Peer-memory multi-rank exchange (plg_ctx_create_p2p, include/plingam_b200.h).

Every exchange of a multi-rank causal order — round 0's entropy tiles and each pruned stage's
M values — is a store into every rank's arena plus a device-side flag barrier. Checked on one
B200 two ways:

* a one-rank peer context routes every exchange through its own arena (in-process): same
  order and winning-k bits as a local context, pruned and exhaustive rounds, search scores;
* two, three and four processes on the same GPU, each a rank of a world-2/3/4 context, arenas
  mapped across processes with CUDA IPC (the mechanism used between GPUs over NVLink), handles
  exchanged through files: every rank returns the single-rank order and winning-k bits (at
  four ranks with the multi-rank refinement ladder, which changes only which pairs are
  evaluated).
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _data(d, n, seed, kind="laplace"):
    import paper_2403_03772_b200 as plg

    dag = plg.gen_sparse_dag(d, avg_parents=2.0, seed=seed)
    return plg.sample_lingam(dag, n, seed=seed, kind=kind)


@pytest.mark.parametrize("prune", [True, False])
def test_p2p_self_exchange_matches_local(plg, prune):
    X = _data(260, 3000, 17)
    local = plg.Engine(0)
    peer = plg.Engine.peer(0, 0, 1, 300)
    for e in (local, peer):
        e.set_prune(prune)
    o_local = local.causal_order(X)
    k_local = [float(v).hex() for v in local.round_k()]
    for _ in range(4):  # direct, direct, graph capture, graph replay
        assert peer.causal_order(X) == o_local
        assert [float(v).hex() for v in peer.round_k()] == k_local
    c1, s1 = local.search(X, list(range(260)))
    c2, s2 = peer.search(X, list(range(260)))
    assert c1 == c2 and np.array_equal(np.asarray(s1), np.asarray(s2))


def test_p2p_arena_bounds(plg):
    peer = plg.Engine.peer(0, 0, 1, 50)
    with pytest.raises(plg.Error) as e:
        peer.causal_order(_data(60, 500, 3))
    assert e.value.code == "OutOfRange"


_RANK = r"""
import json, os, sys, time
sys.path.insert(0, %r)
import numpy as np
import paper_2403_03772_b200 as plg
rank, world, tmp, d, n, seed = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], %d, %d, %d
dag = plg.gen_sparse_dag(d, avg_parents=2.0, seed=seed)
X = plg.sample_lingam(dag, n, seed=seed, kind="laplace")
eng = plg.Engine.peer(0, rank, world, d)
with open(os.path.join(tmp, "h%%d.tmp" %% rank), "wb") as f:
    f.write(eng.p2p_handle())
os.replace(os.path.join(tmp, "h%%d.tmp" %% rank), os.path.join(tmp, "h%%d" %% rank))
handles = []
for r in range(world):
    p = os.path.join(tmp, "h%%d" %% r)
    t0 = time.time()
    while not os.path.exists(p):
        if time.time() - t0 > 120:
            raise SystemExit("no handle from rank %%d" %% r)
        time.sleep(0.05)
    handles.append(open(p, "rb").read())
eng.p2p_connect(handles)
out = []
for prune in (True, False):
    eng.set_prune(prune)
    order = eng.causal_order(X)
    out.append({"order": order, "k": [float(v).hex() for v in eng.round_k()]})
c, s = eng.search(X, list(range(d)))
out.append({"chosen": c, "scores": [float(v).hex() for v in s]})
# a device-side error mid-order (an exact duplicate column: the round after its twin is
# chosen raises ZeroVariance) must surface on every rank, collectively, without a hang
Xd = np.asfortranarray(X.copy())
Xd[:, d - 3] = Xd[:, 5]
try:
    eng.causal_order(Xd)
    out.append({"error": None})
except plg.Error as e:
    out.append({"error": e.code, "col": e.col})
order = eng.causal_order(X)  # the context stays usable
out.append({"after_error": order == out[0]["order"]})
print(json.dumps(out))
"""


@pytest.mark.parametrize("world", [2, 3, 4])
def test_p2p_ranks_across_processes(plg, tmp_path, world):
    d, n, seed = 200, 2000, 29
    src = _RANK % (ROOT, d, n, seed)
    procs = [subprocess.Popen([sys.executable, "-c", src, str(r), str(world), str(tmp_path)],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(world)]
    outs = []
    for p in procs:
        try:
            so, se = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        assert p.returncode == 0, se[-2000:]
        outs.append(json.loads(so.strip().splitlines()[-1]))
    X = _data(d, n, seed)
    local = plg.Engine(0)
    ref = []
    for prune in (True, False):
        local.set_prune(prune)
        ref.append({"order": local.causal_order(X), "k": [float(v).hex() for v in local.round_k()]})
    c, s = local.search(X, list(range(d)))
    ref.append({"chosen": c, "scores": [float(v).hex() for v in s]})
    Xd = np.asfortranarray(X.copy())
    Xd[:, d - 3] = Xd[:, 5]
    with pytest.raises(plg.Error) as e:
        local.causal_order(Xd)
    ref.append({"error": e.value.code, "col": e.value.col})
    ref.append({"after_error": True})
    for out in outs:
        assert out == ref


def test_bench_two_ranks_on_one_gpu(tmp_path):
    # bench.py's multi-rank path end to end under torchrun (peer-memory exchange across the two
    # processes, max-over-ranks timing, one JSON line from rank 0), both ranks sharing cuda:0
    # through the PLG_BENCH_SHARED_GPU test hook (a gloo process group instead of NCCL)
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, PLG_BENCH_SHARED_GPU="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--config", "c4", "--steps", "1", "--warmup", "3", "--no-ncu"],
                         env=env, capture_output=True, text=True, timeout=900, cwd=str(tmp_path))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and "peer memory" in rec["config"]["parallelism"]
    assert rec["pruning"]["fraction_evaluated"] < 0.2 and rec["e2e"]["h2d_bytes_per_step"] > 0
    assert out.stderr.count("peer-memory exchange") == 2


def test_p2p_two_ranks_c3_golden(tmp_path):
    # a BASELINE config through the peer-memory exchange across two processes (sharing cuda:0):
    # every rank's whole C3 order and every round's winning k against the committed golden
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(ROOT, "tools", "p2p_scale_check.py"), "--config", "c3", "--shared-gpu"],
                         capture_output=True, text=True, timeout=900, cwd=str(tmp_path))
    assert out.returncode == 0, out.stderr[-3000:]
    rec = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert rec["all_ok"] and rec["k_bits_equal_across_ranks"], rec
