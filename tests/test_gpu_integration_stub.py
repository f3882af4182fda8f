"""INTEGRATION.md §3's ctypes stub, executed verbatim: the documented binding a maintainer
would paste into the reference's Python package must work against the built library."""

import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub_source() -> str:
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text.split("## 3. Python without a C++ rebuild (ctypes stub)", 1)[1]
    m = re.search(r"```python\n(.*?)```", sec, re.S)
    assert m, "INTEGRATION.md §3 has no python block"
    return m.group(1)


def test_stub_is_extractable():
    src = _stub_source()
    assert "plg_causal_order" in src and "plg_ctx_create" in src


@pytest.mark.gpu
def test_integration_ctypes_stub_verbatim(monkeypatch, plg):
    import oracle_lib

    monkeypatch.chdir(ROOT)  # the stub loads the library by its repo-relative path
    ns = {}
    exec(compile(_stub_source(), "INTEGRATION.md#3", "exec"), ns)
    dag = plg.gen_sparse_dag(30, avg_parents=2.0, seed=4)
    X = plg.sample_lingam(dag, 2000, seed=4, kind="laplace")
    assert ns["causal_order"](X) == oracle_lib.causal_order(X)
    bad = np.asfortranarray(X.copy())
    bad[5, 3] = np.nan
    with pytest.raises(RuntimeError, match=r"error 1 \(row 5, col 3\)"):
        ns["causal_order"](bad)


def _p2p_python_source() -> str:
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text.split("## 8. Multi-GPU through peer memory", 1)[1]
    blocks = re.findall(r"```python\n(.*?)```", sec, re.S)
    assert blocks, "INTEGRATION.md §8 has no python block"
    return blocks[0]


@pytest.mark.gpu
def test_integration_peer_memory_snippet_verbatim(plg):
    # INTEGRATION.md §8's Python block, as written, in a one-rank torch.distributed group
    import socket

    import torch.distributed as dist

    import oracle_lib

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        dag = plg.gen_sparse_dag(40, avg_parents=2.0, seed=8)
        X = plg.sample_lingam(dag, 3000, seed=8, kind="laplace")
        ns = {"local_rank": 0, "rank": 0, "world": 1, "d": 40, "X": X}
        exec(compile(_p2p_python_source(), "INTEGRATION.md#8", "exec"), ns)
        assert ns["order"] == oracle_lib.causal_order(X)
    finally:
        dist.destroy_process_group()
