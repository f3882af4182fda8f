"""CLI: argument handling and exit codes on CPU
(plingam_cli.cpp:363-374), end-to-end discover / var-discover on the GPU."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, cwd):
    p = subprocess.run([sys.executable, "-m", "paper_2403_03772_b200", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    return p.returncode, p.stdout, p.stderr


def test_cli_usage_and_io_errors(tmp_path):
    rc, _, err = run(["discover"], tmp_path)
    assert rc == 1 and "--input" in err
    rc, _, err = run(["discover", "--input", str(tmp_path / "missing.csv")], tmp_path)
    assert rc == 2 and "IoError" in err
    rc, _, err = run(["var-discover", "--input", "x.csv", "--lag", "0"], tmp_path)
    assert rc == 1 and "InvalidFlags" in err
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b\n1,2\n3,\n")
    rc, _, err = run(["discover", "--input", str(bad)], tmp_path)
    assert rc == 2 and "ParseError" in err


@pytest.mark.gpu
def test_cli_discover_csv_and_binary(tmp_path, plg):
    dag = plg.gen_two_level_dag(8, seed=3)
    X = plg.sample_lingam(dag, 4000, seed=3)
    csv = tmp_path / "data.csv"
    with open(csv, "w") as f:
        f.write(",".join(f"x{j}" for j in range(8)) + "\n")
        for row in X:
            f.write(",".join("%.17g" % v for v in row) + "\n")
    rc, out, err = run(["discover", "--input", str(csv), "--out", str(tmp_path / "a")], tmp_path)
    assert rc == 0, err
    rep = json.loads(out.strip().splitlines()[-1])
    assert rep["order"] == plg.causal_order(X) and rep["dims"] == 8 and rep["samples"] == 4000
    assert len(rep["manifest"]["input_digest"]) == 16
    B = np.loadtxt(tmp_path / "a" / "adjacency.csv", delimiter=",", skiprows=1)
    assert np.allclose(B, plg.fit_direct_lingam(X).weights, rtol=1e-12, atol=1e-15)
    order = [int(v) for v in open(tmp_path / "a" / "order.txt").read().split()]
    assert order == rep["order"]
    npy = tmp_path / "data.npy"
    np.save(npy, X)
    rc, out, err = run(["discover", "--input", str(npy), "--out", str(tmp_path / "b")], tmp_path)
    assert rc == 0, err
    assert json.loads(out.strip().splitlines()[-1])["order"] == rep["order"]
    raw = tmp_path / "data.f64"
    np.asfortranarray(X).T.tofile(raw)  # column-major bytes
    rc, out, err = run(["discover", "--input", str(raw), "--dims", "8", "--colmajor", "--out",
                        str(tmp_path / "c")], tmp_path)
    assert rc == 0, err
    assert json.loads(out.strip().splitlines()[-1])["order"] == rep["order"]


@pytest.mark.gpu
def test_cli_var_discover(tmp_path, plg):
    dag = plg.gen_two_level_dag(4, seed=5)
    X = plg.sample_svar(dag, [np.asfortranarray(np.eye(4) * 0.4)], T=3000, burn_in=100, seed=5)
    npy = tmp_path / "ts.npy"
    np.save(npy, X)
    rc, out, err = run(["var-discover", "--input", str(npy), "--lag", "1", "--out", str(tmp_path / "v")], tmp_path)
    assert rc == 0, err
    rep = json.loads(out.strip().splitlines()[-1])
    assert rep["order"] == plg.fit_var_lingam(X, lag=1).b0.order and rep["rows_used"] == 3000
    for f in ("b0.csv", "b_lag1.csv", "m_lag1.csv", "report.json"):
        assert (tmp_path / "v" / f).exists()
