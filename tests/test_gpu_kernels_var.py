"""GPU checks of the element-kernel surface (plingam::kernels, kernels.hpp:25-70) and of
the VarLiNGAM path (var_lingam.cpp:55-70) against the CPU oracle and the goldens."""

import hashlib
import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_standardize_and_residual_bit_exact(plg, oracle):  # test_kernels.cpp:12-61
    s = plg.standardize([1.0, 2.0, 3.0])
    assert s[0] == pytest.approx(-1.224744871391589, rel=1e-9) and abs(s[1]) <= 1e-12
    assert list(plg.residual([1.0, 2.0, 3.0], [1.0, 0.0, -1.0])) == pytest.approx([2.0, 2.0, 2.0], rel=1e-12)
    xi = np.array([1.0, 1.0, -1.0, -1.0])
    assert plg.residual(xi, [1.0, -1.0, 1.0, -1.0]).tobytes() == xi.tobytes()
    rng = np.random.default_rng(3)
    for _ in range(10):
        x = rng.laplace(size=777) * 3 + 1
        y = rng.uniform(size=777)
        assert plg.standardize(x).tobytes() == oracle.standardize(x).tobytes()
        assert plg.residual(x, y).tobytes() == oracle.residual(x, y).tobytes()
        assert np.all(plg.residual(x, x) == 0.0)


def test_kernel_error_paths(plg):  # test_kernels.cpp:33-74
    with pytest.raises(plg.Error) as e:
        plg.standardize([5.0, 5.0, 5.0])
    assert e.value.code == "ZeroVariance" and str(e.value) == "standardize: constant input"
    with pytest.raises(plg.Error) as e:
        plg.standardize([1.0])
    assert e.value.code == "TooShort"
    with pytest.raises(plg.Error) as e:
        plg.residual([1.0, 2.0, 3.0], [1.0, 2.0])
    assert e.value.code == "LengthMismatch"
    with pytest.raises(plg.Error) as e:
        plg.residual([1.0, 2.0, 3.0], [2.0, 2.0, 2.0])
    assert e.value.code == "ZeroVariance"
    z = np.zeros(10)
    with pytest.raises(plg.Error) as e:
        plg.diff_mutual_info(np.ones(10), np.ones(10), z, z)
    assert e.value.code == "ZeroVariance"


def test_entropy_and_mi_against_oracle(plg, oracle):  # test_kernels.cpp:118-192
    rng = np.random.default_rng(53)
    for _ in range(20):
        n = 50 + int(rng.uniform() * 2000)
        xi = oracle.standardize(rng.uniform(size=n))
        xj = oracle.standardize(rng.laplace(size=n))
        ri, rj = oracle.residual(xi, xj), oracle.residual(xj, xi)
        assert plg.entropy_approx(xi) == pytest.approx(oracle.entropy_approx(xi), rel=1e-13)
        fwd = plg.diff_mutual_info(xi, xj, ri, rj)
        assert fwd == pytest.approx(oracle.diff_mutual_info(xi, xj, ri, rj), abs=1e-12)
        assert fwd == -plg.diff_mutual_info(xj, xi, rj, ri)  # exact antisymmetry
        assert plg.entropy_approx(xi) == plg.entropy_approx(-xi)  # exact sign-flip invariance
    g = oracle.standardize(rng.normal(size=100000))
    assert plg.entropy_approx(g) == pytest.approx(0.5 * (1.0 + math.log(2.0 * math.pi)), rel=0.01)


def test_var_lingam_transform_identity(plg):  # test_var_lingam.cpp:117-133, test_smoke.py:52-58
    dag = plg.gen_two_level_dag(4, seed=5)
    X = plg.sample_svar(dag, [np.asfortranarray(np.eye(4) * 0.4)], T=3000, burn_in=100, seed=5)
    model = plg.fit_var_lingam(X, lag=1)
    expected = (np.eye(4) - model.b0.weights) @ model.m_raw[0]
    assert np.allclose(model.b_lagged[0], expected, atol=1e-14)
    W = model.b0.weights
    pos = {v: p for p, v in enumerate(model.b0.order)}
    assert all(W[i, j] == 0.0 for i in range(4) for j in range(4) if pos[j] >= pos[i])


def test_var_lingam_independent_residuals(plg):  # test_var_lingam.cpp:99-115
    dag = plg.gen_two_level_dag(3, seed=0, edge_prob=1e-12)
    m1 = np.asfortranarray([[0.5, 0.0, 0.1], [0.0, -0.4, 0.0], [0.1, 0.0, 0.3]])
    X = plg.sample_svar(dag, [m1], T=20000, burn_in=500, seed=51)
    model = plg.fit_var_lingam(X, lag=1)
    assert np.all(np.abs(model.b_lagged[0] - model.m_raw[0]) < 0.1)


def test_c4_golden_order(plg):
    """BASELINE configs[3]: VarLiNGAM lag 1 on a d=500, T=2500 SVAR (residuals 2499 x 500)."""
    path = os.path.join(GOLDEN, "c4_order.json")
    if not os.path.exists(path):
        pytest.skip("c4 golden not generated")
    with open(path) as f:
        fx = json.load(f)
    d = 500
    b0 = plg.gen_sparse_dag(d, avg_parents=2.0, seed=1, wmin=0.1, wmax=0.5)
    b1 = np.diag(plg.uniform_vector(d, 1, 0.2, 0.5))
    X = plg.sample_svar(b0, [np.asfortranarray(b1)], T=2500, burn_in=500, seed=1, noise=(0.0, 1.0), kind="laplace")
    _, res = plg._estimate_var_qr(X, 1)  # the golden's input: the reference's QR residuals
    assert hashlib.sha256(np.asfortranarray(res).tobytes(order="F")).hexdigest() == fx["sha256"]
    _, res_gpu = plg.estimate_var(X, 1)  # the device path (normal equations) feeds fit_var_lingam
    assert np.max(np.abs(res_gpu - res)) <= 1e-10 * np.max(np.abs(res))
    model = plg.fit_var_lingam(X, lag=1)
    assert model.b0.order == fx["order"]
    for t, row in fx["B_rows"].items():
        ref = np.asarray(row)
        assert np.all(np.abs(model.b0.weights[int(t)] - ref) <= 1e-6 * np.maximum(1.0, np.abs(ref)))


def _svar(plg, d, T, seed, lag_diag=0.4, burn=200, kind="uniform", lags=1):
    dag = plg.gen_sparse_dag(d, avg_parents=1.0, seed=seed, wmin=0.1, wmax=0.4)
    Ms = [np.asfortranarray(np.eye(d) * (lag_diag / lags)) for _ in range(lags)]
    return plg.sample_svar(dag, Ms, T=T, burn_in=burn, seed=seed, kind=kind)


@pytest.mark.parametrize("d,T,lag,seed", [(6, 3000, 1, 3), (6, 3000, 2, 4), (40, 2000, 1, 5), (120, 1500, 3, 6)])
def test_estimate_var_device_matches_qr(plg, d, T, lag, seed):
    """estimate_var on the device (scaled normal equations + Cholesky + refinement) against
    the reference's method (column-pivoted QR, host restatement) and numpy lstsq."""
    X = _svar(plg, d, T, seed, kind="laplace", lags=lag)
    ms, res = plg.estimate_var(X, lag)
    ms_q, res_q = plg._estimate_var_qr(X, lag)
    scale = np.max(np.abs(res_q))
    assert res.shape == res_q.shape and len(ms) == len(ms_q) == lag
    assert np.max(np.abs(res - res_q)) <= 1e-10 * scale
    for a, b in zip(ms, ms_q):
        assert np.max(np.abs(a - b)) <= 1e-10 * max(1.0, np.max(np.abs(b)))
    Z = np.hstack([np.ones((T - lag, 1))] + [X[lag - t:T - t] for t in range(1, lag + 1)])
    B = np.linalg.lstsq(Z, X[lag:], rcond=None)[0]
    assert np.max(np.abs(res - (X[lag:] - Z @ B))) <= 1e-10 * scale


def test_estimate_var_device_errors(plg):  # test_var_lingam.cpp:61-80, same codes as the host QR
    rng = np.random.default_rng(31)
    bad = rng.uniform(size=(100, 3))
    bad[4, 1] = np.inf
    for X, lag, code in ((np.full((100, 2), 3.5), 1, "SingularDesign"), (rng.uniform(size=(5, 3)), 1, "InsufficientRows"),
                         (rng.uniform(size=(100, 3)), 0, "OutOfRange"), (bad, 1, "NonFinite")):
        with pytest.raises(plg.Error) as e:
            plg.estimate_var(X, lag)
        assert e.value.code == code
        with pytest.raises(plg.Error) as e2:
            plg._estimate_var_qr(X, lag)
        assert e2.value.code == code


def _sampled_rounds(engine, oracle, X, rounds):
    """the GPU's working state after r rounds, searched by the oracle (all host
    cores), must give the GPU's own next choice; scores agree to 1e-8 relative."""
    full = engine.causal_order(X)
    for r in rounds:
        active, cols, prefix = engine.round_state(X, r)
        assert prefix == full[:r]
        c_ref, s_ref = oracle.search_causal_order(cols, list(range(len(active))), workers=os.cpu_count(), fast=True)
        assert active[c_ref] == full[r], r
        _, s_gpu = engine.search(cols, list(range(len(active))))
        fin = np.isfinite(s_ref)
        assert np.all(np.abs(np.asarray(s_gpu)[fin] - s_ref[fin]) <= 1e-8 * np.abs(s_ref[fin]) + 1e-15)
    return full


@pytest.mark.slow
def test_c3_sampled_rounds(engine, oracle):
    """BASELINE configs[2] (d=1000, n=10000, heavy-tailed noise): sampled-round parity."""
    import bench

    X = bench.make_input("c3")
    full = _sampled_rounds(engine, oracle, X, (0, 500, 990))
    assert sorted(full) == list(range(1000))


@pytest.mark.slow
def test_c5_sampled_rounds(engine, oracle):
    """BASELINE configs[4] (d=2000, n=10000): late-round parity (u = 500 and 10)."""
    import bench

    X = bench.make_input("c5")
    _sampled_rounds(engine, oracle, X, (1500, 1990))


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_full_order_golden(engine, name):
    """BASELINE configs[2] / configs[4], whole causal order against the CPU oracle: the
    golden is the oracle's exact pruned run (orc_causal_order_pruned, bit-identical order
    and winning k to its faithful mode, tests/test_oracle_kats.py). The GPU order must be
    identical, every round's winning k within the score bar (1e-9 relative)."""
    import bench

    path = os.path.join(GOLDEN, f"{name}_order_full.json")
    if not os.path.exists(path):
        pytest.skip(f"{name} full golden not generated")
    with open(path) as f:
        fx = json.load(f)
    X = np.asfortranarray(bench.make_input(name))
    assert hashlib.sha256(X.tobytes(order="F")).hexdigest() == fx["sha256"]
    order = engine.causal_order(X)
    assert order == fx["order"]
    k_gpu = np.asarray(engine.round_k())
    k_ref = np.array([float.fromhex(v) for v in fx["winner_k"]])
    assert k_gpu.shape == k_ref.shape
    assert np.all(np.abs(k_gpu - k_ref) <= 1e-9 * np.abs(k_ref) + 1e-15), np.max(np.abs(k_gpu - k_ref) / np.abs(k_ref))
