"""CPU-only checks of the product boundary: the C-ABI library loads and exports every
symbol include/plingam_b200.h declares, the host-side round schedule is a partition,
the package fails loudly without a GPU, and the synthetic generators are deterministic."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "plingam_b200.h")
LIB = os.path.join(ROOT, "paper_2403_03772_b200", "libplingam_b200.so")


class RoundPlan(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in
                ("nb", "ntiles", "tiles_per_rank", "tile_begin", "tile_count", "nseg", "seg_len", "replicated")]


@pytest.fixture(scope="module")
def cabi():
    lib = ctypes.CDLL(LIB)
    lib.plg_version.restype = ctypes.c_char_p
    return lib


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|void|const char\*)\s+(plg_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol(cabi):
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(cabi, s), s
    assert cabi.plg_version().decode().startswith("plingam_b200")


def test_round_plan_partitions_tiles(cabi):
    for u in (2, 3, 31, 32, 33, 100, 128, 129, 999, 2000):
        for world in (1, 2, 3, 4, 8):
            covered = []
            segs = set()
            for rank in range(world):
                p = RoundPlan()
                assert cabi.plg_plan_round(u, 10000, rank, world, ctypes.byref(p)) == 0
                assert p.nb == (u + 31) // 32 and p.ntiles == p.nb * (p.nb + 1) // 2
                assert p.replicated == (u <= 128)
                segs.add((p.nseg, p.seg_len))
                if p.replicated:  # small rounds: every rank evaluates every pair, no exchange
                    assert (p.tile_begin, p.tile_count, p.tiles_per_rank) == (0, p.ntiles, p.ntiles)
                    continue
                covered += list(range(p.tile_begin, p.tile_begin + p.tile_count))
                assert p.tiles_per_rank * world >= p.ntiles
                assert p.tile_begin == min(p.ntiles, rank * p.tiles_per_rank)
            if u > 128:
                assert covered == list(range(p.ntiles)), (u, world)
            # segmentation (hence every entropy bit) does not depend on the rank count
            assert len(segs) == 1
            nseg, seg_len = segs.pop()
            assert seg_len % (16 if u <= 128 else 64) == 0
            assert (nseg - 1) * seg_len < 10000 <= nseg * seg_len


def test_round_plan_segmentation_independent_of_world(cabi):
    for u in range(2, 300, 7):
        plans = set()
        for world in (1, 2, 4, 8):
            p = RoundPlan()
            cabi.plg_plan_round(u, 10000, 0, world, ctypes.byref(p))
            plans.add((p.nseg, p.seg_len))
        assert len(plans) == 1


def test_tile_decode_upper_triangle(cabi):
    bi, bj = ctypes.c_int32(), ctypes.c_int32()
    for nb in (1, 2, 5, 63):
        seen = []
        for t in range(nb * (nb + 1) // 2):
            assert cabi.plg_tile_decode(t, nb, ctypes.byref(bi), ctypes.byref(bj)) == 0
            seen.append((bi.value, bj.value))
        assert seen == [(i, j) for i in range(nb) for j in range(i, nb)]
        assert cabi.plg_tile_decode(nb * (nb + 1) // 2, nb, ctypes.byref(bi), ctypes.byref(bj)) != 0


def test_invalid_plan_arguments(cabi):
    p = RoundPlan()
    assert cabi.plg_plan_round(1, 10, 0, 1, ctypes.byref(p)) != 0
    assert cabi.plg_plan_round(5, 10, 2, 2, ctypes.byref(p)) != 0


def test_package_fails_loudly_without_gpu(plg):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    X = np.asfortranarray(np.random.default_rng(0).uniform(size=(100, 3)))
    with pytest.raises(plg.Error) as e:
        plg.causal_order(X)
    assert e.value.code == "DeviceError"
    with pytest.raises(plg.Error) as e:  # the VarLiNGAM front-end has no CPU fallback either
        plg.estimate_var(np.asfortranarray(np.random.default_rng(1).uniform(size=(200, 3))), 1)
    assert e.value.code == "DeviceError"


def test_host_validation_before_device(plg):
    # argument errors of the reference surface are raised before any device work
    X = np.asfortranarray(np.random.default_rng(0).uniform(size=(10, 3)))
    with pytest.raises(plg.Error) as e:
        plg.search_causal_order_parallel(X, [0, 1], 0)
    assert e.value.code == "OutOfRange"
    with pytest.raises(plg.Error) as e:
        plg.fit_direct_lingam(X, workers=0)
    assert e.value.code == "OutOfRange"
    with pytest.raises(plg.Error) as e:
        plg.fit_direct_lingam(X, edge_threshold=-1.0)
    assert e.value.code == "OutOfRange"


def test_generators_deterministic(plg):
    d1 = plg.gen_two_level_dag(10, seed=42000)
    d2 = plg.gen_two_level_dag(10, seed=42000)
    assert np.array_equal(d1.weights, d2.weights) and d1.order == d2.order
    X1 = plg.sample_lingam(d1, 500, seed=1)
    X2 = plg.sample_lingam(d2, 500, seed=1)
    assert X1.tobytes() == X2.tobytes() and X1.flags["F_CONTIGUOUS"]
    W = d1.weights
    pos = {v: p for p, v in enumerate(d1.order)}
    assert all(pos[j] < pos[i] for i in range(10) for j in range(10) if W[i, j] != 0.0)
    s = plg.gen_sparse_dag(200, avg_parents=2.0, seed=1)
    indeg = (s.weights != 0).sum(axis=1)
    assert 1.5 < indeg.mean() < 2.5
    L = plg.sample_lingam(s, 20000, seed=1, kind="laplace")
    assert L.shape == (20000, 200) and np.all(np.isfinite(L))


def test_uniform_generator_matches_reference_rng(plg):
    """rng.hpp:14-43: mt19937_64, uniform = (u64 >> 11) * 2^-53. numpy's MT19937 is the
    32-bit twister, so check against an independent mt19937_64 in pure Python."""

    class MT64:
        def __init__(self, seed):
            self.mt = [0] * 312
            self.idx = 312
            self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
            for i in range(1, 312):
                self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF

        def next(self):
            if self.idx >= 312:
                for i in range(312):
                    x = (self.mt[i] & 0xFFFFFFFF80000000) | (self.mt[(i + 1) % 312] & 0x7FFFFFFF)
                    xa = x >> 1
                    if x & 1:
                        xa ^= 0xB5026F5AA96619E9
                    self.mt[i] = self.mt[(i + 156) % 312] ^ xa
                self.idx = 0
            y = self.mt[self.idx]
            self.idx += 1
            y ^= (y >> 29) & 0x5555555555555555
            y ^= (y << 17) & 0x71D67FFFEDA60000
            y ^= (y << 37) & 0xFFF7EEE000000000
            y ^= y >> 43
            return y

    # sample_lingam with an empty DAG: row r, variable j = uniform draw r*d + j (simgen.cpp:59-81)
    dag = plg.gen_two_level_dag(2, seed=0, edge_prob=1e-12)
    X = plg.sample_lingam(dag, 3, seed=7)
    rng = MT64(7)
    expect = np.array([[(rng.next() >> 11) * 2.0 ** -53 for _ in range(2)] for _ in range(3)])
    assert np.array_equal(X, expect)


# ---------------------------------------------------------------- VarLiNGAM front-end (host)

def _svar(plg, d, T, seed, lag_diag=0.4, burn=200, kind="uniform", b0=None):
    dag = b0 if b0 is not None else plg.gen_sparse_dag(d, avg_parents=1.0, seed=seed, wmin=0.1, wmax=0.4)
    M1 = np.asfortranarray(np.eye(d) * lag_diag)
    return plg.sample_svar(dag, [M1], T=T, burn_in=burn, seed=seed, kind=kind)


def test_estimate_var_matches_lstsq(plg):
    # the host QR restatement (the reference's method; parity reference of the device path)
    X = _svar(plg, 6, 3000, 3)
    ms, res = plg._estimate_var_qr(X, 1)
    Z = np.hstack([np.ones((X.shape[0] - 1, 1)), X[:-1]])
    B = np.linalg.lstsq(Z, X[1:], rcond=None)[0]
    assert np.allclose(ms[0], B[1:].T, atol=1e-12)
    assert np.allclose(res, X[1:] - Z @ B, atol=1e-12)
    ms2, res2 = plg._estimate_var_qr(X, 2)
    assert len(ms2) == 2 and res2.shape == (X.shape[0] - 2, 6)


def test_estimate_var_reference_contracts(plg):  # test_var_lingam.cpp:39-97
    rng = np.random.default_rng(11)
    ms, res = plg._estimate_var_qr(rng.uniform(size=(10000, 3)), 1)
    assert np.all(np.abs(ms[0]) < 0.05) and res.shape[0] == 9999
    ar = _svar(plg, 2, 10000, 21, lag_diag=0.5, b0=plg.gen_two_level_dag(2, seed=0, edge_prob=1e-12))
    # (a 2-variable empty DAG; the AR(1) coefficient of each variable is recovered)
    assert abs(plg._estimate_var_qr(ar, 1)[0][0][0, 0] - 0.5) <= 0.05
    X = _svar(plg, 3, 4000, 41)
    _, res = plg._estimate_var_qr(X, 1)
    for eq in range(3):
        for reg in range(3):
            lagged = X[:-1, reg]
            c = np.mean((res[:, eq] - res[:, eq].mean()) * (lagged - lagged.mean()))
            assert abs(c) <= 1e-8 * res[:, eq].std() * lagged.std()


def test_estimate_var_errors(plg):  # test_var_lingam.cpp:61-80
    with pytest.raises(plg.Error) as e:
        plg._estimate_var_qr(np.full((100, 2), 3.5), 1)
    assert e.value.code == "SingularDesign"
    rng = np.random.default_rng(31)
    with pytest.raises(plg.Error) as e:
        plg._estimate_var_qr(rng.uniform(size=(5, 3)), 1)
    assert e.value.code == "InsufficientRows"
    with pytest.raises(plg.Error) as e:
        plg._estimate_var_qr(rng.uniform(size=(100, 3)), 0)
    assert e.value.code == "OutOfRange"
    bad = rng.uniform(size=(100, 3))
    bad[4, 1] = np.inf
    with pytest.raises(plg.Error) as e:
        plg._estimate_var_qr(bad, 1)
    assert e.value.code == "NonFinite"


def test_sample_svar_deterministic_and_stable(plg):
    a = _svar(plg, 20, 500, 9, kind="laplace")
    b = _svar(plg, 20, 500, 9, kind="laplace")
    assert a.tobytes() == b.tobytes() and np.all(np.isfinite(a))
    dag = plg.gen_sparse_dag(4, 2.0, seed=1)
    with pytest.raises(plg.Error) as e:  # explosive lag matrix trips the overflow guard
        plg.sample_svar(dag, [np.asfortranarray(np.eye(4) * 3.0)], T=2000, burn_in=0, seed=1)
    assert e.value.code == "UnstableSystem"


def test_oracle_generators_match_package(plg):
    """bench.py's reference arm builds its inputs with the oracle's generators (no product
    library in that process): they must be the package's generators bit for bit."""
    import oracle_lib

    for d, seed in ((7, 3), (40, 11)):
        a = plg.gen_two_level_dag(d, seed=seed)
        W, order = oracle_lib.gen_two_level_dag(d, seed)
        assert np.array_equal(a.weights, W) and list(a.order) == list(order)
        Xa = plg.sample_lingam(a, 300, seed=seed)
        Xo = oracle_lib.sample_lingam((W, order), 300, seed)
        assert np.array_equal(Xa, Xo)
    for kind in ("uniform", "laplace", "t3", "gauss"):
        a = plg.gen_sparse_dag(60, avg_parents=2.0, seed=5)
        dag = oracle_lib.gen_sparse_dag(60, 2.0, 5)
        assert np.array_equal(a.weights, dag[0]) and list(a.order) == list(dag[1])
        Xa = plg.sample_lingam(a, 500, seed=9, noise=(0.0, 1.0), kind=kind)
        Xo = oracle_lib.sample_lingam(dag, 500, 9, (0.0, 1.0), kind)
        assert np.array_equal(Xa, Xo), kind


class Status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("row", ctypes.c_int64), ("col", ctypes.c_int64),
                ("msg", ctypes.c_char * 256)]


def test_peer_context_argument_checks(cabi):
    # plg_ctx_create_p2p validates its arguments before touching a device (PLG_OutOfRange = 11)
    ctx = ctypes.c_void_p()
    st = Status()
    for rank, world, dims in ((0, 9, 100), (2, 2, 100), (-1, 2, 100), (0, 2, 1)):
        rc = cabi.plg_ctx_create_p2p(0, rank, world, dims, ctypes.byref(ctx), ctypes.byref(st))
        assert rc == 11 and st.code == 11, (rank, world, dims, st.msg)
        assert not ctx.value
    assert cabi.plg_p2p_handle(None, ctypes.create_string_buffer(64), ctypes.byref(st)) == 11
    assert cabi.plg_p2p_connect(None, ctypes.create_string_buffer(128), ctypes.byref(st)) == 11
