"""ctypes wrapper of the CPU oracle (oracle/liboracle.so) — test infrastructure only.

The oracle restates the reference hot path (proj/src/kernels.cpp, ordering.cpp,
types.cpp, direct_lingam.cpp) in C; see oracle/plingam_oracle.h. Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline leg load it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB_PATH = os.path.join(ORACLE_DIR, "liboracle.so")

ERROR_NAMES = [
    "NonFinite", "ZeroVariance", "TooFewSamples", "TooShort", "LengthMismatch",
    "DimensionMismatch", "EmptyCandidates", "SingularDesign", "InsufficientRows",
    "UnstableSystem", "OutOfRange", "InvalidIndex",
]


class OracleError(Exception):
    def __init__(self, code: int, row: int, col: int, msg: str):
        super().__init__(msg)
        self.code = ERROR_NAMES[code - 1] if 1 <= code <= len(ERROR_NAMES) else str(code)
        self.row = row
        self.col = col


class _Status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("row", ctypes.c_int64), ("col", ctypes.c_int64),
                ("msg", ctypes.c_char * 256)]


_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int32)


def build() -> str:
    src = [os.path.join(ORACLE_DIR, f) for f in ("plingam_oracle.c", "simgen_oracle.c", "plingam_oracle.h", "Makefile")]
    if not os.path.exists(LIB_PATH) or any(os.path.getmtime(s) > os.path.getmtime(LIB_PATH) for s in src):
        subprocess.run(["make", "-C", ORACLE_DIR], check=True, capture_output=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.orc_gaussian_entropy.restype = ctypes.c_double
        for name in ("orc_mean", "orc_variance_pop", "orc_std_pop", "orc_entropy_approx"):
            getattr(L, name).restype = ctypes.c_double
            getattr(L, name).argtypes = [_D, ctypes.c_int64]
        L.orc_covariance_pop.restype = ctypes.c_double
        L.orc_covariance_pop.argtypes = [_D, _D, ctypes.c_int64]
        L.orc_log_cosh.restype = ctypes.c_double
        L.orc_log_cosh.argtypes = [ctypes.c_double]
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _ip(a: np.ndarray):
    return a.ctypes.data_as(_I)


def _check(rc: int, st: _Status):
    if rc:
        raise OracleError(st.code, st.row, st.col, st.msg.decode())


def _col(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


def _mat(X) -> np.ndarray:
    return np.asfortranarray(X, dtype=np.float64)


def mean(x):
    x = _col(x)
    return lib().orc_mean(_dp(x), x.size)


def variance_pop(x):
    x = _col(x)
    return lib().orc_variance_pop(_dp(x), x.size)


def std_pop(x):
    x = _col(x)
    return lib().orc_std_pop(_dp(x), x.size)


def covariance_pop(x, y):
    x, y = _col(x), _col(y)
    return lib().orc_covariance_pop(_dp(x), _dp(y), x.size)


def log_cosh(u: float) -> float:
    return lib().orc_log_cosh(float(u))


def gaussian_entropy() -> float:
    return lib().orc_gaussian_entropy()


def standardize(x) -> np.ndarray:
    x = _col(x)
    out = np.empty_like(x)
    st = _Status()
    _check(lib().orc_standardize(_dp(x), ctypes.c_int64(x.size), _dp(out), ctypes.byref(st)), st)
    return out


def residual(xi, xj) -> np.ndarray:
    xi, xj = _col(xi), _col(xj)
    if xi.size != xj.size:
        raise OracleError(5, -1, -1, "residual: length mismatch")
    out = np.empty_like(xi)
    st = _Status()
    _check(lib().orc_residual(_dp(xi), _dp(xj), ctypes.c_int64(xi.size), _dp(out), ctypes.byref(st)), st)
    return out


def entropy_approx(u) -> float:
    u = _col(u)
    return lib().orc_entropy_approx(_dp(u), u.size)


def entropy_of_normalized(r) -> float:
    r = _col(r)
    out = ctypes.c_double()
    st = _Status()
    _check(lib().orc_entropy_of_normalized(_dp(r), ctypes.c_int64(r.size), ctypes.byref(out), ctypes.byref(st)), st)
    return out.value


def diff_mutual_info(xi, xj, ri_j, rj_i) -> float:
    a = [_col(v) for v in (xi, xj, ri_j, rj_i)]
    if len({v.size for v in a}) != 1:
        raise OracleError(5, -1, -1, "diff_mutual_info: length mismatch")
    out = ctypes.c_double()
    st = _Status()
    _check(lib().orc_diff_mutual_info(*[_dp(v) for v in a], ctypes.c_int64(a[0].size), ctypes.byref(out),
                                      ctypes.byref(st)), st)
    return out.value


def validate(X) -> None:
    X = _mat(X)
    st = _Status()
    n, d = X.shape
    _check(lib().orc_validate(_dp(X), ctypes.c_int64(n), ctypes.c_int32(d), ctypes.c_int64(max(n, 1)),
                              ctypes.byref(st)), st)


def search_causal_order(X, U, workers: int = 1, fast: bool = False):
    X = _mat(X)
    n, d = X.shape
    U = np.ascontiguousarray(U, dtype=np.int32)
    chosen = ctypes.c_int32(-1)
    scores = np.empty(d, dtype=np.float64)
    st = _Status()
    _check(lib().orc_search_causal_order(_dp(X), ctypes.c_int64(n), ctypes.c_int32(d), ctypes.c_int64(max(n, 1)),
                                         _ip(U), ctypes.c_int32(U.size), ctypes.c_int32(workers),
                                         ctypes.c_int32(1 if fast else 0), ctypes.byref(chosen), _dp(scores),
                                         ctypes.byref(st)), st)
    return chosen.value, scores


def regress_out(X, exog: int, remaining) -> np.ndarray:
    X = _mat(X)
    n, d = X.shape
    rem = np.ascontiguousarray(remaining, dtype=np.int32)
    out = np.empty((n, rem.size), dtype=np.float64, order="F")
    st = _Status()
    _check(lib().orc_regress_out(_dp(X), ctypes.c_int64(n), ctypes.c_int32(d), ctypes.c_int64(max(n, 1)),
                                 ctypes.c_int32(exog), _ip(rem), ctypes.c_int32(rem.size), _dp(out),
                                 ctypes.byref(st)), st)
    return out


def causal_order(X, parallel: bool = False, workers: int = 1, fast: bool = False, max_rounds: int = -1,
                 return_scores: bool = False):
    X = _mat(X)
    n, d = X.shape
    order = np.full(max(d, 1), -1, dtype=np.int32)
    rounds = (d - 1) if max_rounds < 0 else min(max_rounds, max(d - 1, 0))
    scores = np.zeros((max(rounds, 1), max(d, 1)), dtype=np.float64) if return_scores else None
    st = _Status()
    _check(lib().orc_causal_order(_dp(X), ctypes.c_int64(n), ctypes.c_int32(d), ctypes.c_int64(max(n, 1)),
                                  ctypes.c_int32(1 if parallel else 0), ctypes.c_int32(workers),
                                  ctypes.c_int32(1 if fast else 0), ctypes.c_int32(max_rounds), _ip(order),
                                  _dp(scores) if return_scores else None, ctypes.byref(st)), st)
    nout = d if max_rounds < 0 or rounds == d - 1 else rounds
    out = [int(v) for v in order[:nout]]
    return (out, scores[:rounds]) if return_scores else out


def causal_order_pruned(X, workers: int = 1, return_second: bool = False):
    """Exact pruned rounds (orc_causal_order_pruned): (order, winning k per round, pairs),
    plus, with return_second, a lower bound of each round's runner-up k."""
    X = _mat(X)
    n, d = X.shape
    order = np.full(max(d, 1), -1, dtype=np.int32)
    wk = np.zeros(max(d - 1, 1), dtype=np.float64)
    sk = np.zeros(max(d - 1, 1), dtype=np.float64)
    pairs = ctypes.c_int64(0)
    st = _Status()
    _check(lib().orc_causal_order_pruned(_dp(X), ctypes.c_int64(n), ctypes.c_int32(d), ctypes.c_int64(max(n, 1)),
                                         ctypes.c_int32(workers), _ip(order), _dp(wk), _dp(sk), ctypes.byref(pairs),
                                         ctypes.byref(st)), st)
    out = ([int(v) for v in order[:d]], wk[: max(d - 1, 0)], pairs.value)
    return out + (sk[: max(d - 1, 0)],) if return_second else out


def fit_weights(X, order):
    X = _mat(X)
    n, d = X.shape
    o = np.ascontiguousarray(order, dtype=np.int32)
    B = np.zeros((d, d), dtype=np.float64, order="F")
    pinv = ctypes.c_int32(0)
    st = _Status()
    _check(lib().orc_fit_weights(_dp(X), ctypes.c_int64(n), ctypes.c_int32(d), ctypes.c_int64(n), _ip(o), _dp(B),
                                 ctypes.byref(pinv), ctypes.byref(st)), st)
    return B, bool(pinv.value)


def fit_weights_prefix(X, order, workers: int | None = None):
    """Weights from one prefix QR of the order-permuted centred design (the large-d
    reference; cross-checked against the per-target column-pivoted QR of fit_weights).
    Returns (B, used_pinv, n_dependent)."""
    X = _mat(X)
    n, d = X.shape
    o = np.ascontiguousarray(order, dtype=np.int32)
    B = np.zeros((d, d), dtype=np.float64, order="F")
    pinv = ctypes.c_int32(0)
    ndep = ctypes.c_int32(0)
    st = _Status()
    w = workers if workers is not None else (os.cpu_count() or 1)
    _check(lib().orc_fit_weights_prefix(_dp(X), ctypes.c_int64(n), ctypes.c_int32(d), ctypes.c_int64(n), _ip(o),
                                        ctypes.c_int32(w), _dp(B), ctypes.byref(pinv), ctypes.byref(ndep),
                                        ctypes.byref(st)), st)
    return B, bool(pinv.value), int(ndep.value)


def fit_weights_targets(X, order, positions):
    """Per-target column-pivoted QR (the faithful route) for the targets at the given order
    positions only; B rows of the other targets are zero."""
    X = _mat(X)
    n, d = X.shape
    o = np.ascontiguousarray(order, dtype=np.int32)
    pos = np.ascontiguousarray(positions, dtype=np.int32)
    B = np.zeros((d, d), dtype=np.float64, order="F")
    pinv = ctypes.c_int32(0)
    st = _Status()
    _check(lib().orc_fit_weights_targets(_dp(X), ctypes.c_int64(n), ctypes.c_int32(d), ctypes.c_int64(n), _ip(o),
                                         _ip(pos), ctypes.c_int32(len(pos)), _dp(B), ctypes.byref(pinv),
                                         ctypes.byref(st)), st)
    return B, bool(pinv.value)


_NOISE = {"uniform": 0, "laplace": 1, "t3": 2, "gauss": 3}


def gen_two_level_dag(d: int, seed: int, edge_prob: float = 0.5):
    """(W, order) as the package's gen_two_level_dag (simgen_oracle.c; no product library)."""
    W = np.zeros((d, d), dtype=np.float64, order="F")
    order = np.zeros(d, dtype=np.int32)
    if lib().orc_gen_two_level_dag(ctypes.c_int32(d), ctypes.c_uint64(seed), ctypes.c_double(edge_prob), _dp(W),
                                   _ip(order)):
        raise ValueError("gen_two_level_dag: d must be >= 2")
    return W, order


def gen_sparse_dag(d: int, avg_parents: float = 2.0, seed: int = 1, wmin: float = 0.5, wmax: float = 1.5):
    W = np.zeros((d, d), dtype=np.float64, order="F")
    order = np.zeros(d, dtype=np.int32)
    if lib().orc_gen_sparse_dag(ctypes.c_int32(d), ctypes.c_double(avg_parents), ctypes.c_uint64(seed),
                                ctypes.c_double(wmin), ctypes.c_double(wmax), _dp(W), _ip(order)):
        raise ValueError("gen_sparse_dag: d must be >= 2")
    return W, order


def sample_lingam(dag, n: int, seed: int, noise=(0.0, 1.0), kind: str = "uniform"):
    W, order = dag
    d = W.shape[0]
    X = np.zeros((n, d), dtype=np.float64, order="F")
    if lib().orc_sample_lingam(_dp(np.asfortranarray(W)), _ip(np.ascontiguousarray(order, dtype=np.int32)),
                               ctypes.c_int32(d), ctypes.c_int64(n), ctypes.c_uint64(seed),
                               ctypes.c_int32(_NOISE[kind]), ctypes.c_double(noise[0]), ctypes.c_double(noise[1]),
                               _dp(X)):
        raise MemoryError("sample_lingam")
    return X


# ---- the reference's own code (oracle/_ref/libplingam_ref.so, oracle/Makefile.ref): the
# unmodified proj/src/{kernels,ordering,types,error}.cpp against a minimal Eigen stand-in ----

REF_LIB_PATH = os.path.join(ORACLE_DIR, "_ref", "libplingam_ref.so")
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_LIB_PATH)


def ref_lib():
    global _ref
    if _ref is None:
        L = ctypes.CDLL(REF_LIB_PATH)
        I64 = ctypes.POINTER(ctypes.c_int64)
        L.ref_causal_order.argtypes = [_D, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _I, _I,
                                       I64, I64]
        L.ref_search.argtypes = [_D, ctypes.c_int64, ctypes.c_int32, _I, ctypes.c_int32, ctypes.c_int32, _I, _D, _I,
                                 I64, I64]
        _ref = L
    return _ref


def _ref_check(rc, code, row, col, what):
    if rc:
        raise OracleError(code.value, row.value, col.value, f"reference {what} failed")


def ref_causal_order(X, parallel: bool = False, workers: int = 1):
    """plingam::causal_order (proj/src/ordering.cpp:213-244), the reference's code itself."""
    X = _mat(X)
    n, d = X.shape
    order = np.zeros(max(d, 1), dtype=np.int32)
    code, row, col = ctypes.c_int32(0), ctypes.c_int64(0), ctypes.c_int64(0)
    rc = ref_lib().ref_causal_order(_dp(X), n, d, int(parallel), workers, _ip(order), ctypes.byref(code),
                                    ctypes.byref(row), ctypes.byref(col))
    _ref_check(rc, code, row, col, "causal_order")
    return [int(v) for v in order[:d]]


def ref_search_causal_order(X, U, workers: int = 1):
    """plingam::search_causal_order[_parallel] (proj/src/ordering.cpp:101-176)."""
    X = _mat(X)
    n, d = X.shape
    Ua = np.ascontiguousarray(U, dtype=np.int32)
    scores = np.zeros(d, dtype=np.float64)
    chosen = ctypes.c_int32(-1)
    code, row, col = ctypes.c_int32(0), ctypes.c_int64(0), ctypes.c_int64(0)
    rc = ref_lib().ref_search(_dp(X), n, d, _ip(Ua), len(Ua), workers, ctypes.byref(chosen), _dp(scores),
                              ctypes.byref(code), ctypes.byref(row), ctypes.byref(col))
    _ref_check(rc, code, row, col, "search_causal_order")
    return int(chosen.value), scores
