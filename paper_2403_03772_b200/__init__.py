"""B200-native DirectLiNGAM causal-order search (arXiv 2403.03772 hot path).

Drop-in for the reference ``plingam`` package's causal-order surface
(proj/python/plingam/__init__.py, proj/bindings/pymodule.cpp:79-144): the same
functions, argument meaning and ``Error`` behaviour, computed by hand-written sm_100a
kernels in ``libplingam_b200.so`` through its C-ABI (include/plingam_b200.h).

There is no CPU fallback: if the compiled extension is missing the import fails, and
without a CUDA device every call raises ``Error`` with ``code == "DeviceError"``.
"""

from ._core import _estimate_var_qr  # noqa: F401  (test reference: the reference's host QR)
from ._core import (  # noqa: F401  (re-export, as the reference package does)
    Engine,
    Error,
    SimDag,
    VarModel,
    WeightedDag,
    __version__,
    causal_order,
    diff_mutual_info,
    engine_version,
    entropy_approx,
    estimate_var,
    fit_direct_lingam,
    fit_var_lingam,
    gen_sparse_dag,
    gen_two_level_dag,
    init_distributed,
    nccl_unique_id,
    regress_out,
    reset,
    residual,
    sample_lingam,
    sample_svar,
    search_causal_order,
    search_causal_order_parallel,
    set_device,
    standardize,
    to_edges,
    uniform_vector,
)

__all__ = [
    "Engine",
    "Error",
    "SimDag",
    "VarModel",
    "WeightedDag",
    "__version__",
    "causal_order",
    "diff_mutual_info",
    "engine_version",
    "entropy_approx",
    "estimate_var",
    "fit_direct_lingam",
    "fit_var_lingam",
    "gen_sparse_dag",
    "gen_two_level_dag",
    "init_distributed",
    "nccl_unique_id",
    "regress_out",
    "reset",
    "residual",
    "sample_lingam",
    "sample_svar",
    "search_causal_order",
    "search_causal_order_parallel",
    "set_device",
    "standardize",
    "to_edges",
    "uniform_vector",
]
