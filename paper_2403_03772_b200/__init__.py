"""B200-native DirectLiNGAM causal-order search (arXiv 2403.03772 hot path).

Drop-in for the reference ``plingam`` package's causal-order surface
(proj/python/plingam/__init__.py, proj/bindings/pymodule.cpp:103-144): the same
functions, argument meaning and ``Error`` behaviour, computed by hand-written sm_100a
kernels in ``libplingam_b200.so`` through its C-ABI (include/plingam_b200.h).

There is no CPU fallback: if the compiled extension is missing the import fails.
"""

from ._core import (  # noqa: F401  (re-export, as the reference package does)
    Engine,
    Error,
    SimDag,
    WeightedDag,
    __version__,
    causal_order,
    engine_version,
    fit_direct_lingam,
    gen_sparse_dag,
    gen_two_level_dag,
    init_distributed,
    nccl_unique_id,
    regress_out,
    reset,
    sample_lingam,
    search_causal_order,
    search_causal_order_parallel,
    set_device,
    to_edges,
)

__all__ = [
    "Engine",
    "Error",
    "SimDag",
    "WeightedDag",
    "__version__",
    "causal_order",
    "engine_version",
    "fit_direct_lingam",
    "gen_sparse_dag",
    "gen_two_level_dag",
    "init_distributed",
    "nccl_unique_id",
    "regress_out",
    "reset",
    "sample_lingam",
    "search_causal_order",
    "search_causal_order_parallel",
    "set_device",
    "to_edges",
]
