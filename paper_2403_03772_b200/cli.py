"""Command line front-end mirroring the reference CLI's `discover` and `var-discover`
(proj/tools/plingam_cli.cpp:105-266), on the B200 engine.

    python -m paper_2403_03772_b200 discover --input data.csv --out results/
    python -m paper_2403_03772_b200 discover --input data.npy --out results/      # binary
    torchrun --nproc-per-node 8 -m paper_2403_03772_b200 discover --input x.npy --gpus 8
    python -m paper_2403_03772_b200 var-discover --input series.csv --lag 1 --out results/

Inputs: CSV with a header row (as the reference's read_csv), `.npy` (any float array,
samples x variables), or raw little-endian float64 `.f64` with `--dims` (column-major if
`--colmajor`, else row-major). Outputs as the reference: adjacency.csv (or b0.csv,
b_lag*.csv, m_lag*.csv), order.txt and report.json (manifest with the FNV-1a digest of
the input). Exit codes as exit_code_for (plingam_cli.cpp:363-374): 1 flags/range,
3 singular/unstable, 2 other data errors.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

from . import _core

VERSION = "0.1.0"


def _err(code: str, msg: str) -> "_core.Error":
    e = _core.Error(msg)
    e.code, e.row, e.col = code, -1, -1
    return e


def _exit_code(code: str) -> int:
    if code in ("InvalidFlags", "OutOfRange"):
        return 1
    if code in ("SingularDesign", "UnstableSystem"):
        return 3
    return 2


def read_input(path: str, dims: int | None = None, colmajor: bool = False, allow_missing: bool = False):
    """(matrix samples x variables float64 Fortran-ordered, variable names)."""
    if path.endswith(".npy"):
        X = np.load(path)
        if X.ndim != 2:
            raise _err("DimensionMismatch", "input: .npy must be 2-D")
        names = [f"x{j}" for j in range(X.shape[1])]
    elif path.endswith(".f64"):
        if not dims:
            raise _err("InvalidFlags", "input: --dims is required for raw .f64 input")
        raw = np.fromfile(path, dtype="<f8")
        if raw.size % dims:
            raise _err("ParseError", "input: file size is not a multiple of --dims")
        X = raw.reshape((dims, -1)).T if colmajor else raw.reshape((-1, dims))
        names = [f"x{j}" for j in range(dims)]
    else:
        import pandas as pd

        try:
            df = pd.read_csv(path, skipinitialspace=True)
        except FileNotFoundError:
            raise _err("IoError", f"cannot open {path}")
        names = [str(c).strip() for c in df.columns]
        try:
            X = df.to_numpy(dtype=np.float64)
        except ValueError as e:
            raise _err("ParseError", f"{path}: {e}")
        if not allow_missing and np.isnan(X).any():
            r, c = np.argwhere(np.isnan(X))[0]
            raise _err("ParseError", f"{path}: missing value at row {r + 2}, column {c + 1}")
    return np.asfortranarray(X, dtype=np.float64), names


def _write_matrix(path: str, names, M) -> None:
    with open(path, "w") as f:
        f.write(",".join(names) + "\n")
        for row in np.asarray(M):
            f.write(",".join("%.17g" % v for v in row) + "\n")


def _manifest(command: str, config: dict, digest: str) -> dict:
    return {"command": command, "config": config, "input_digest": digest, "artifact_version": VERSION}


def _setup_gpus(gpus: int, dims: int, transport: str = "p2p") -> None:
    """--gpus N under torchrun: every rank maps every rank's exchange arena (peer memory,
    the default) or joins one NCCL communicator inside the engine (--transport nccl)."""
    if gpus <= 1:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != gpus:
        raise _err("InvalidFlags", f"--gpus {gpus} needs {gpus} processes (torchrun --nproc-per-node {gpus})")
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    if transport == "nccl":
        obj = [_core.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        _core.init_distributed(local, rank, world, obj[0])
        return

    def allgather(handle: bytes):
        out = [None] * world
        dist.all_gather_object(out, handle)
        return out

    _core.init_peer(local, rank, world, max(2, dims), allgather)


def run_discover(args) -> int:
    X, names = read_input(args.input, args.dims, args.colmajor)
    _setup_gpus(args.gpus, X.shape[1], args.transport)
    rank = int(os.environ.get("RANK", "0"))
    dag = _core.fit_direct_lingam(X, edge_threshold=args.threshold)
    order, B, used_pinv, phases = dag.order, dag.weights, dag.used_pinv, dag.phases
    edges = int(((np.abs(B) > args.threshold) & ~np.eye(B.shape[0], dtype=bool)).sum())
    report = {
        "manifest": _manifest("discover", {"input": args.input, "out": args.out, "gpus": args.gpus,
                                           "threshold": args.threshold}, _core.digest_file(args.input)),
        "dims": int(X.shape[1]), "samples": int(X.shape[0]), "order": order, "n_edges": edges,
        "used_pinv": bool(used_pinv), "ordering_seconds": phases["ordering_seconds"],
        "total_seconds": phases["total_seconds"],
    }
    if rank == 0:
        os.makedirs(args.out, exist_ok=True)
        _write_matrix(os.path.join(args.out, "adjacency.csv"), names, B)
        with open(os.path.join(args.out, "order.txt"), "w") as f:
            f.write("".join(f"{v}\n" for v in order))
        with open(os.path.join(args.out, "report.json"), "w") as f:
            f.write(json.dumps(report) + "\n")
        print(json.dumps(report))
    return 0


def run_var_discover(args) -> int:
    if args.lag < 1:
        raise _err("InvalidFlags", "var-discover: --lag must be >= 1")
    X, names = read_input(args.input, args.dims, args.colmajor)
    steps = ["drop_incomplete"]
    if names and names[0] == "t":  # optional leading timestamp column (plingam_cli.cpp:161-176)
        X, names = np.asfortranarray(X[:, 1:]), names[1:]
    rows_in = X.shape[0]
    if args.difference:  # preprocess.cpp:68-76
        X = np.asfortranarray(np.diff(X, axis=0))
        steps.append("first_difference")
    model = _core.fit_var_lingam(X, lag=args.lag)
    os.makedirs(args.out, exist_ok=True)
    _write_matrix(os.path.join(args.out, "b0.csv"), names, model.b0.weights)
    for tau in range(1, model.lag + 1):
        _write_matrix(os.path.join(args.out, f"b_lag{tau}.csv"), names, model.b_lagged[tau - 1])
        _write_matrix(os.path.join(args.out, f"m_lag{tau}.csv"), names, model.m_raw[tau - 1])
    W = model.b0.weights
    report = {
        "manifest": _manifest("var-discover", {"input": args.input, "out": args.out, "lag": args.lag,
                                               "difference": args.difference, "threshold": args.threshold},
                              _core.digest_file(args.input)),
        "preprocessing": steps, "dims_used": int(X.shape[1]), "rows_before_difference": int(rows_in),
        "rows_used": int(X.shape[0]), "order": model.b0.order,
        "n_instantaneous_edges": int(((np.abs(W) > args.threshold) & ~np.eye(W.shape[0], dtype=bool)).sum()),
        "used_pinv": bool(model.b0.used_pinv),
    }
    with open(os.path.join(args.out, "report.json"), "w") as f:
        f.write(json.dumps(report) + "\n")
    print(json.dumps(report))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2403_03772_b200",
                                 description="DirectLiNGAM / VarLiNGAM causal discovery on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("discover", "var-discover"):
        p = sub.add_parser(name)
        p.add_argument("--input", required=True)
        p.add_argument("--out", default=".")
        p.add_argument("--threshold", type=float, default=0.05)
        p.add_argument("--dims", type=int, default=None, help="variables, for raw .f64 input")
        p.add_argument("--colmajor", action="store_true", help="raw .f64 input is column-major")
        p.add_argument("--parallel", action="store_true", help="accepted for compatibility (no effect)")
        p.add_argument("--workers", type=int, default=0, help="accepted for compatibility (no effect)")
        if name == "discover":
            p.add_argument("--gpus", type=int, default=1, help="ranks of a torchrun job sharing the search")
            p.add_argument("--transport", choices=["p2p", "nccl"], default="p2p",
                           help="multi-GPU exchange: peer memory (default) or NCCL")
        else:
            p.add_argument("--lag", type=int, default=1)
            p.add_argument("--difference", action="store_true")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 1
    try:
        return run_discover(args) if args.cmd == "discover" else run_var_discover(args)
    except _core.Error as e:
        code = getattr(e, "code", "Error")
        print(f"error ({code}): {e}", file=sys.stderr)
        return _exit_code(code if isinstance(code, str) else "")


if __name__ == "__main__":
    sys.exit(main())
