"""Benchmark: DirectLiNGAM causal-order search (arXiv 2403.03772 hot path) on B200.

Metric (BASELINE.json): causal-order wall seconds and pair-evaluations/s at d=2000,
n=10000 (config C5), on N GPUs, beside the reference CPU path on the host cores.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c5]
    torchrun --nproc-per-node N bench.py --gpus N ...       (one process per GPU)

A step is one full causal_order over the synthetic matrix. `value` is measured with the
matrix already resident in HBM (device time from CUDA events on the engine stream, max
over ranks); `e2e` is the same metric through the public API with the matrix in pinned
host memory (H2D copy and D2H of the order inside the timed region).
pair-evals = P(d) = (d+1) d (d-1) / 3 ordered (i, j) evaluations of Alg. 1 per fit: the
reference's work for the same order, so value = P(d) / wall is reference-equivalent. The
engine's exact pruning (prune_kernels.cu) evaluates only the pairs that decide each round's
argmin; `pruning` reports how many it actually evaluated, and the roofline is computed on
those executed evaluations. --no-prune times the exhaustive rounds instead.
"""

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (d, n, generator description)
    "c1": (10, 1000, "two-level DAG (gen_two_level_dag), U(0,1) noise, seed 42000"),
    "c2": (100, 10000, "sparse ER DAG (avg 2 parents, |w| in [0.5,1.5]), Laplace(0,1) noise, seed 1"),
    "c3": (1000, 10000, "sparse ER DAG (avg 2 parents), Student-t3 noise, seed 1 (Perturb-seq shaped)"),
    "c4": (500, 2499, "VarLiNGAM lag 1: residuals of a d=500, T=2500 SVAR (sparse B0, diagonal B1, Laplace noise)"),
    "c5": (2000, 10000, "sparse ER DAG (avg 2 parents, |w| in [0.5,1.5]), Laplace(0,1) noise, seed 1"),
}
FP64_OPS_PER_EDE = 31     # FP64-pipe instructions per EDE in the pair kernel inner loop (cuobjdump SASS)
LIBDEVICE_OPS_PER_EDE = 70  # SURVEY.md §8d algorithmic basis (libdevice exp/log1p)
FP64_PEAK_TFLOPS = 33.85  # measured DFMA microbenchmark on this pool's B200 (tools/probe/fp64_peak.cu)


def _hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 7700.0  # B200_PROFILING.md fallback


HBM_PEAK_GBS = _hbm_peak()


def pair_evals(d: int) -> int:
    return (d + 1) * d * (d - 1) // 3


def make_input(name: str):
    import paper_2403_03772_b200 as plg

    d, n, _ = CONFIGS[name]
    if name == "c1":
        dag = plg.gen_two_level_dag(d, seed=42000)
        return plg.sample_lingam(dag, n, seed=42000)
    if name == "c4":  # same generator as tests/golden/make_golden.py c4_series()
        b0 = plg.gen_sparse_dag(d, avg_parents=2.0, seed=1, wmin=0.1, wmax=0.5)
        b1 = np.asfortranarray(np.diag(plg.uniform_vector(d, 1, 0.2, 0.5)))
        X = plg.sample_svar(b0, [b1], T=2500, burn_in=500, seed=1, noise=(0.0, 1.0), kind="laplace")
        return plg.estimate_var(X, 1)[1]
    kind = "t3" if name == "c3" else "laplace"
    dag = plg.gen_sparse_dag(d, avg_parents=2.0, seed=1)
    return plg.sample_lingam(dag, n, seed=1, noise=(0.0, 1.0), kind=kind)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=10)

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        except OSError:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = np.array([float(r[1]) for r in rows])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(float(r[2]) for r in rows)),
                "reasons": reasons, "samples": len(rows),
                "power_w_max": float(max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit()))}


def load_ncu_traffic(suffix):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    for path in sorted(
            [os.path.join(ROOT, "profiles", f) for f in os.listdir(os.path.join(ROOT, "profiles"))]
            if os.path.isdir(os.path.join(ROOT, "profiles")) else [], reverse=True):
        if path.endswith(suffix):
            try:
                return json.load(open(path)).get("dram_bytes_per_launch")
            except (OSError, ValueError):
                return None
    return None


def cpu_baseline(X: np.ndarray, target_seconds: float = 15.0):
    """The reference CPU path (faithful oracle port: both residual directions per ordered
    pair, static thread partition, -O3 -ffp-contract=off) on a bounded sample: one search
    round over the first S columns at the full n, S sized for ~target_seconds."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib

    cores = os.cpu_count() or 1
    n = X.shape[0]
    S = min(48, X.shape[1])
    t0 = time.perf_counter()
    oracle_lib.search_causal_order(np.asfortranarray(X[:, :S]), list(range(S)), workers=cores)
    dt = time.perf_counter() - t0
    rate = S * (S - 1) / dt
    S2 = int(min(X.shape[1], max(S, (target_seconds * rate) ** 0.5)))
    if S2 > S:
        t0 = time.perf_counter()
        oracle_lib.search_causal_order(np.asfortranarray(X[:, :S2]), list(range(S2)), workers=cores)
        dt = time.perf_counter() - t0
        rate = S2 * (S2 - 1) / dt
        S = S2
    return {"value": rate, "unit": "pair-evals/s", "cores": cores, "kind": "port",
            "sample": f"one search round over the first {S} columns at n={n} ({S * (S - 1)} ordered pair-evals, "
                      f"{dt:.1f} s); faithful oracle (reference cannot build: Eigen3 absent)",
            "seconds": dt}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    import torch

    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()


def run_reference(args, world, rank):
    if rank != 0:
        return
    d, n, desc = CONFIGS[args.config]
    X = make_input(args.config)
    for _ in range(args.warmup if args.warmup < 1 else 1):
        pass
    samples = [cpu_baseline(X, target_seconds=args.cpu_seconds) for _ in range(max(1, args.steps))]
    rate = float(np.median([s["value"] for s in samples]))
    wall = pair_evals(d) / rate
    line = {
        "metric": "causal-order pair-evals/s (and wall s) at d=2000,n=10k",
        "impl": "reference", "value": rate, "unit": "pair-evals/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall * 1e3, "wall_s_extrapolated": wall,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: {desc}",
        "config": {"workload": f"{args.config.upper()} d={d} n={n}", "d": d, "n": n},
        "cpu_baseline": {k: samples[-1][k] for k in ("unit", "cores", "kind", "sample")} | {"value": rate},
        "e2e": {"value": rate, "unit": "pair-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import torch

    import paper_2403_03772_b200 as plg

    d, n, desc = CONFIGS[args.config]
    if world > 1:
        import torch.distributed as dist

        obj = [plg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng = plg.Engine.distributed(local, rank, world, obj[0])
    else:
        torch.cuda.set_device(local)
        eng = plg.Engine(local)
    eng.set_prune(not args.no_prune)
    X = make_input(args.config)
    dX = torch.from_numpy(np.ascontiguousarray(X.T)).to(f"cuda:{local}")  # column j contiguous
    ptr = dX.data_ptr()
    for _ in range(args.warmup):
        order = eng.causal_order_device(ptr, n, d, n)
    barrier(world)

    dev_ms, launches, pairs_done = [], 0, 0
    with ClockSampler(local) as clocks:
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            order = eng.causal_order_device(ptr, n, d, n)
            st = eng.stats()
            dev_ms.append(st["total_ms"])
            launches += st["launches"]
            pairs_done += st["pairs_evaluated"]
        barrier(world)
        wall = time.perf_counter() - t0
    clk = clocks.summary()
    dev_s = allreduce_max(sum(dev_ms) / 1e3, world)
    wall = allreduce_max(wall, world)
    # one more (untimed) step with per-launch CUDA events: the pair-evaluation and
    # residualisation launch times behind the rooflines (their events would otherwise add
    # ~1% to the timed steps)
    eng.set_detail_timing(True)
    eng.causal_order_device(ptr, n, d, n)
    st = eng.stats()
    eng.set_detail_timing(False)
    pair_ms = [st["pair_ms"] * args.steps]
    pair_launches = st["pair_launches"] * args.steps
    resid_ms = st["resid_ms"] * args.steps
    resid_bytes = st["resid_bytes"] * args.steps
    P = pair_evals(d)
    value = P * args.steps / dev_s

    # e2e: the public API with the matrix in pinned host memory
    pinned = torch.empty((d, n), dtype=torch.float64, pin_memory=True)
    pinned.copy_(torch.from_numpy(np.ascontiguousarray(X.T)))
    Xh = pinned.numpy().T  # F-contiguous (n, d) view, zero-copy into the binding
    e2e_orders = []
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_orders.append(eng.causal_order(Xh))
    barrier(world)
    e2e_s = allreduce_max(time.perf_counter() - t0, world)
    st_e2e = eng.stats()
    assert all(o == order for o in e2e_orders), "host and device entry points disagree"

    if rank != 0:
        return
    pair_s = sum(pair_ms) / 1e3 / args.steps
    # executed work: every evaluated unordered pair computes both residual entropies over n
    pairs_step = pairs_done / args.steps
    ede = 2 * n * pairs_step
    # the pair-evaluation kernels' share of the step and their FP64-pipe roofline
    achieved = FP64_OPS_PER_EDE * 2 * ede / (pair_s * world) / 1e12 if pair_s > 0 else None
    pruned = not args.no_prune
    line = {
        "metric": "causal-order pair-evals/s (and wall s) at d=2000,n=10k",
        "value": value, "unit": "pair-evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_s * 1e3 / args.steps, "causal_order_wall_s": dev_s / args.steps,
        "host_wall_ms_per_step": wall * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: {desc}; generated on host, random DAG weights",
        "config": {"workload": f"{args.config.upper()} d={d} n={n}", "d": d, "n": n,
                   "parallelism": f"pair tiles sharded over {world} GPU(s), one ncclAllGather per round"
                   if world > 1 else "single GPU",
                   "l2": "input larger than L2 (FP64 matrix %.0f MB vs 126 MB L2)" % (8 * n * d / 1e6)},
        "pruning": {"enabled": pruned, "pairs_evaluated_per_step": pairs_step,
                    "pairs_exhaustive_per_step": P // 2,
                    "fraction_evaluated": pairs_step / (P // 2),
                    "executed_pair_evals_per_s": 2 * pairs_step * args.steps / dev_s,
                    "note": "exact branch and bound on each round's k: rows whose partial k (a sum of "
                            "non-negative terms) exceeds an exactly computed k cannot win; the order and "
                            "the winner's k bits equal the exhaustive rounds' (tests/test_gpu_prune.py)"},
        "roofline": {"bound": "fp64",
                     "kernel": "prune_pairs_kernel (pair lists) + pair_kernel (round 0)" if pruned
                     else "pair_kernel+finalize", "unit": "TFLOP/s",
                     "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                     "frac": achieved / FP64_PEAK_TFLOPS if achieved else None,
                     "traffic": load_ncu_traffic("prune_pairs_ncu.json" if pruned else "pair_kernel_ncu.json"),
                     "traffic_note": "dram read+write bytes of one launch of the dominant kernel (ncu --set full, "
                                     "profiles/); algorithmic bytes: one pass over the listed pairs' columns "
                                     "per launch — compute-bound, L2 serves the re-reads",
                     "basis": f"{FP64_OPS_PER_EDE} FP64-pipe instructions per EDE (SASS of both kernels' inner "
                              f"loops) x 2 flops over the EXECUTED EDE = 2 n x pairs evaluated; time = CUDA "
                              f"events around every pair-evaluation launch ({pair_launches // max(1, args.steps)} "
                              f"per step, one extra untimed step); peak = measured DFMA rate (no FP64 figure in "
                              f"MEASURED_PEAKS.json)",
                     "libdevice_basis_frac": (LIBDEVICE_OPS_PER_EDE * 2 * ede / (pair_s * world) / 1e12)
                     / FP64_PEAK_TFLOPS if pair_s > 0 else None,
                     "pair_share_of_step": pair_s / (dev_s / args.steps),
                     "residualize": {
                         "bound": "hbm", "kernel": "resid_ent_kernel (residualisation + next round's column "
                                                   "entropies, fused)",
                         "unit": "GB/s", "achieved": resid_bytes / (resid_ms / 1e3) / 1e9 if resid_ms > 0 else None,
                         "peak": HBM_PEAK_GBS,
                         "frac": (resid_bytes / (resid_ms / 1e3) / 1e9) / HBM_PEAK_GBS if resid_ms > 0 else None,
                         "bytes_per_step": resid_bytes / args.steps,
                         "share_of_step": resid_ms / 1e3 / dev_s,
                         "note": "algorithmic bytes (2(u-1)+1) n 8 per round (read + write of the u-1 "
                                 "remaining columns, one read of the root); the same pass evaluates "
                                 "(u-1) n EDE of column entropies, so the kernel is not purely HBM-bound"}},
        "e2e": {"value": P * args.steps / e2e_s, "unit": "pair-evals/s",
                "h2d_bytes_per_step": int(st_e2e["h2d_bytes"]), "d2h_bytes_per_step": int(st_e2e["d2h_bytes"]),
                "wall_s_per_step": e2e_s / args.steps},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(X, target_seconds=args.cpu_seconds)
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c5")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-prune", action="store_true", help="exhaustive rounds (every pair, every round)")
    args = ap.parse_args()
    world, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
