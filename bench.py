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
    # transparency case (not a BASELINE config): C5's shape with Gaussian noise, where no
    # variable is identifiable and every row's k is alike -- the exact pruning's worst case
    "c5g": (2000, 10000, "sparse ER DAG (avg 2 parents), Gaussian N(0,1) noise, seed 1 (non-identifiable noise)"),
    # C5's shape with no edges at all: every variable is exchangeable and every row's k is
    # alike, the hardest case for the exact pruning
    "c5x": (2000, 10000, "2000 independent Laplace(0,1) columns (empty DAG), seed 1 (exchangeable: pruning worst case)"),
}
# SASS of the pair kernels' inner loops (cuobjdump): per EDE 16 DFMA + 9 DADD + 6 DMUL
FP64_INSTR_PER_EDE = 31   # FP64-pipe instructions (each one pipe slot: the utilisation basis)
FP64_FLOPS_PER_EDE = 47   # real flops (DFMA = 2)
LIBDEVICE_OPS_PER_EDE = 70  # SURVEY.md §8d algorithmic basis (libdevice exp/log1p)
FP64_PEAK_FALLBACK = 33.85  # DFMA TFLOP/s measured by tools/probe/fp64_peak.cu in round 1 (used if the probe fails)


def _hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 7700.0  # B200_PROFILING.md fallback


HBM_PEAK_GBS = _hbm_peak()


def pair_evals(d: int) -> int:
    return (d + 1) * d * (d - 1) // 3


def _noise_kind(name: str) -> str:
    return {"c3": "t3", "c5g": "gauss"}.get(name, "laplace")


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
    dag = plg.gen_sparse_dag(d, avg_parents=0.0 if name == "c5x" else 2.0, seed=1)
    return plg.sample_lingam(dag, n, seed=1, noise=(0.0, 1.0), kind=_noise_kind(name))


def make_input_oracle(name: str):
    """The same matrices from the oracle's generators (oracle/simgen_oracle.c, bit-identical
    to the package's, tests/test_host_cpu.py): the reference arm never loads the product.
    C4's VAR residuals are not reproduced (no oracle SVAR/QR front-end): a least-squares VAR
    residual matrix of the same shape; the per-pair CPU cost does not depend on the values."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib

    d, n, _ = CONFIGS[name]
    if name == "c1":
        return oracle_lib.sample_lingam(oracle_lib.gen_two_level_dag(d, 42000), n, 42000)
    if name == "c4":
        T = n + 1
        dag = oracle_lib.gen_sparse_dag(d, 2.0, 1, 0.1, 0.5)
        E = oracle_lib.sample_lingam(dag, T, 1, (0.0, 1.0), "laplace")
        rng = np.random.default_rng(1)
        a = rng.uniform(0.2, 0.5, size=d)
        Y = np.zeros_like(E)
        for t in range(T):
            Y[t] = E[t] + (a * Y[t - 1] if t else 0.0)
        Z = np.hstack([np.ones((T - 1, 1)), Y[:-1]])
        coef, *_ = np.linalg.lstsq(Z, Y[1:], rcond=None)
        return np.asfortranarray(Y[1:] - Z @ coef)
    dag = oracle_lib.gen_sparse_dag(d, 0.0 if name == "c5x" else 2.0, 1)
    return oracle_lib.sample_lingam(dag, n, 1, (0.0, 1.0), _noise_kind(name))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def fp64_peak(device: int):
    """DFMA TFLOP/s of this GPU measured now (tools/probe/libfp64peak.so), or the round-1
    figure if the probe is missing."""
    import ctypes

    path = os.path.join(ROOT, "tools", "probe", "libfp64peak.so")
    try:
        L = ctypes.CDLL(path)
        tf, sms = ctypes.c_double(0.0), ctypes.c_int(0)
        if L.fp64_dfma_peak(device, 5, ctypes.byref(tf), ctypes.byref(sms)) == 0 and tf.value > 0:
            return tf.value, f"measured in this job: best of 5 DFMA launches ({sms.value} SMs, tools/probe/fp64_peak_lib.cu)"
    except OSError:
        pass
    return FP64_PEAK_FALLBACK, "round-1 DFMA probe figure (in-job probe unavailable)"


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
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary
    (fallback when the in-job measurement is unavailable)."""
    prof = os.path.join(ROOT, "profiles")
    for path in sorted([os.path.join(prof, f) for f in os.listdir(prof)] if os.path.isdir(prof) else [],
                       reverse=True):
        if path.endswith(suffix):
            try:
                return json.load(open(path)).get("dram_bytes_per_launch"), os.path.relpath(path, ROOT)
            except (OSError, ValueError):
                return None, None
    return None, None


def measure_traffic(config: str, prune: bool, timeout: float = 240.0):
    """DRAM bytes (read + write) of one launch of the dominant pair kernel, measured in this
    job: ncu on a child process running the same causal order (tools/traffic_probe.py),
    profiling only launch #300 of the kernel (a large-u pruned round) or #1 (exhaustive
    round 0). Returns (bytes, note) or (None, why)."""
    kern = "prune_pairs_kernel" if prune else "pair_kernel"
    skip = 300 if prune else 0
    fd, csv = tempfile.mkstemp(suffix=".csv")
    os.close(fd)
    cmd = ["ncu", "--clock-control", "none", "--kernel-name", f"regex:{kern}", "--launch-skip", str(skip),
           "--launch-count", "1", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--csv", "--log-file", csv, sys.executable, os.path.join(ROOT, "tools", "traffic_probe.py"), config,
           "1" if prune else "0"]
    try:
        subprocess.run(cmd, timeout=timeout, check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        vals = {}
        import csv as _csv

        with open(csv) as f:
            rows = [r for r in _csv.reader(line for line in f if not line.startswith("=="))]
        hdr = rows[0]
        for r in rows[1:]:
            rec = dict(zip(hdr, r))
            vals[rec["Metric Name"]] = (float(rec["Metric Value"].replace(",", "")), rec.get("Metric Unit", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
        tot = sum(v * scale.get(u, 1) for k, (v, u) in vals.items() if k.startswith("dram__bytes"))
        return tot, f"ncu in this job: {kern} launch {skip + 1} of a {config.upper()} causal order"
    except (OSError, subprocess.SubprocessError, ValueError, KeyError, IndexError) as e:
        return None, f"in-job ncu failed ({type(e).__name__})"
    finally:
        if os.path.exists(csv):
            os.unlink(csv)


def _total_pairs(d: int, n: int, alpha: float, beta: float) -> float:
    """Cost model of a full faithful fit: sum over rounds u = d..2 of alpha u(u-1) n + beta u n
    (SURVEY.md §8d)."""
    u = np.arange(2, d + 1, dtype=np.float64)
    return float(np.sum(alpha * u * (u - 1) * n + beta * u * n))


def cpu_baseline(X: np.ndarray, target_seconds: float = 15.0, full_max_seconds: float = 90.0):
    """The reference CPU path (faithful oracle port: both residual directions per ordered
    pair, static thread partition over all host threads, -O3 -ffp-contract=off).

    Two search rounds over the first S1 < S2 columns at the full n (S2 sized for
    ~target_seconds) fit the per-round cost t(u) = alpha u(u-1) n + beta u n; a full fit
    whose predicted time is under full_max_seconds is then run and timed whole, otherwise
    its time is the cost model's extrapolation (labelled). value = P(d) / full-fit seconds."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib

    cores = os.cpu_count() or 1
    n, d = X.shape
    # the reference's own code when it was built (oracle/_ref: proj/src compiled unmodified
    # against an Eigen stand-in), else the bit-identical restatement (tests/test_oracle_kats.py)
    use_ref = oracle_lib.ref_available()
    search = oracle_lib.ref_search_causal_order if use_ref else oracle_lib.search_causal_order

    def one_round(S):
        t0 = time.perf_counter()
        search(np.asfortranarray(X[:, :S]), list(range(S)), workers=cores)
        return time.perf_counter() - t0

    S1 = min(48, d)
    t1 = one_round(S1)
    rate = S1 * (S1 - 1) / t1
    S2 = int(min(d, max(S1, (target_seconds * rate) ** 0.5)))
    if S2 > S1 + 8:
        t2 = one_round(S2)
        # t = a S(S-1) n + b S n through both points
        A = np.array([[S1 * (S1 - 1) * n, S1 * n], [S2 * (S2 - 1) * n, S2 * n]], dtype=np.float64)
        alpha, beta = np.linalg.solve(A, np.array([t1, t2]))
        if beta < 0 or alpha <= 0:  # noise: all of it per pair
            alpha, beta = t2 / (S2 * (S2 - 1) * n), 0.0
    else:
        S2, t2 = S1, t1
        alpha, beta = t1 / (S1 * (S1 - 1) * n), 0.0
    predicted = _total_pairs(d, n, alpha, beta)
    sample = (f"search rounds over the first {S1} and {S2} columns at n={n} ({t1:.1f} s + {t2:.1f} s) fit "
              f"t(u) = alpha u(u-1) n + beta u n (alpha={alpha:.3e} s, beta={beta:.3e} s)")
    if predicted <= full_max_seconds:
        t0 = time.perf_counter()
        if use_ref:
            oracle_lib.ref_causal_order(np.asfortranarray(X), True, cores)
        else:
            oracle_lib.causal_order(np.asfortranarray(X), parallel=True, workers=cores)
        wall = time.perf_counter() - t0
        how = "measured"
        sample += f"; then the whole causal order timed: {wall:.2f} s (model predicted {predicted:.2f} s)"
    else:
        wall = predicted
        how = "extrapolated"
        sample += f"; whole causal order extrapolated from the model: {wall:.0f} s"
    sample += ("; the reference's own proj/src code (oracle/_ref, compiled unmodified against an Eigen "
               "stand-in with glibc exp/log1p: Eigen3 is absent from the image)" if use_ref else
               "; faithful oracle port (bit-identical to the reference code where that is built)")
    return {"value": pair_evals(d) / wall, "unit": "pair-evals/s", "cores": cores,
            "kind": "reference" if use_ref else "port",
            "cpu_model": cpu_model(), "sample": sample, "full_fit_s": wall, "full_fit": how,
            "alpha_s": float(alpha), "beta_s": float(beta), "seconds": t1 + t2 + (wall if how == "measured" else 0)}


# Test hook (not for measurements): PLG_BENCH_SHARED_GPU=1 runs every rank of a torchrun job
# on cuda:0 with a gloo process group, so the multi-rank path (peer-memory exchange across
# processes, max-over-ranks timing, the JSON line) can be exercised on a one-GPU box.
SHARED_GPU = os.environ.get("PLG_BENCH_SHARED_GPU") == "1"


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if SHARED_GPU else int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        if SHARED_GPU:
            dist.init_process_group("gloo")
        else:
            # NCCL's INIT lines (one per rank) let the driver verify the rank count
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cpu" if SHARED_GPU else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    import torch

    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()


def run_reference(args, world, rank):
    """The reference CPU implementation of the path (faithful oracle port, all host threads)
    on the same workload; inputs from the oracle's generators, so this process never loads
    the product library. Each step = cpu_baseline()'s bounded sample."""
    if rank != 0:
        return
    d, n, desc = CONFIGS[args.config]
    X = make_input_oracle(args.config)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib

    search = oracle_lib.ref_search_causal_order if oracle_lib.ref_available() else oracle_lib.search_causal_order
    for _ in range(args.warmup):  # warm-up: one small search round (threads, page cache)
        S = min(16, d)
        search(np.asfortranarray(X[:, :S]), list(range(S)), workers=os.cpu_count() or 1)
    # each step one bounded sample; the per-step budget shrinks with K so that the whole arm
    # stays within a few minutes (the extrapolation only needs two search rounds)
    per_step = min(args.cpu_seconds, max(3.0, 90.0 / max(1, args.steps)))
    samples = [cpu_baseline(X, target_seconds=per_step) for _ in range(max(1, args.steps))]
    rate = float(np.median([s["value"] for s in samples]))
    wall = pair_evals(d) / rate
    line = {
        "metric": "causal-order pair-evals/s (and wall s) at d=2000,n=10k",
        "impl": "reference", "value": rate, "unit": "pair-evals/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall * 1e3, "causal_order_wall_s": wall,
        "wall_kind": samples[-1]["full_fit"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: {desc}",
        "config": {"workload": f"{args.config.upper()} d={d} n={n}", "d": d, "n": n},
        "cpu_baseline": {k: samples[-1][k] for k in ("unit", "cores", "kind", "sample", "cpu_model")} | {"value": rate},
        "e2e": {"value": rate, "unit": "pair-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import torch

    import paper_2403_03772_b200 as plg

    d, n, desc = CONFIGS[args.config]
    if world > 1 and args.transport == "nccl":
        import torch.distributed as dist

        obj = [plg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng = plg.Engine.distributed(local, rank, world, obj[0])
    elif world > 1:
        # peer-memory exchange: every rank maps every rank's arena (CUDA IPC over NVLink); the
        # 64-byte handles travel once through torch.distributed, the fits themselves have no
        # collective and no host synchronisation. If any rank cannot map its peers, every rank
        # falls back to the NCCL exchange (decided collectively).
        import torch.distributed as dist

        torch.cuda.set_device(local)
        eng, why = None, ""
        try:
            eng = plg.Engine.peer(local, rank, world, d)
            handle = eng.p2p_handle()
        except plg.Error as e:
            handle, why = b"", str(e)
        handles = [None] * world
        dist.all_gather_object(handles, handle)
        ok = all(len(h) == 64 for h in handles)
        if ok:
            try:
                eng.p2p_connect(handles)
            except plg.Error as e:
                ok, why = False, str(e)
        flags = [None] * world
        dist.all_gather_object(flags, ok)
        if all(flags):
            print(f"[bench] rank {rank}/{world} on cuda:{local}: peer-memory exchange, {world - 1} peer arenas "
                  f"mapped", file=sys.stderr, flush=True)
        else:
            print(f"[bench] rank {rank}: peer memory unavailable ({why or 'another rank failed'}); NCCL exchange",
                  file=sys.stderr, flush=True)
            args.transport = "nccl"
            del eng
            obj = [plg.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            eng = plg.Engine.distributed(local, rank, world, obj[0])
        dist.barrier()
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
    peak_tf, peak_src = fp64_peak(local)  # after the timed region: same clocks regime, no interference

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
    pruned = not args.no_prune
    # the pair-evaluation kernels' FP64-pipe utilisation: pipe instructions issued per second
    # (x 2, in DFMA-equivalent TFLOP/s) against the DFMA rate measured in this job
    pipe_tf = FP64_INSTR_PER_EDE * 2 * ede / (pair_s * world) / 1e12 if pair_s > 0 else None
    flops_tf = FP64_FLOPS_PER_EDE * ede / (pair_s * world) / 1e12 if pair_s > 0 else None
    traffic, traffic_src = (None, None)
    if not args.no_ncu and world == 1:
        traffic, traffic_src = measure_traffic(args.config, pruned)
    if traffic is None and args.config == "c5":  # the committed summaries are C5 launches
        why = traffic_src
        traffic, traffic_src = load_ncu_traffic("prune_pairs_ncu.json" if pruned else "pair_kernel_ncu.json")
        traffic_src = f"committed ncu --set full summary {traffic_src}" + (f" ({why})" if why else "")
    elif traffic is None:
        traffic_src = traffic_src or "not measured (--no-ncu)"
    line = {
        "metric": "causal-order pair-evals/s (and wall s) at d=2000,n=10k",
        "value": value, "unit": "pair-evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_s * 1e3 / args.steps, "causal_order_wall_s": dev_s / args.steps,
        "host_wall_ms_per_step": wall * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic: {desc}; generated on host, random DAG weights",
        "config": {"workload": f"{args.config.upper()} d={d} n={n}", "d": d, "n": n,
                   "parallelism": (f"pair lists sharded over {world} GPUs, exchanged through peer memory "
                                   f"(NVLink stores + device flag barrier, no collective)"
                                   if args.transport == "p2p" else
                                   f"pair lists sharded over {world} GPUs, one ncclAllGather per stage")
                   if world > 1 else "single GPU",
                   "l2": "input larger than L2 (FP64 matrix %.0f MB vs 126 MB L2)" % (8 * n * d / 1e6)},
        "pruning": {"enabled": pruned, "pairs_evaluated_per_step": pairs_step,
                    "pairs_exhaustive_per_step": P // 2,
                    "fraction_evaluated": pairs_step / (P // 2),
                    "executed_pair_evals_per_s": 2 * pairs_step * args.steps / dev_s,
                    "note": "exact branch and bound on each round's k: rows whose partial k (a sum of "
                            "non-negative terms) exceeds an exactly computed k cannot win; the order and "
                            "the winner's k bits equal the exhaustive rounds' (tests/test_gpu_prune.py)"},
        "roofline": {"bound": "fp64-pipe",
                     "kernel": "prune_pairs_kernel (pair lists) + pair_kernel (round 0)" if pruned
                     else "pair_kernel+finalize", "unit": "TFLOP/s",
                     "achieved": pipe_tf, "peak": peak_tf,
                     "frac": pipe_tf / peak_tf if pipe_tf else None,
                     "fp64_pipe_utilisation": pipe_tf / peak_tf if pipe_tf else None,
                     "real_flops_tflops": flops_tf,
                     "real_flops_frac": flops_tf / peak_tf if flops_tf else None,
                     "traffic": traffic,
                     "traffic_source": traffic_src,
                     "traffic_note": "dram read+write bytes of one launch of the dominant kernel; the pair "
                                     "kernels are compute-bound (L2 serves most column re-reads)",
                     "basis": f"FP64-pipe utilisation: {FP64_INSTR_PER_EDE} FP64-pipe instructions per EDE (SASS "
                              f"of both kernels' inner loops: 16 DFMA + 9 DADD + 6 DMUL) x 2 (DFMA-equivalent "
                              f"flops) over the EXECUTED EDE = 2 n x pairs evaluated; real flops "
                              f"{FP64_FLOPS_PER_EDE}/EDE reported beside it; time = CUDA events around every "
                              f"pair-evaluation launch ({pair_launches // max(1, args.steps)} per step, one extra "
                              f"untimed step); peak: {peak_src}",
                     "libdevice_basis_frac": (LIBDEVICE_OPS_PER_EDE * 2 * ede / (pair_s * world) / 1e12)
                     / peak_tf if pair_s > 0 else None,
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
    ap.add_argument("--no-ncu", action="store_true", help="skip the in-job ncu traffic measurement")
    ap.add_argument("--transport", choices=["p2p", "nccl"], default="p2p",
                    help="multi-GPU exchange: peer memory (default) or ncclAllGather")
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
