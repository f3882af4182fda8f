"""Summarise an ncu --set full report of the pair kernel into profiles/ (JSON + markdown).

    python tools/ncu_summary.py gpurun_out/pair12_c5.ncu-rep profiles/r1_pair_kernel_ncu [--note "..."]

Reads the raw page (`ncu -i … --page raw --csv`) locally; no GPU needed.
"""

import argparse
import csv
import io
import json
import subprocess


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(m, key, scale=1.0):
    v = m.get(key, ("", ""))[0].replace(",", "")
    try:
        return float(v) * scale
    except ValueError:
        return None


def to_bytes(m, key):
    v, u = m.get(key, ("", ""))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out_prefix")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    m = raw_metrics(args.rep)
    dur = num(m, "gpu__time_duration.sum")
    unit = m.get("gpu__time_duration.sum", ("", ""))[1].lower()
    dur_ms = dur * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                    "s": 1e3, "second": 1e3}.get(unit, 1e-6)
    clk = num(m, "smsp__cycles_elapsed.avg.per_second")
    clk_unit = m.get("smsp__cycles_elapsed.avg.per_second", ("", ""))[1].lower()
    clk_ghz = clk * {"ghz": 1.0, "mhz": 1e-3, "hz": 1e-9, "cycle/second": 1e-9, "cycle/nsecond": 1.0}.get(clk_unit, 1.0) \
        if clk is not None else None
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(m, k) for k in m
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(v for v in stalls.values() if v)
    summary = {
        "report": args.rep,
        "kernel": m.get("Kernel Name", ("", ""))[0] or "pair_kernel",
        "note": args.note,
        "duration_ms": dur_ms,
        "sm_clock_ghz": clk_ghz,
        "fp64_pipe_pct_of_peak": num(m, "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
        "issue_slots_busy_pct": num(m, "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "ipc_active": num(m, "sm__inst_executed.avg.per_cycle_active"),
        "warps_active_per_sm": num(m, "sm__warps_active.avg.per_cycle_active"),
        "registers_per_thread": num(m, "launch__registers_per_thread"),
        "block_size": num(m, "launch__block_size"),
        "grid_size": num(m, "launch__grid_size"),
        "dram_bytes_read": to_bytes(m, "dram__bytes_read.sum"),
        "dram_bytes_write": to_bytes(m, "dram__bytes_write.sum"),
        "l2_hit_pct": num(m, "lts__t_sector_hit_rate.pct"),
        "smem_bank_conflicts_ld": num(m, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
        "stall_share_pct": {k: round(100 * v / tot, 2) for k, v in sorted(stalls.items(), key=lambda x: -(x[1] or 0))
                            if v and tot and 100 * v / tot >= 0.5},
    }
    r, w = summary["dram_bytes_read"], summary["dram_bytes_write"]
    summary["dram_bytes_per_launch"] = (r or 0) + (w or 0) if r is not None else None
    with open(args.out_prefix + ".json", "w") as f:
        json.dump(summary, f, indent=1)
    with open(args.out_prefix + ".md", "w") as f:
        f.write(f"# ncu --set full: {summary['kernel'][:80]}\n\n{args.note}\n\n| metric | value |\n|---|---|\n")
        for k, v in summary.items():
            if k in ("stall_share_pct", "note", "kernel"):
                continue
            f.write(f"| {k} | {v} |\n")
        f.write("\nWarp stall sampling (share of samples):\n\n| reason | % |\n|---|---|\n")
        for k, v in summary["stall_share_pct"].items():
            f.write(f"| {k} | {v} |\n")
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
