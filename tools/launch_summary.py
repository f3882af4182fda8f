"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_summary.py gpurun_out/launches_all.csv [--md out.md]
"""
import argparse
import collections
import csv


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
        out.append((d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", ""),
                    v * scale.get(d["Metric Unit"], 1e-6)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--md")
    ap.add_argument("--title", default="")
    args = ap.parse_args()
    launches = load(args.csv)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, ms in launches:
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values())
    lines = [f"# Launch list: {args.title}", "",
             "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: shares, not absolutes).",
             "", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {v[0]} | {v[1]:.3f} | {100 * v[1] / tot:.2f}% |")
    lines.append(f"| total | {len(launches)} | {tot:.3f} | 100% |")
    text = "\n".join(lines) + "\n"
    print(text)
    if args.md:
        open(args.md, "w").write(text)


if __name__ == "__main__":
    main()
