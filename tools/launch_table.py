"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) of
`tools/run_one.py --repeat R` into a per-kernel table for the LAST repeat (one e^H).

The repeats are split at the launches of `k_validate` (the first kernel of every plan).
Usage: python tools/launch_table.py gpurun_out/launches.csv [title] > profiles/....md
"""
import csv
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        rows.append((r["Kernel Name"], float(r["Metric Value"]) * (1e-6 if r["Metric Unit"] == "ns" else 1e-3)))
    starts = [i for i, (k, _) in enumerate(rows) if k.startswith("k_validate")]
    last = rows[starts[-1]:] if starts else rows
    agg = OrderedDict()
    for k, ms in last:
        name = k.split("(")[0]
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + ms)
    tot = sum(t for _, t in agg.values())
    print(f"### {title}\n")
    print("Serialised, cold-cache per-launch times (ncu `--metrics gpu__time_duration.sum "
          "--clock-control none`): compare shares, not absolutes.\n")
    print("| kernel | launches | ms | share |\n|---|---|---|---|")
    for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {c} | {t:.2f} | {100 * t / tot:.1f} % |")
    print(f"| total | {sum(c for c, _ in agg.values())} | {tot:.1f} | |")


if __name__ == "__main__":
    main()
