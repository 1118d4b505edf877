"""Summarise ncu captures for profiles/ (run on the CPU box; ncu -i reads the reports).

    python tools/summarize_ncu.py gpurun_out/prof.ncu-rep [...] > profiles/rNN_kernel.md
    python tools/summarize_ncu.py --launches gpurun_out/launches.csv > profiles/rNN_launches.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy", "Registers Per Thread",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Executed Instructions", "Issue Slots Busy", "Dynamic Shared Memory Per Block",
        "Block Limit Registers", "Block Limit Shared Mem"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg",
       "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def summarize(rep):
    out = [f"### {rep}", ""]
    det = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "details", "--csv"]))))
    if det:
        h = det[0]
        ki = h.index("Kernel Name")
        mi, ui, vi = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
        kern = det[1][ki] if len(det) > 1 else "?"
        out.append(f"kernel: `{kern}`")
        out.append("")
        out.append("| metric | value | unit |")
        out.append("|---|---|---|")
        seen = set()
        for r in det[1:]:
            if r[mi] in KEYS and r[mi] not in seen:
                seen.add(r[mi])
                out.append(f"| {r[mi]} | {r[vi]} | {r[ui]} |")
    raw = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    if len(raw) > 2:
        h, units, v = raw[0], raw[1], raw[2]
        out += ["", "| raw counter | value | unit |", "|---|---|---|"]
        for k in RAW:
            if k in h:
                i = h.index(k)
                out.append(f"| {k} | {v[i]} | {units[i]} |")
        stalls = []
        for k, x, u in zip(h, v, units):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(x), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        stalls.sort(reverse=True)
        out += ["", "top stall reasons (pc sampling share): " +
                ", ".join(f"{k} {100 * s / tot:.0f}%" for s, k in stalls[:6])]
    out.append("")
    return "\n".join(out)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                 "msecond": 1.0, "s": 1e3, "second": 1e3}.get(r[ui].strip(), 1.0)
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", "")) * scale
        cnt[name] += 1
    allms = sum(tot.values())
    out = [f"### launch list {path}", "",
           f"{sum(cnt.values())} launches, {allms:.1f} ms total (ncu, serialised, cold caches)", "",
           "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.append(f"| `{k}` | {cnt[k]} | {tot[k]:.1f} | {100 * tot[k] / allms:.1f}% |")
    out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        for rep in sys.argv[1:]:
            print(summarize(rep))
