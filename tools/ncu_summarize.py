"""Summarise an ncu report / launch list into profiles/ (run here, no GPU needed).

    python tools/ncu_summarize.py full   <report.ncu-rep> <kernel-key> <out.json> [<name regex>]
    python tools/ncu_summarize.py launches <launches.csv> <out.json>

`full` extracts the metrics the roofline uses (DRAM bytes, duration, FP64 pipe,
occupancy, stall mix, SASS opcode mix) and merges them under <kernel-key> into
<out.json>; `launches` aggregates a gpu__time_duration launch list by kernel.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import Counter, defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum", "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * scale.get(unit, 1)


def full(rep, key, out, kfilter=None):
    sel = ["-k", "regex:" + kfilter] if kfilter else []
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, *sel, "--page", "raw", "--csv"))))
    h, units = rows[0], rows[1]
    launches = []
    for vals in rows[2:]:
        d = {}
        for i, name in enumerate(h):
            if name in KEYS or "issue_stalled" in name and name.endswith("per_issue_active.ratio"):
                try:
                    d[name] = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                if name.startswith("dram__bytes") or name.startswith("lts__t_bytes"):
                    d[name] = to_bytes(vals[i].replace(",", ""), units[i])
                if name == "gpu__time_duration.sum":
                    d[name] = float(vals[i]) * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
                                                "ms": 1e-3, "msecond": 1e-3}.get(units[i], 1e-9)
        d["kernel"] = vals[h.index("Kernel Name")] if "Kernel Name" in h else ""
        launches.append(d)
    # SASS opcode mix from the source page
    src = list(csv.reader(io.StringIO(ncu("-i", rep, *sel, "--page", "source", "--csv",
                                          "--print-source", "sass"))))
    mix = Counter()
    if len(src) > 2:
        hh = src[1]
        iS, iE = hh.index("Source"), hh.index("Instructions Executed")
        for r in src[2:]:
            if len(r) < len(hh) or not r[iS].split():
                continue
            toks = r[iS].split()
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            if not (r[iE] or "0").isdigit():
                continue  # a repeated header
            mix[op.split(".")[0]] += int(r[iE] or 0)
    tot = sum(mix.values()) or 1
    L = launches[0]
    summary = {
        "report": os.path.basename(rep),
        "kernel": L.get("kernel"),
        "duration_s": L.get("gpu__time_duration.sum"),
        "dram_bytes_read": L.get("dram__bytes_read.sum"),
        "dram_bytes_write": L.get("dram__bytes_write.sum"),
        "dram_bytes_per_launch": (L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)),
        "metrics": {k: v for k, v in L.items() if k != "kernel"},
        "sass_mix": {k: round(v / tot, 4) for k, v in mix.most_common(12)},
    }
    data = json.load(open(out)) if os.path.exists(out) else {}
    data[key] = summary
    json.dump(data, open(out, "w"), indent=1)
    print(json.dumps(summary, indent=1))


def launches(path, out):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    h = rows[0]
    agg = defaultdict(list)
    for r in rows[1:]:
        if len(r) == len(h) and r[h.index("Metric Name")] == "gpu__time_duration.sum":
            agg[r[h.index("Kernel Name")]].append(float(r[h.index("Metric Value")]))
    tot = sum(sum(v) for v in agg.values())
    res = {k: {"launches": len(v), "mean_ns": sum(v) / len(v), "share": sum(v) / tot}
           for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}
    json.dump({"source": os.path.basename(path), "kernels": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5] if len(sys.argv) > 5 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
