"""Summarise `ncu --set full` captures into the JSON files kept under profiles/.

    python profiles/extract_ncu.py gpurun_out/prof_win6.ncu-rep \
        window_fwd=k_window_fwd window_bwd=k_window_bwd  [--out profiles/r01_ncu_full_metrics.json]

Each NAME=REGEX picks the first kernel of the report whose name matches REGEX
and records the metrics below (value, unit).  With --out the entries are merged
into that file, and `profiles/traffic.json` (DRAM bytes read+write per launch,
read by bench.py) is updated for the same names.
"""

from __future__ import annotations

import csv
import io
import json
import os
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__warps_eligible.avg.per_cycle_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]
STALL = re.compile(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio")


def kernels(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        res.append({h: (v, u) for h, v, u in zip(hdr, r, units)})
    return res


def summarise(k: dict) -> dict:
    d = {"Kernel Name": k["Kernel Name"][0]}
    for m in METRICS:
        if m in k:
            d[m] = list(k[m])
    stalls = {}
    for name, (v, _) in k.items():
        mt = STALL.fullmatch(name)
        if mt:
            try:
                x = float(v)
            except ValueError:
                continue
            if x >= 0.05:
                stalls[mt.group(1)] = round(x, 3)
    d["stall_cycles_per_issued_instruction"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    return d


def to_bytes(v: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    return float(v) * scale


def main(argv):
    out = None
    if "--out" in argv:
        i = argv.index("--out")
        out = argv[i + 1]
        argv = argv[:i] + argv[i + 2:]
    rep, picks = argv[0], [a.split("=", 1) for a in argv[1:]]
    ks = kernels(rep)
    res = {}
    for name, rx in picks:
        k = next(k for k in ks if re.search(rx, k["Kernel Name"][0]))
        res[name] = summarise(k)
        res[name]["source_report"] = os.path.basename(rep)
    if out is None:
        print(json.dumps(res, indent=1))
        return
    cur = json.load(open(out)) if os.path.exists(out) else {}
    cur.update(res)
    json.dump(cur, open(out, "w"), indent=1)
    tpath = os.path.join(os.path.dirname(out), "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for name, d in res.items():
        rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
        traffic[name] = round(to_bytes(*rd) + to_bytes(*wr))
    json.dump(traffic, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
