"""Summarise ncu outputs into profiles/: a launch list (per-kernel share of
device time) and the key metrics of a --set full capture."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Theoretical Occupancy", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Executed Instructions", "Dynamic Shared Memory Per Block",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Grid Size"]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[h + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0].replace("void ", "")
            tot[name] += float(r[vi].replace(",", ""))
            cnt[name] += 1
    all_ns = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "total_us": round(v / 1e3, 2),
             "avg_us": round(v / cnt[k] / 1e3, 2), "share": round(v / all_ns, 4)}
            for k, v in sorted(tot.items(), key=lambda kv: -kv[1])]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    res = {}
    rd = csv.reader(io.StringIO(out))
    hdr = next(rd)
    for r in rd:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in KEYS:
            res[d["Metric Name"]] = f'{d["Metric Value"]} {d.get("Metric Unit", "")}'.strip()
            res["kernel"] = d.get("Kernel Name", "")[:120]
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rd = list(csv.reader(io.StringIO(raw)))
    if len(rd) > 2:
        hdr, units, vals = rd[0], rd[1], rd[2]
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                  "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                  "smsp__sass_inst_executed_op_shared_ld.sum",
                  "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                  "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                  "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                  "gpu__time_duration.sum", "launch__registers_per_thread",
                  "sm__warps_active.avg.pct_of_peak_sustained_active"):
            if m in hdr:
                i = hdr.index(m)
                res[m] = f"{vals[i]} {units[i]}"
    return res


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if mode == "launches" else full(path), indent=1))
