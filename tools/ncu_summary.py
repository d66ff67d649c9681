"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/ncu_summary.py <round-tag> gpurun_out/prof_<op>.ncu-rep ... [--launches gpurun_out/launches.csv]
                                [--out DIR]   (default profiles/; on the GPU box write under gpurun_out/)

Writes profiles/<tag>_<op>.txt (key counters, stall reasons) per report,
profiles/<tag>_launches.txt (per-launch durations and each kernel's share),
and updates profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        res.append({h[i]: (v[i], u[i]) for i in range(min(len(h), len(v)))})
    return res


def summarise(tag, rep):
    op = os.path.basename(rep).split("_", 1)[1].replace(".ncu-rep", "")
    recs = raw(rep)
    lines = [f"# ncu --set full --clock-control none summary: {os.path.basename(rep)} ({tag})", ""]
    traffic = None
    for r in recs:
        name = r.get("Kernel Name", ("?", ""))[0]
        lines.append(f"kernel: {name}")
        for k in KEYS:
            if k in r:
                lines.append(f"  {k:70s} {r[k][0]:>20s} {r[k][1]}")
        stalls = sorted(((float(v[0]), k) for k, v in r.items()
                         if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                         and v[0] not in ("", "n/a")), reverse=True)[:8]
        lines.append("  top stall reasons (warps per issue):")
        for val, k in stalls:
            lines.append(f"    {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {val:.3f}")
        try:
            rd = float(r["dram__bytes_read.sum"][0]) * (1e6 if r["dram__bytes_read.sum"][1] == "Mbyte" else 1e9 if r["dram__bytes_read.sum"][1] == "Gbyte" else 1e3 if r["dram__bytes_read.sum"][1] == "Kbyte" else 1)
            wr = float(r["dram__bytes_write.sum"][0]) * (1e6 if r["dram__bytes_write.sum"][1] == "Mbyte" else 1e9 if r["dram__bytes_write.sum"][1] == "Gbyte" else 1e3 if r["dram__bytes_write.sum"][1] == "Kbyte" else 1)
            traffic = rd + wr
            lines.append(f"  dram traffic per launch: {traffic:.4g} B")
        except (KeyError, ValueError):
            pass
        lines.append("")
    with open(os.path.join(PROF, f"{tag}_{op}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    return op, traffic


def launches(tag, path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = {}
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list ({tag})",
             "# cold-cache, serialised: compare each kernel's SHARE, not absolute times", ""]
    for r in rows[start + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0]
            ns = float(r[vi].replace(",", ""))
            lines.append(f"{ns/1e3:12.1f} us  {name}")
            tot[name] = tot.get(name, 0.0) + ns
    s = sum(tot.values())
    lines += ["", "share of summed device time:"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"  {100*v/s:6.2f}%  {k}")
    with open(os.path.join(PROF, f"{tag}_launches.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    tag = sys.argv[1]
    args = sys.argv[2:]
    if "--out" in args:
        i = args.index("--out")
        PROF = os.path.abspath(args[i + 1])
        args = args[:i] + args[i + 2:]
    os.makedirs(PROF, exist_ok=True)
    tj = os.path.join(PROF, "ncu_traffic.json")
    if not os.path.exists(tj) and os.path.exists(os.path.join(ROOT, "profiles", "ncu_traffic.json")):
        tj_src = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    else:
        tj_src = tj
    traffic = json.load(open(tj_src)) if os.path.exists(tj_src) else {}
    if "--launches" in args:
        i = args.index("--launches")
        launches(tag, args[i + 1])
        args = args[:i] + args[i + 2:]
    for rep in args:
        op, t = summarise(tag, rep)
        if t is not None:
            traffic[op] = t
    traffic["_source"] = f"dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full ({tag})"
    json.dump(traffic, open(tj, "w"), indent=1)
