"""Writes a compact text summary of an ncu report (speed-of-light, occupancy,
stall reasons, DRAM bytes, tensor pipe, top source lines) for profiles/."""
import csv, io, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
lines = []
det = run("--page", "details", "--csv")
keep = ("Duration", "Throughput", "Registers", "Occupancy", "Warp Cycles Per Issued", "Ipc",
        "Grid Size", "Block Size", "Shared Memory", "Avg. Active Threads", "Branch Efficiency",
        "Hit Rate", "Block Limit")
rows = list(csv.reader(io.StringIO(det)))
if rows:
    h = rows[0]
    ks, km, ku, kv = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    for r in rows[1:]:
        if len(r) > kv and any(k in r[km] for k in keep):
            lines.append(f"{r[ks][:36]:36s} | {r[km]:40s} | {r[ku]:12s} | {r[kv]}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
d = dict(zip(raw[0], raw[2]))
lines.append("")
for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "smsp__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active"):
    if k in d:
        lines.append(f"{k} = {d[k]} {raw[1][raw[0].index(k)]}")
st = sorted(((float(d[k]), k) for k in raw[0] if k.startswith("smsp__average_warps_issue_stalled_")
             and k.endswith("_per_issue_active.ratio") and d.get(k) not in (None, "")), reverse=True)
lines.append("stall reasons (warps per issue):")
lines += [f"  {v:7.3f} {k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')}" for v, k in st[:10]]
lines.append("")
lines.append(subprocess.run([sys.executable, "scripts/ncu_lines.py", rep, "30"], capture_output=True,
                            text=True).stdout)
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:60]))
