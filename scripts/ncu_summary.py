"""Summarise an ncu report: SOL, occupancy, top stall reasons, hottest SASS lines."""
import csv, io, subprocess, sys
rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else ""
def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))
rows = page("details")
hdr = rows[0]
ki, si, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Value", "Metric Unit"))
keep = {"Duration", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L2 Cache Throughput", "L1/TEX Cache Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "Active Warps Per Scheduler", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"}
for r in rows[1:]:
    if kern in r[ki] and r[mi] in keep:
        print(f"  {r[mi]:40s} {r[vi]} {r[ui]}")
raw = page("raw")
h = raw[0]
for r in raw[2:]:
    if kern not in r[h.index("Kernel Name")]:
        continue
    vals = []
    for name, v in zip(h, r):
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                vals.append((float(v.replace(",", "")), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in vals) or 1
    print("  stall reasons:", ", ".join(f"{n} {100*v/tot:.1f}%" for v, n in sorted(vals, reverse=True)[:8]))
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
                 "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                 "smsp__inst_executed_op_shared_ld.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
                 "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active"):
        if name in h:
            print(f"  {name:60s} {r[h.index(name)]} {raw[1][h.index(name)]}")
    break
src = page("source", ["--kernel-name", f"regex:{kern}"] if kern else [])
if len(src) > 2:
    hdr = src[1]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in src[2:]:
        try:
            data.append((float(r[si]), r[1][:100]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    data.sort(reverse=True)
    print("  hottest SASS:")
    seen = 0
    for v, s in data[:24:2]:
        print(f"    {100*v/tot:5.1f}%  {s}")
