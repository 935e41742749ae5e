"""Append the headline ncu counters of a report's kernel to a profiles/*.json
table the bench reads (roofline.traffic / ncu):
    python scripts/ncu_metrics_json.py report.ncu-rep "<key>" profiles/ncu_r2_metrics.json [kernel-substr]"""
import csv, io, json, os, subprocess, sys
rep, key, out = sys.argv[1], sys.argv[2], sys.argv[3]
kern = sys.argv[4] if len(sys.argv) > 4 else ""
raw = list(csv.reader(io.StringIO(subprocess.run(
    ["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
h, units = raw[0], raw[1]
row = next(r for r in raw[2:] if kern in r[h.index("Kernel Name")])
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "sm__inst_executed.avg.per_cycle_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__warps_eligible.avg.per_cycle_active"]
d = json.load(open(out)) if os.path.exists(out) else {}
ent = {"report": f"gpurun_out/{os.path.basename(rep)} (ncu --set full --clock-control none)",
       "kernel": row[h.index("Kernel Name")]}
for w in want:
    if w in h:
        v = row[h.index(w)].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        u = units[h.index(w)]
        # bytes in MB like the round-1 table (the bench multiplies by 1e6)
        if w.startswith("dram__bytes"):
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}.get(u, 1.0)
            v, u = v * scale, "Mbyte"
        ent[w] = {"value": v, "unit": u}
d[key] = ent
json.dump(d, open(out, "w"), indent=1)
print(key, {k: v for k, v in ent.items() if k.startswith("dram") or k.startswith("gpu")})
