"""Attribute ncu per-SASS stall samples to CUDA source lines (via nvdisasm -g)."""
import csv, io, re, subprocess, sys, collections, glob
rep, kern, cubin = sys.argv[1], sys.argv[2], sys.argv[3]
per_unit = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
sass = [(float(r[si] or 0), float(r[ii] or 0), r[1]) for r in rows[2:] if len(r) > ii]
lst = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*\.section\s+\.text\.", lst)
best = None
for fb in funcs:
    name = fb.split(",")[0].strip()
    ins, cur = [], None
    for line in fb.split("\n"):
        lm = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', line)
        if lm:
            cur = f"{lm.group(1)}:{lm.group(2)}"
        if re.match(r"\s*/\*[0-9a-f]{4,}\*/", line):
            ins.append(cur)
    if kern in name and abs(len(ins) - len(sass)) <= 4:
        if best is None or abs(len(ins) - len(sass)) < abs(len(best[1]) - len(sass)):
            best = (name, ins)
if best is None:
    sys.exit(f"no matching function ({len(sass)} sass rows)")
agg_s, agg_i = collections.Counter(), collections.Counter()
for (s, n, txt), loc in zip(sass, best[1]):
    agg_s[loc] += s
    agg_i[loc] += n
tot = sum(agg_s.values()) or 1
print("function", best[0], "instr/unit total", sum(agg_i.values()) / per_unit)
for loc, v in agg_s.most_common(40):
    line = ""
    if loc:
        f, l = loc.split(":")
        try:
            line = open(f"/root/repo/paper_1708_08640_b200/csrc/{f}").read().split("\n")[int(l) - 1].strip()[:70]
        except Exception:
            pass
    print(f"{100*v/tot:5.1f}%  inst/unit={agg_i[loc]/per_unit:8.1f}  {str(loc):18s} {line}")
