"""Per-source-line warp-stall samples from an ncu report (--import-source, -lineinfo):
   python scripts/ncu_src_lines.py report.ncu-rep [N] [stall-column-substring]"""
import csv, collections, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = hdr = None
agg, ins, src = collections.Counter(), collections.Counter(), {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        try:
            v = float(r[si] or 0)
        except ValueError:
            continue
        k = (cur, int(r[0]))
        agg[k] += v
        src[k] = r[1]
        try:
            ins[k] += float(r[ii] or 0)
        except ValueError:
            pass
tot = sum(agg.values()) or 1
print("total stall samples", tot)
for k, v in agg.most_common(top):
    print("%5.1f%%  %-12s:%4d  inst %.2e  %s" % (100 * v / tot, k[0], k[1], ins[k], src[k].strip()[:72]))
