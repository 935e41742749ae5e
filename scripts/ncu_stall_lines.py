"""Per-source-line samples of ONE stall reason from an ncu report:
   python scripts/ncu_stall_lines.py report.ncu-rep stall_long_sb [N]"""
import csv, collections, io, subprocess, sys
rep, col = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = hdr = None
agg, src = collections.Counter(), {}
for r in csv.reader(io.StringIO(out)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si = hdr.index(col)
        continue
    if hdr and len(r) == len(hdr) and r[0]:
        try:
            v = float(r[si] or 0)
        except ValueError:
            continue
        k = (cur, int(r[0]))
        agg[k] += v
        src[k] = r[1]
tot = sum(agg.values()) or 1
print(col, "samples", tot)
for k, v in agg.most_common(top):
    print("%5.1f%%  %-12s:%4d  %s" % (100 * v / tot, k[0], k[1], src[k].strip()[:80]))
