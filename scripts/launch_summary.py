"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        k = r[hdr.index("Kernel Name")].replace("cmtfb::", "")[:90]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        u = r[hdr.index("Metric Unit")]
        v *= {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(u, 1.0)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{t:10.2f} ms  x{n:3d}  {k}")
