"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel count and mean (us)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"]) / (1000.0 if d["Metric Unit"] == "ns" else 1.0)
        agg.setdefault(d["Kernel Name"].split("(")[0][:70], []).append(v)
tot = 0.0
for k, v in agg.items():
    print(f"{len(v):4d} x {sum(v)/len(v):9.1f} us  {k}")
