"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel name, count and mean / total device time (us)."""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0]
    v = float(r[iv].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "nsecond"
    us = v / 1e3 if unit.startswith("n") else (v * 1e3 if unit.startswith("m") else v)
    agg.setdefault(name, []).append(us)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:40s} n={len(v):5d} mean {sum(v)/len(v):10.2f} us  total {sum(v):12.1f} us  {100*sum(v)/tot:5.1f} %")
