"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.OrderedDict()
tot = 0.0
for r in rows[hdr_i + 1:]:
    if len(r) <= vi: continue
    v = float(r[vi].replace(",", "")); u = r[ui]
    us = v / 1000.0 if u in ("ns", "nsecond") else (v if u in ("us", "usecond") else v * 1000.0)
    name = r[ki].split("(")[0]
    c, t = agg.get(name, (0, 0.0)); agg[name] = (c + 1, t + us); tot += us
print(f"total {tot:.1f} us over {sum(c for c,_ in agg.values())} launches")
for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.1f} us {100*t/tot:5.1f}%  {c:4d}x  {name}")
