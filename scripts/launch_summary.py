"""Summarise an ncu --csv launch list by kernel: total gpu__time_duration and, if present,
DRAM read+write bytes per launch (development aid for profiles/)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
idi = hdr.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    if r[mi] == "gpu__time_duration.sum":
        v = v / 1000.0 if u in ("ns", "nsecond") else (v if u in ("us", "usecond") else v * 1000.0)
    elif u.lower() in ("kbyte", "kb"):
        v *= 1e3
    elif u.lower() in ("mbyte", "mb"):
        v *= 1e6
    elif u.lower() in ("gbyte", "gb"):
        v *= 1e9
    per[r[idi]][r[mi]] = v
    names[r[idi]] = r[ki].split("(")[0]
agg = collections.OrderedDict()
for lid, mets in per.items():
    nm = names[lid]
    c, t, b = agg.get(nm, (0, 0.0, 0.0))
    agg[nm] = (c + 1, t + mets.get("gpu__time_duration.sum", 0.0),
               b + mets.get("dram__bytes_read.sum", 0.0) + mets.get("dram__bytes_write.sum", 0.0))
tot = sum(t for _, t, _ in agg.values())
print(f"total {tot:.1f} us over {sum(c for c, _, _ in agg.values())} launches")
for nm, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    extra = f"  dram {b / c / 1e6:8.2f} MB/launch ({b / (t * 1e-6) / 1e9:7.0f} GB/s)" if b else ""
    print(f"{t:9.1f} us {100 * t / tot:5.1f}%  {c:3d}x  {nm}{extra}")
