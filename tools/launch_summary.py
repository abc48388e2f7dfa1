"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum): per-kernel count / us."""
import collections
import csv
import sys

U = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        k = r[ki].split("(")[0]
        if k.startswith("void at::") or k.startswith("at::"):
            continue
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", "")) * U.get(r[ui], 0)
    print(path, "total us %.1f" % sum(v[1] for v in agg.values()))
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
        print("   %-44s %5d %9.1f" % (k[:44], v[0], v[1]))
