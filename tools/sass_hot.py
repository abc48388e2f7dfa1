"""Hot SASS of one kernel from an ncu report (dev tool):
usage: sass_hot.py report.ncu-rep kernel_regex [n]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if len(r) > 3)
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[hi + 1:]:
    if len(r) < len(hdr):
        continue
    try:
        ex = float(r[ix["Instructions Executed"]] or 0)
        st = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    data.append((r[ix["Address"]], r[ix["Source"]], ex, st))
tot_ex = sum(d[2] for d in data) or 1
tot_st = sum(d[3] for d in data) or 1
print(f"instructions {tot_ex:.0f}  stall samples {tot_st:.0f}")
mode = sys.argv[4] if len(sys.argv) > 4 else "seq"
if mode == "seq":
    for a, s, ex, st in data:
        if ex / tot_ex > 0.002 or st / tot_st > 0.004:
            print(f"{a:>6s} {100*ex/tot_ex:5.2f}% ex {100*st/tot_st:5.2f}% st  {s[:90]}")
else:
    for a, s, ex, st in sorted(data, key=lambda d: -d[3])[:n]:
        print(f"{a:>6s} {100*ex/tot_ex:5.2f}% ex {100*st/tot_st:5.2f}% st  {s[:90]}")
