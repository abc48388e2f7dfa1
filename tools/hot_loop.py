"""Hot SASS lines of a kernel in address order, with executed counts and stall samples
(dev tool).  usage: hot_loop.py report.ncu-rep kernel_regex [fraction_of_max=0.3]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
frac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass",
                      "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
seen, data = set(), []
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or r[0] in seen:
        continue
    seen.add(r[0])
    try:
        data.append((int(r[0], 16), r[ix["Source"]].strip(), int(r[ix["Instructions Executed"]]),
                     int(r[ix["Warp Stall Sampling (All Samples)"]])))
    except ValueError:
        continue
tot = sum(d[2] for d in data)
tst = sum(d[3] for d in data)
mx = max(d[2] for d in data)
hot = sorted(d for d in data if d[2] >= mx * frac)
print(f"instructions {tot}  stall samples {tst}  hot lines {len(hot)} "
      f"({sum(d[2] for d in hot) / tot:.1%} of instructions, {sum(d[3] for d in hot) / tst:.1%} of stalls)")
for a, src, ie, st in hot:
    print(f"{a & 0xffff:5x} {ie:10d} {st:6d} {st / tst:6.1%}  {src}")
