"""Per-kernel / host-gap breakdown of one public-API k-d / hybrid rebuild (dev tool):
torch.profiler (CUPTI) over classify+build_index after warm-up.
usage: kd_breakdown.py N KIND T"""
import sys
import time

sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8

n, kind, t = int(sys.argv[1]), sys.argv[2], float(sys.argv[3])
v = vs.Volume.from_u8(gen_blobs_u8((n, n, n), max(1, 25600 * n**3 // 1024**3), seed=7, sigma=3.0))
tf = vs.TransferFunction.ramp(t)
for _ in range(3):
    vs.report_stats(vs.build_index(kind, vs.classify(v, tf, dilate=True)))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    ix = vs.build_index(kind, vs.classify(v, tf, dilate=True))
    vs.report_stats(ix)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
print(f"{n} {kind} t={t}: wall {wall*1e3:.3f} ms")
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t00 = evs[0].time_range.start if evs else 0
show = int(sys.argv[4]) if len(sys.argv) > 4 else 40
for e in evs[:show]:
    print(f"  {e.time_range.start - t00:9.1f} +{e.time_range.end - e.time_range.start:8.1f} us  {e.name[:70]}")
agg = {}
for e in evs:
    k = e.name[:60]
    c, d = agg.get(k, (0, 0.0))
    agg[k] = (c + 1, d + e.time_range.end - e.time_range.start)
print(f"  device span {evs[-1].time_range.end - t00:.1f} us; busy {sum(d for _, d in agg.values()):.1f} us")
for k, (c, d) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
    print(f"  {d:9.1f} us {c:5d}x  {k}")
