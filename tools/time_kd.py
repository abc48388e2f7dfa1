"""Wall-clock k-d / hybrid rebuild times (dev tool): median of R builds after one warm-up.
usage: time_kd.py [N ...]"""
import statistics
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8

sizes = [int(a) for a in sys.argv[1:]] or [512, 1024]
import os

KINDS = os.environ.get("KINDS", "kd-shallow kd-deep-mls32 kd-deep-mls128 kd-binned-mls32 hybrid").split()
for n in sizes:
    v = vs.Volume.from_u8(gen_blobs_u8((n, n, n), max(1, 25600 * n**3 // 1024**3), seed=7, sigma=3.0))
    for t in (0.6, 0.3, 0.0):
        b = vs.classify(v, vs.TransferFunction.ramp(t), dilate=True)
        b.packed()
        torch.cuda.synchronize()
        for kind in KINDS:
            if n > 512 and kind.startswith("kd-deep"):
                continue
            vs.build_index(kind, b)
            ts = []
            for _ in range(5):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                idx = vs.build_index(kind, b)
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            st = vs.report_stats(idx)
            print(f"{n} t={t} {kind:16s} {statistics.median(ts)*1e3:8.2f} ms  "
                  f"nodes {st['node_count']} height {st['height']}", flush=True)
