"""ncu target: one k-d build (dev tool).  usage: prof_kd.py N kind t"""
import sys
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8

n, kind, t = int(sys.argv[1]), sys.argv[2], float(sys.argv[3])
v = vs.Volume.from_u8(gen_blobs_u8((n, n, n), max(1, 25600 * n**3 // 1024**3), seed=7, sigma=3.0))
tf = vs.TransferFunction.ramp(t)
b = vs.classify(v, tf, dilate=True)
b.packed()
torch.cuda.synchronize()
import time
for rep in range(int(sys.argv[4]) if len(sys.argv) > 4 else 2):  # first: warm-up
    t0 = time.perf_counter()
    idx = vs.build_index(kind, b)
    torch.cuda.synchronize()
    print("build ms", round((time.perf_counter() - t0) * 1e3, 3), vs.report_stats(idx), flush=True)
