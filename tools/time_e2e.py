"""Split of the public-API frame loop (dev tool): host wall time per step component."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.tiles import TileRenderer

n = 1024
v = vs.Volume.from_u8(gen_blobs_u8((n, n, n), 25600, seed=7, sigma=3.0))
luts = [vs.TransferFunction.ramp(0.6 - 0.6 * k / 63).lut for k in range(64)]
cams = [vs.Camera.orbit(v.dims, 360.0 * k / 64, 15.0, width=1920, height=1080) for k in range(64)]
tr = TileRenderer(1920, 1080)
acc = np.zeros(5)
K = 32
for k in range(K + 3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tf = vs.TransferFunction(luts[k % 64])
    t1 = time.perf_counter()
    b = vs.classify(v, tf, dilate=True)
    idx = vs.build_index("lbvh", b)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    fr = tr.frame(v, tf, idx, cams[k % 64])
    t4 = time.perf_counter()
    if k >= 3:
        acc += [t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0]
print("per step ms: tf %.3f  classify+build (host) %.3f  build drain %.3f  frame %.3f  total %.3f"
      % tuple(acc / K * 1e3))
