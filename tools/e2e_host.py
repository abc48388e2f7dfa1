import sys, time
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.tiles import TileRenderer
n = 1024
v = vs.Volume.from_u8(gen_blobs_u8((n, n, n), 25600, seed=7, sigma=3.0))
luts = [vs.TransferFunction.ramp(0.6 - 0.6 * k / 63).lut for k in range(64)]
cams = [vs.Camera.orbit(v.dims, 360.0 * k / 64, 15.0, width=1920, height=1080) for k in range(64)]
tr = TileRenderer(1920, 1080)
bs = torch.cuda.Stream()
import collections
acc = collections.defaultdict(float)
def step(k, side):
    t0 = time.perf_counter()
    ctx = torch.cuda.stream(bs) if side else torch.cuda.stream(torch.cuda.current_stream())
    with ctx:
        tf = vs.TransferFunction(luts[k % 64]); t1 = time.perf_counter()
        b = vs.classify(v, tf, dilate=True); t2 = time.perf_counter()
        idx = vs.build_index("lbvh", b); t3 = time.perf_counter()
    if side: torch.cuda.current_stream().wait_stream(bs)
    p = tr.frame_async(v, tf, idx, cams[k % 64]); t4 = time.perf_counter()
    acc["tf"] += t1 - t0; acc["classify"] += t2 - t1; acc["build"] += t3 - t2; acc["frame_async"] += t4 - t3
    return p, (tf, b, idx)
for side in (False, True):
    for k in range(3): step(k, side)[0].result()
    torch.cuda.synchronize()
    acc.clear()
    K = 48
    t0 = time.perf_counter()
    pend = None
    w = 0.0
    for k in range(K):
        nxt = step(k, side)
        if pend:
            a = time.perf_counter(); pend[0].result(); w += time.perf_counter() - a
        pend = nxt
    pend[0].result()
    tot = time.perf_counter() - t0
    print("side" if side else "same", "per step ms total %.3f  result-wait %.3f  " % (tot / K * 1e3, w / K * 1e3) +
          "  ".join(f"{k} {v / K * 1e3:.3f}" for k, v in acc.items()), flush=True)
