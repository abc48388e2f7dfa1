"""Quick render timing (dev tool): 1080p frame of a synthetic volume through each index."""
import sys, time, json
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.render import RenderTarget, render_rows, index_desc, volume_desc, camera_desc

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
W, H = (1920, 1080)
u8 = gen_blobs_u8((n, n, n), n=max(1, 25600 * n**3 // 1024**3), seed=7, sigma=3.0)
v = vs.Volume(u8)
tf = vs.TransferFunction.ramp(0.3)
b = vs.classify(v, tf, dilate=True)
out = {}
for kind in ["lbvh", "grid", "naive"]:
    idx = vs.build_index(kind, b)
    cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=W, height=H)
    tgt = RenderTarget(W, H)
    d = index_desc(idx); vd = volume_desc(v); cd = camera_desc(cam)
    for _ in range(2):
        render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 5
    e0.record()
    for _ in range(K):
        render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    s = int(tgt.total.item())
    out[kind] = {"ms": ms, "fps": 1e3 / ms, "samples": s, "Msamples_s": s / ms / 1e3}
    print(kind, out[kind], flush=True)
print(json.dumps(out))
