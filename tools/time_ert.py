"""1080p LBVH frame with and without early ray termination (dev tool)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.render import RenderTarget, render_rows, index_desc, volume_desc, camera_desc

v = vs.Volume.from_u8(gen_blobs_u8((1024,) * 3, 25600, seed=7, sigma=3.0))
cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=1920, height=1080)
for t in (0.6, 0.3, 0.0):
    tf = vs.TransferFunction.ramp(t)
    idx = vs.build_index("lbvh", vs.classify(v, tf, dilate=True))
    d, vd, cd = index_desc(idx), volume_desc(v), camera_desc(cam)
    res = {}
    for eps in (0.0, 1e-3):
        tgt = RenderTarget(1920, 1080, want_rgba64=True)
        for _ in range(2):
            render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd, ert_eps=eps)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd, ert_eps=eps)
        e1.record()
        torch.cuda.synchronize()
        res[eps] = (e0.elapsed_time(e1) / 5, int(tgt.total.item()), tgt.rgba64.clone())
    err = float((res[1e-3][2] - res[0.0][2]).abs().max())
    print(f"t={t} parity {res[0.0][0]:.3f} ms ({res[0.0][1]} samples)  ert1e-3 {res[1e-3][0]:.3f} ms "
          f"({res[1e-3][1]} samples)  max|dRGBA| {err:.2e}", flush=True)
