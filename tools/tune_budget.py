"""k_segments traversal-budget sweep (dev tool)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200 import _lib
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.render import RenderTarget, render_rows, index_desc, volume_desc, camera_desc

v = vs.Volume(gen_blobs_u8((1024,) * 3, 25600, seed=7, sigma=3.0))
cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=1920, height=1080)
for t in (0.6, 0.3, 0.0):
    tf = vs.TransferFunction.ramp(t)
    idx = vs.build_index("lbvh", vs.classify(v, tf, dilate=True))
    tgt = RenderTarget(1920, 1080)
    d, vd, cd = index_desc(idx), volume_desc(v), camera_desc(cam)
    out = []
    for bud in (1, 2, 4, 8, 1000):
        _lib.lib().vs_set_render_tuning(bud, 1)
        for _ in range(2):
            render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd)
        e1.record()
        torch.cuda.synchronize()
        out.append(f"b{bud}:{e0.elapsed_time(e1) / 5:.3f}")
    _lib.lib().vs_set_render_tuning(1, 1)
    print(t, " ".join(out), flush=True)
