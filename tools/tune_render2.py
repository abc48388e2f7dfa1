"""Fused vs two-phase rendering at 1080p for several TFs (dev tool)."""
import sys, json
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200 import _lib
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.render import RenderTarget, render_rows, index_desc, volume_desc, camera_desc

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["lbvh", "grid", "naive"]
ts = [float(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0.3]
u8 = gen_blobs_u8((n, n, n), n=max(1, 25600 * n**3 // 1024**3), seed=7, sigma=3.0)
v = vs.Volume(u8)
cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=1920, height=1080)
res = {}
for t in ts:
    tf = vs.TransferFunction.ramp(t)
    b = vs.classify(v, tf, dilate=True)
    for kind in kinds:
        idx = vs.build_index(kind, b)
        d = index_desc(idx); vd = volume_desc(v); cd = camera_desc(cam)
        for opts, cap, tb in [(1, 32, 1)]:
            _lib.lib().vs_set_render_options(opts)  # noqa
            _lib.lib().vs_set_render_tuning(tb, 1)
            tgt = RenderTarget(1920, 1080, seg_cap=cap)
            render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 3
            res[f"{kind} t={t} opts={opts} cap={cap} tb={tb}"] = (ms, int(tgt.total.item()))
            print(kind, t, "opts", opts, "cap", cap, "tb", tb, round(ms, 2), int(tgt.total.item()), flush=True)
print(json.dumps(res))
