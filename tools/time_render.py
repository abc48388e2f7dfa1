"""1080p render timing per index kind / TF / renderer option set (dev tool).
usage: time_render.py N [kinds] [thresholds] [opts,...]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200 import _lib
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.render import RenderTarget, render_rows, index_desc, volume_desc, camera_desc

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["lbvh", "grid", "naive"]
ts = [float(t) for t in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0.6, 0.3, 0.0]
opts = [int(o) for o in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1, 3]
W, H = 1920, 1080
v = vs.Volume.from_u8(gen_blobs_u8((n, n, n), n=max(1, 25600 * n**3 // 1024**3), seed=7, sigma=3.0))
cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=W, height=H)
for t in ts:
    tf = vs.TransferFunction.ramp(t)
    b = vs.classify(v, tf, dilate=True)
    for kind in kinds:
        idx = vs.build_index(kind, b)
        res = {}
        tgt = RenderTarget(W, H, want_rgba64=True)
        d, vd, cd = index_desc(idx), volume_desc(v), camera_desc(cam)
        for o in opts:
            for _ in range(2):
                render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd, flags=o)
            torch.cuda.synchronize()
            K, reps = 10, []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(K):
                    render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd, flags=o)
                e1.record()
                torch.cuda.synchronize()
                reps.append(e0.elapsed_time(e1) / K)
            res[o] = (sorted(reps)[2], int(tgt.total.item()), tgt.rgba64.clone())
        same = all(torch.equal(res[o][2], res[opts[0]][2]) for o in opts)
        s = res[opts[0]][1]
        print(f"t={t} {kind:6s} samples {s:11d}  " +
              "  ".join(f"opt{o} {res[o][0]:7.3f} ms" for o in opts) +
              f"  ({s / res[opts[0]][0] / 1e6:6.1f} Gsamples/s)  equal={same}", flush=True)
