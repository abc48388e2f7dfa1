"""ncu target: one 1080p frame per index kind on the 1024^3 blob volume.
usage: prof_render.py N kinds [threshold] [seg_cap]"""
import sys
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.render import RenderTarget, render_rows

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["lbvh", "naive"]
t = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
cap = int(sys.argv[4]) if len(sys.argv) > 4 else 16
u8 = gen_blobs_u8((n, n, n), n=max(1, 25600 * n**3 // 1024**3), seed=7, sigma=3.0)
v = vs.Volume.from_u8(u8)
tf = vs.TransferFunction.ramp(t)
b = vs.classify(v, tf, dilate=True)
cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=1920, height=1080)
tgt = RenderTarget(1920, 1080, seg_cap=cap)
for kind in kinds:
    idx = vs.build_index(kind, b)
    render_rows(v, tf, idx, cam, tgt)
torch.cuda.synchronize()
