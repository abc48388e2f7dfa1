"""ncu target: one 1080p frame per index kind on the 1024^3 blob volume."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.render import RenderTarget, render_rows

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ["lbvh", "naive"]
u8 = gen_blobs_u8((n, n, n), n=max(1, 25600 * n**3 // 1024**3), seed=7, sigma=3.0)
v = vs.Volume(u8)
tf = vs.TransferFunction.ramp(0.3)
b = vs.classify(v, tf, dilate=True)
cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=1920, height=1080)
tgt = RenderTarget(1920, 1080)
for kind in kinds:
    idx = vs.build_index(kind, b)
    render_rows(v, tf, idx, cam, tgt)
torch.cuda.synchronize()
