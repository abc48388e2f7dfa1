import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8
v = vs.Volume.from_u8(gen_blobs_u8((1024,)*3, 25600, seed=7, sigma=3.0))
cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=1920, height=1080)
for t in (0.6, 0.3, 0.0):
    tf = vs.TransferFunction.ramp(t)
    idx = vs.build_index("lbvh", vs.classify(v, tf, dilate=True))
    rgba, samples = vs.render_float(v, tf, idx, cam)
    a = rgba[..., 3]
    print(t, "alpha>=0.999:", float((a >= 0.999).mean()), "alpha>=0.99:", float((a>=0.99).mean()), "mean A", float(a.mean()), "samples", int(samples.sum()))
