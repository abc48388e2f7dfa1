"""Lattice-range counts per ray (dev tool): how many rays overflow the segment buffer."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.render import RenderTarget, render_rows

v = vs.Volume.from_u8(gen_blobs_u8((1024,) * 3, 25600, seed=7, sigma=3.0))
cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=1920, height=1080)
for t in (0.6, 0.3, 0.0):
    tf = vs.TransferFunction.ramp(t)
    b = vs.classify(v, tf, dilate=True)
    for kind in ("lbvh", "grid"):
        idx = vs.build_index(kind, b)
        tgt = RenderTarget(1920, 1080)
        render_rows(v, tf, idx, cam, tgt)
        torch.cuda.synchronize()
        npix = 1920 * 1080
        counts = tgt.ws[npix * tgt.seg_cap * 8: npix * tgt.seg_cap * 8 + npix * 4].view(torch.int32)
        c = counts.float()
        print(f"t={t} {kind}: mean {c.mean():.1f} max {int(c.max())} >16 {(c > 16).float().mean():.4f} "
              f">32 {(c > 32).float().mean():.4f} >64 {(c > 64).float().mean():.4f}", flush=True)
