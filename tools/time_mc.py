"""4-channel 1080p render timing at fixed TFs (dev tool): median of 5 x 10 frames.
usage: time_mc.py [N]"""
import statistics
import sys
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.multichannel import classify_multi, interleaved_quads
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.tiles import TileRenderer

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
nb = max(1, 25600 * n ** 3 // 1024 ** 3)
vols = [vs.Volume.from_u8(gen_blobs_u8((n, n, n), n=nb, seed=7 + c, sigma=3.0)) for c in range(4)]
interleaved_quads(vols)
tiles = TileRenderer(1920, 1080)
cam = vs.Camera.orbit(vols[0].dims, 30.0, 15.0, width=1920, height=1080)
for t in (0.6, 0.3, 0.0):
    tfs = [vs.TransferFunction.ramp(t) for _ in range(4)]
    idx = vs.build_index("lbvh", classify_multi(vols, tfs, dilate=True))
    tiles.render_multi(vols, tfs, idx, cam)
    reps = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            tiles.render_multi(vols, tfs, idx, cam, checked=False)
        b.record()
        torch.cuda.synchronize()
        reps.append(a.elapsed_time(b) / 10)
    print(f"t={t} 4-channel {statistics.median(reps):7.3f} ms  samples {tiles.sample_total()}",
          flush=True)
