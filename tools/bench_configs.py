"""Every BASELINE.json config on one B200 (dev/evidence tool; bench.py is the driver contract).

configs[0] 64^3   LBVH build + 256x256 render
configs[1] 256^3  LBVH vs macro grid: build + 1024x1024 render
configs[2] 512^3  SVT sweep k-d (shallow, deep mls32/mls128), binned k-d, LBVH: 3 TFs
configs[3] 1024^3 hybrid vs LBVH: per-TF rebuild + 1920x1080 render
Builds: TF-change rebuild (classify + build), device-synchronised, median of 5 after warm-up.
Renders: mean of 3 frames at az 30 / el 15 (dt 0.5, trilinear), samples per frame.
Writes one JSON document to stdout."""
import json
import statistics
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.render import RenderTarget, camera_desc, index_desc, render_rows, volume_desc
from paper_1912_09596_b200.synth import gen_blobs_u8

CONFIGS = [
    ("configs[0]", 64, 16, [0.3], ["lbvh", "grid"], (256, 256)),
    ("configs[1]", 256, 400, [0.3], ["lbvh", "grid"], (1024, 1024)),
    ("configs[2]", 512, 3200, [0.6, 0.3, 0.0],
     ["lbvh", "grid", "kd-shallow", "kd-deep-mls32", "kd-deep-mls128", "kd-binned-mls32", "hybrid"],
     (1024, 1024)),
    ("configs[3]", 1024, 25600, [0.6, 0.3, 0.0], ["lbvh", "grid", "hybrid", "kd-shallow",
                                                 "kd-binned-mls32"], (1920, 1080)),
]


def timed_build(v, tf, kind, reps=5):
    times = []
    idx = None
    for r in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        idx = vs.build_index(kind, vs.classify(v, tf, dilate=True))
        st = vs.report_stats(idx)
        torch.cuda.synchronize()
        if r:
            times.append(time.perf_counter() - t0)
    return idx, statistics.median(times) * 1e3, st


def timed_render(v, tf, idx, w, h, reps=3):
    cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=w, height=h)
    tgt = RenderTarget(w, h)
    d, vd, cd = index_desc(idx), volume_desc(v), camera_desc(cam)
    render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        render_rows(v, tf, idx, cam, tgt, idx_desc=d, vol_desc=vd, cam_desc=cd)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, int(tgt.total.item())


out = {"device": torch.cuda.get_device_name(0), "configs": []}
for name, n, nb, ts, kinds, (w, h) in CONFIGS:
    v = vs.Volume.from_u8(gen_blobs_u8((n, n, n), nb, seed=7, sigma=3.0))
    for t in ts:
        tf = vs.TransferFunction.ramp(t)
        occ = 100.0 * vs.occupancy(vs.classify(v, tf))
        rec = {"config": name, "dims": n, "blobs": nb, "ramp_t": t, "occupancy_pct": occ,
               "viewport": [w, h], "kinds": {}}
        for kind in ["naive"] + kinds:
            idx, bms, st = (None, 0.0, {"node_count": 0, "height": 0}) if kind == "naive" else \
                timed_build(v, tf, kind, reps=3 if n >= 512 else 5)
            rms, samples = timed_render(v, tf, idx, w, h)
            rec["kinds"][kind] = {"rebuild_ms": bms, **st, "render_ms": rms,
                                  "fps": 1e3 / rms, "samples": samples,
                                  "Msamples_s": samples / rms / 1e3}
            print(name, t, kind, rec["kinds"][kind], file=sys.stderr, flush=True)
        out["configs"].append(rec)
    del v
    torch.cuda.empty_cache()
print(json.dumps(out))
