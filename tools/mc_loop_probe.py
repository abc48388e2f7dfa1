"""Why is the 4-channel device loop slower than its e2e loop?  (dev probe)
Times 32 sweep frames: (a) bench-style (rebuild on a side stream || render, two buffers),
(b) rebuild then render on one stream, (c) render only (fixed index), (d) public API frames."""
import sys
sys.path.insert(0, ".")
import torch
import bench as B
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.engine import LbvhRebuilder
from paper_1912_09596_b200.multichannel import classify_multi, interleaved_quads
from paper_1912_09596_b200.render import tf_device
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.tiles import TileRenderer

n, K = 1024, 32
nch = int(sys.argv[1]) if len(sys.argv) > 1 else 4
vols = [vs.Volume.from_u8(gen_blobs_u8((n, n, n), 25600, seed=7 + c, sigma=3.0)) for c in range(nch)]
if nch > 1:
    interleaved_quads(vols)
    tfs = B.channel_tfs(nch)
else:
    tfs = [[tf] for tf in B.sweep_tfs()]
cams = B.cameras(vols[0].dims)
params = torch.stack([torch.stack([tf.params() for tf in tl]) for tl in tfs])
for tl in tfs:
    for tf in tl:
        tf_device(tf, 0.5)
src = vols if nch > 1 else vols[0]
rbs = [LbvhRebuilder(src, warm=True).capture(), LbvhRebuilder(src, warm=True).capture()]
idxs = [r.index() for r in rbs]
tiles = TileRenderer(1920, 1080)
import os
st = torch.cuda.Stream(priority=int(os.environ.get("PRIO", "-1")))
sb = torch.cuda.Stream()


def render(tl, idx, cam):
    if nch > 1:
        tiles.render_multi(vols, tl, idx, cam, checked=False)
    else:
        tiles.render(vols[0], tl[0], idx, cam)
built = [torch.cuda.Event(), torch.cuda.Event()]
rendered = [torch.cuda.Event(), torch.cuda.Event()]


def timed(fn):
    torch.cuda.synchronize()
    for k in range(4):
        fn(k, B.sweep_j(k, K))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        sb.wait_stream(st)
        for k in range(K):
            fn(k, B.sweep_j(k, K))
        st.wait_stream(sb)
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


def a(k, j):
    b = k % 2
    with torch.cuda.stream(sb):
        sb.wait_event(rendered[b])
        rbs[b].rebuild(params[j])
        built[b].record(sb)
    st.wait_event(built[b])
    with torch.cuda.stream(st):
        render(tfs[j], idxs[b], cams[j])
    rendered[b].record(st)


def bb(k, j):
    with torch.cuda.stream(st):
        rbs[0].rebuild(params[j])
        render(tfs[j], idxs[0], cams[j])


def c(k, j):
    with torch.cuda.stream(st):
        render(tfs[j], idxs[0], cams[j])


def d(k, j):
    with torch.cuda.stream(st):
        tl = [vs.TransferFunction(t.lut) for t in tfs[j]]
        b = classify_multi(vols, tl, dilate=True) if nch > 1 else vs.classify(vols[0], tl[0], dilate=True)
        ix = vs.build_index("lbvh", b)
        render(tl, ix, cams[j])


for name, fn in (("a bench loop", a), ("b serial", bb), ("c render only", c), ("d public API", d),
                 ("a again", a)):
    print(f"{name:16s} {timed(fn):7.3f} ms/frame", flush=True)
