import sys; sys.path.insert(0,'.')
import torch, numpy as np
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.engine import LbvhRebuilder
from paper_1912_09596_b200.multichannel import classify_multi
from paper_1912_09596_b200.synth import gen_blobs_u8
from paper_1912_09596_b200.tiles import TileRenderer
import bench as B
n=1024
vols=[vs.Volume.from_u8(gen_blobs_u8((n,)*3, 25600, seed=7+c, sigma=3.0)) for c in range(4)]
tfs=B.channel_tfs(4); cams=B.cameras(vols[0].dims)
params = torch.stack([torch.stack([tf.params() for tf in tl]) for tl in tfs])
rb=LbvhRebuilder(vols).capture(); idx=rb.index()
tr=TileRenderer(1920,1080)
for j in (0, 32, 63):
    rb.rebuild(params[j])
    a=tr.render_multi(vols, tfs[j], idx, cams[j], checked=True).clone(); ta=tr.sample_total()
    b=tr.render_multi(vols, tfs[j], idx, cams[j], checked=False).clone(); tb=tr.sample_total()
    f=tr.multi_flags()
    pub = vs.build_index("lbvh", classify_multi(vols, tfs[j], dilate=True))
    c=tr.render_multi(vols, tfs[j], pub, cams[j], checked=True).clone(); tc=tr.sample_total()
    print(j, ta, tb, tc, f, torch.equal(a,b), torch.equal(a,c), tr._multi_target.cap)
