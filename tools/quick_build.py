"""Quick build timing (dev tool): every index kind on a synthetic blob volume."""
import sys, time, json
sys.path.insert(0, ".")
import torch
import paper_1912_09596_b200 as vs
from paper_1912_09596_b200.synth import gen_blobs_u8

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else list(vs.INDEX_KINDS)[1:]
ts = [float(t) for t in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0.3]
u8 = gen_blobs_u8((n, n, n), n=max(1, 25600 * n**3 // 1024**3), seed=7, sigma=3.0)
v = vs.Volume(u8)
out = {}
for t in ts:
    tf = vs.TransferFunction.ramp(t)
    for kind in kinds:
        times = []
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            b = vs.classify(v, tf, dilate=True)
            idx = vs.build_index(kind, b)
            st = vs.report_stats(idx)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        out[f"{kind}@{t}"] = {"ms": min(times) * 1e3, **st}
        print(kind, t, out[f"{kind}@{t}"], flush=True)
print(json.dumps(out))
