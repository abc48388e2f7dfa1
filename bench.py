#!/usr/bin/env python
"""Benchmark: interactive transfer-function editing on a synthetic 1024^3 u8 volume (B200).

One step = one interactive TF-change frame, the reference's Session loop (service.py:53-125,
set_tf -> classify -> build_index -> render_frame) on BASELINE.json configs[3]/[4]:

  1. the next TF of a 64-entry ramp sweep (thresholds 0.6 -> 0) reaches the device as a
     64-byte parameter block;
  2. LBVH rebuild: vs_classify_summary (one pass over the u8 volume) -> vs_summary_to_bitmap
     -> vs_lbvh_from_bitmap -> vs_lbvh_brick_grid, replayed as one CUDA graph;
  3. 1920x1080 render through the new index (camera orbiting 360/64 deg per step, dt 0.5,
     trilinear, FP64 parity arithmetic), rows split in interleaved stripes over the ranks and
     gathered with one NCCL all-gather (N > 1).
  Frames are pipelined over two index buffers: frame k+1's rebuild runs on a side stream while
  frame k renders (each render waits for its own rebuild; each rebuild for the render that
  last used its buffer).

  value     frames/s of the whole job, device-timed with CUDA events, max over ranks; volume
            and the sweep's TF tables resident in HBM; input 1 GiB > 126 MB L2.
  e2e       the same frame through the public API (TransferFunction -> classify ->
            build_index -> TileRenderer.frame) with the TF uploaded from pinned host memory
            and the frame's pixels read back to the host every step.
  roofline  k_brick_summary, the HBM-bound kernel of the step (the rebuild's compulsory
            traffic: N^3 u8 read + 4 B/brick summary write over its CUDA-event duration).  The
            render kernel is issue-bound, not HBM/tensor-bound; see "render" and DESIGN.md.
  cpu_baseline  the C oracle port of the reference path (oracle/vs_oracle.c): rebuild at full
            size (1 core) + a row sample of the frame render (all cores), scaled to a frame.

`--impl reference` times that CPU oracle port alone (rank 0; other ranks exit at once).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "hierarchy build ms and render frames/s (Msamples/s) vs CPU ref; % HBM roofline"
FALLBACK_HBM_GBS = 6650.0
W, H = 1920, 1080
NSWEEP = 64
ERT_EPS = 5e-4  # opt-in early ray termination of the "ert" key (north-star RGBA tolerance 1e-3)


def sweep_tfs(k: int = NSWEEP):
    from paper_1912_09596_b200.volume import TransferFunction

    return [TransferFunction.ramp(threshold=0.6 - 0.6 * i / 63) for i in range(k)]


def cameras(dims, k: int = NSWEEP):
    from paper_1912_09596_b200.render import Camera

    return [Camera.orbit(dims, 360.0 * i / k, 15.0, width=W, height=H) for i in range(k)]


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            for key in ("hbm_gbs", "hbm_GBps", "hbm"):
                if key in d:
                    return float(d[key]), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:7]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------------------------------
# CPU reference: the C oracle port of the reference path (oracle/vs_oracle.c; test
# infrastructure -- executed only by --impl reference and the cpu_baseline leg, after the
# GPU arm's timed regions)
# ------------------------------------------------------------------------------------------

class OracleFrames:
    """Full, unscaled interactive frames on the host: classify(dilate) + flag_bricks +
    build_lbvh for the step's TF, then the 1920x1080 render through THAT tree -- the same
    work as one GPU step, on every host core the box has."""

    def __init__(self, u8_host: np.ndarray, threads: int | None = None):
        from oracle import oracle as O

        self.O = O
        self.u8 = u8_host
        self.threads = threads or os.cpu_count() or 1
        O.set_threads(self.threads)

    def frame(self, lut, cam) -> dict:
        O = self.O
        t0 = time.perf_counter()
        bits, _ = O.classify(self.u8, lut, dilate=True)
        coords, codes = O.flag_bricks(bits, 8)
        del bits
        tree = O.build_lbvh(coords, codes, 8, self.u8.shape)
        t1 = time.perf_counter()
        _, samples = O.render("lbvh", self.u8, lut, tree, cam, nthreads=self.threads)
        t2 = time.perf_counter()
        return {"frame_s": t2 - t0, "rebuild_s": t1 - t0, "render_s": t2 - t1,
                "samples": int(samples.sum()), "n_bricks": len(coords)}


def profile_value(name: str, key: str):
    """(value, file) of ``key`` in the newest profiles/r??_<name> (ncu summaries committed
    with the round), or (None, None)."""
    for p in sorted((ROOT / "profiles").glob(f"r??_{name}"), reverse=True):
        try:
            d = json.loads(p.read_text())
        except Exception:
            continue
        if d.get(key) is not None:
            return d[key], f"profiles/{p.name}"
    return None, None


def sweep_j(k: int, steps: int) -> int:
    """Sweep entry of timed step k: the K timed steps stride over the whole 64-TF sweep
    (t = 0.6 -> 0) and the 360-degree orbit whatever K is."""
    return (k * NSWEEP) // max(steps, 1) % NSWEEP


def sweep_desc(steps: int) -> dict:
    js = sorted({sweep_j(k, steps) for k in range(steps)})
    t = [round(0.6 - 0.6 * j / 63, 4) for j in js]
    return {"tfs_timed": len(js), "t_first": t[0], "t_last": t[-1],
            "stride": "j = floor(64 k / steps): every timed step k uses sweep TF j and orbit "
                      "view j"}


# ------------------------------------------------------------------------------------------

def dist_setup():
    import torch
    import torch.distributed as dist

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # VSB200_DIST_BACKEND=gloo: test mode for the N > 1 code path on a single GPU (ranks share
    # the device, frames gathered through host copies); the driver's runs use NCCL
    backend = os.environ.get("VSB200_DIST_BACKEND", "nccl")
    if torch.cuda.is_available():
        local = local % torch.cuda.device_count() if backend == "gloo" else local
        torch.cuda.set_device(local)
    if ws > 1 and not dist.is_initialized():
        if backend == "gloo" or not torch.cuda.is_available():
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, ws, local


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def make_volume(n: int):
    from paper_1912_09596_b200.synth import gen_blobs_u8

    nblobs = max(1, 25600 * n ** 3 // 1024 ** 3)
    return gen_blobs_u8((n, n, n), n=nblobs, seed=7, sigma=3.0), nblobs


def run_reference(args, rank, ws):
    """--impl reference: the oracle port of the reference path on the box's host cores (the
    reference is Python/numba; nothing of it compiles to an oracle/_ref).  Every step is one
    full, unscaled frame of the same workload as the GPU arm: the step's sweep TF is
    classified and its LBVH built at 1024^3, and the 1920x1080 frame is rendered through that
    tree from the step's orbit view.  Rank 0 alone runs (no process group); others exit."""
    if rank != 0:
        return
    n = args.size
    u8d, nblobs = make_volume(n)
    u8 = u8d.cpu().numpy()
    del u8d
    tfs = sweep_tfs()
    cams = cameras(u8.shape)
    of = OracleFrames(u8)
    for k in range(args.warmup):
        of.frame(tfs[k % NSWEEP].lut, cams[k % NSWEEP])
    t0 = time.perf_counter()
    runs = [of.frame(tfs[sweep_j(k, args.steps)].lut, cams[sweep_j(k, args.steps)])
            for k in range(args.steps)]
    wall = time.perf_counter() - t0
    frame_s = wall / args.steps
    value = 1.0 / frame_s
    sample = (f"{args.steps} full {W}x{H} frames at {n}^3 (no scaling): per step the sweep "
              f"TF's classify+flag_bricks+build_lbvh and the render through that tree, "
              f"{of.threads} host threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": frame_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8+f64", "data": "synthetic",
        "config": workload_config(n, nblobs, args.steps),
        "build_ms": 1e3 * statistics.mean(r["rebuild_s"] for r in runs),
        "render_ms": 1e3 * statistics.mean(r["render_s"] for r in runs),
        "timed_region_s": wall,
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": of.threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(n, nblobs, steps):
    return {"workload": f"interactive TF sweep on {n}^3 u8 blobs ({nblobs} blobs, sigma 3, "
                        f"seed 7): LBVH rebuild + {W}x{H} render per frame, 64 ramp TFs "
                        f"t=0.6..0, orbit camera el 15, dt 0.5",
            "frame": "rebuild+render", "brick": 8, **sweep_desc(steps)}


def run_ours(args, rank, ws, local):
    import torch

    import paper_1912_09596_b200 as vs
    from paper_1912_09596_b200.engine import LbvhRebuilder, tf_params_device
    from paper_1912_09596_b200.render import (RenderTarget, camera_desc, index_desc, render_rows,
                                              tf_device, volume_desc)
    from paper_1912_09596_b200.tiles import TileRenderer, shard_presence

    n = args.size
    u8, nblobs = make_volume(n)
    v = vs.Volume.from_u8(u8)
    if ws > 1:
        shard_presence(v)  # the once-per-volume presence pass split by brick x-slabs + all-gather
    tfs = sweep_tfs()
    cams = cameras(v.dims)
    params = tf_params_device(tfs)
    for tf in tfs:
        tf_device(tf, 0.5)  # LUT + opacity-correction tables resident for the sweep
    # two index buffers: frame k+1's rebuild (side stream) overlaps frame k's render.  The
    # volume is resident across the sweep, so TF changes take the warm rebuild (per-volume
    # brick presence masks, SURVEY.md §8d "warm = subsequent"); the cold engine (one-pass
    # volume summary) is timed beside it for the HBM roofline
    rbs = [LbvhRebuilder(v, warm=True).capture(), LbvhRebuilder(v, warm=True).capture()]
    rb = rbs[0]
    rbc = LbvhRebuilder(v).capture()
    idxs = [r.index() for r in rbs]
    ids = [index_desc(i) for i in idxs]
    idx = idxs[0]
    tiles = TileRenderer(W, H)
    vd = volume_desc(v)
    cds = [camera_desc(c) for c in cams]
    # renders on a high-priority stream, rebuilds on a default-priority one: the rebuild's
    # blocks fill the SMs the render leaves idle instead of delaying it
    st = torch.cuda.Stream(priority=-1) if os.environ.get("VSB200_PRIO", "1") == "1" \
        else torch.cuda.current_stream()
    st.wait_stream(torch.cuda.current_stream())
    sb = torch.cuda.Stream()
    built = [torch.cuda.Event(), torch.cuda.Event()]
    rendered = [torch.cuda.Event(), torch.cuda.Event()]

    def step(k, j, ert=0.0):
        b = k % 2
        with torch.cuda.stream(sb):
            sb.wait_event(rendered[b])        # buffer b free: frame k-2 rendered
            rbs[b].rebuild(params[j])
            built[b].record(sb)
        st.wait_event(built[b])
        with torch.cuda.stream(st):
            img = tiles.render(v, tfs[j], idxs[b], cams[j], idx_desc=ids[b], vol_desc=vd,
                               cam_desc=cds[j], ert_eps=ert)
        rendered[b].record(st)
        return img

    # ---- device-resident loop (value) ------------------------------------------------------
    with torch.cuda.stream(st):
        for k in range(args.warmup):
            step(k, k % NSWEEP)
        torch.cuda.synchronize()
        barrier(ws)
        with ClockSampler(local) as clk:
            time.sleep(0.3)
            torch.cuda.synchronize()
            barrier(ws)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            sb.wait_stream(st)
            for k in range(args.steps):
                step(k, sweep_j(k, args.steps))
            st.wait_stream(sb)
            e1.record(st)
            torch.cuda.synchronize()
            total_ms = e0.elapsed_time(e1)
            # the same loop with the opt-in early ray termination (north star: "front-to-back
            # compositing and early ray termination"; not the headline, which is the
            # reference's integrator bit for bit)
            torch.cuda.synchronize()
            e0.record(st)
            sb.wait_stream(st)
            for k in range(args.steps):
                step(k, sweep_j(k, args.steps), ert=ERT_EPS)
            st.wait_stream(sb)
            e1.record(st)
            torch.cuda.synchronize()
            ert_total_ms = e0.elapsed_time(e1)
            # component split (not the headline): rebuild alone, summary kernel alone, render alone
            bev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(3)]
            reps = max(10, min(args.steps, 100))
            for e, engine in zip(bev, (rb, rbc)):  # warm, cold
                e[0].record(st)
                for k in range(reps):
                    engine.rebuild(params[sweep_j(k, reps)])
                e[1].record(st)
            votes = []  # the warm vote kernel alone (the HBM-bound kernel of the timed step)
            for k in range(reps):
                rb.set_tf(params[sweep_j(k, reps)])
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                rb.launch_vote(st.cuda_stream)
                b.record(st)
                rb.launch_build(st.cuda_stream)
                votes.append((a, b))
            summ = []
            for k in range(reps):
                rbc.set_tf(params[sweep_j(k, reps)])
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                rbc.launch_summary(st.cuda_stream)
                b.record(st)
                rbc.launch_tree(st.cuda_stream)
                summ.append((a, b))
            # render alone at the sparse / medium / dense TF (the reference's App. B view)
            render_by_t, ert_by_t = {}, {}
            for t in (0.6, 0.3, 0.0):
                tft = vs.TransferFunction.ramp(t)
                ridx = vs.build_index("lbvh", vs.classify(v, tft, dilate=True))
                rcam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=W, height=H)
                rdesc, rcd = index_desc(ridx), camera_desc(rcam)
                tiles.render(v, tft, ridx, rcam, idx_desc=rdesc, vol_desc=vd, cam_desc=rcd)
                rrep = 5
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                for _ in range(rrep):
                    tiles.render(v, tft, ridx, rcam, idx_desc=rdesc, vol_desc=vd, cam_desc=rcd)
                b.record(st)
                torch.cuda.synchronize()
                render_by_t[t] = (a.elapsed_time(b) / rrep, tiles.sample_total())
                a.record(st)
                for _ in range(rrep):
                    tiles.render(v, tft, ridx, rcam, idx_desc=rdesc, vol_desc=vd, cam_desc=rcd,
                                 ert_eps=ERT_EPS)
                b.record(st)
                torch.cuda.synchronize()
                ert_ms, ert_smp = a.elapsed_time(b) / rrep, tiles.sample_total()
                # ERT frame vs the exact frame (float RGBA, this rank's rows)
                outs = []
                for eps in (0.0, ERT_EPS):
                    tg = RenderTarget(W, H, want_rgba64=True)
                    render_rows(v, tft, ridx, rcam, tg, idx_desc=rdesc, vol_desc=vd,
                                cam_desc=rcd, ert_eps=eps)
                    outs.append(tg.rgba64)
                err = float((outs[0] - outs[1]).abs().max())
                ert_by_t[t] = (ert_ms, ert_smp, err)
                del ridx, outs, tg
            torch.cuda.synchronize()
    total_ms = max_over_ranks(total_ms, ws)
    ms_per_step = total_ms / args.steps
    build_ms = max_over_ranks(bev[0][0].elapsed_time(bev[0][1]) / reps, ws)
    build_cold_ms = max_over_ranks(bev[1][0].elapsed_time(bev[1][1]) / reps, ws)
    render_ms_t = {t: max_over_ranks(ms, ws) for t, (ms, _) in render_by_t.items()}
    ert_ms_t = {t: max_over_ranks(ms, ws) for t, (ms, _, _) in ert_by_t.items()}
    ert_step_ms = max_over_ranks(ert_total_ms, ws) / args.steps
    summ_ms = statistics.median([a.elapsed_time(b) for a, b in summ])
    vote_ms = statistics.median([a.elapsed_time(b) for a, b in votes])
    with torch.cuda.stream(st):
        rb.rebuild(params[0])  # the t = 0.6 index: reported counts and the parity check below
        rbc.rebuild(params[0])
    torch.cuda.synchronize()
    snap = rb.lbvh()
    n_bricks, height = snap.n_bricks, snap.height()

    # ---- parity spot check: the timed (warm) path's index vs the cold engine's and vs a fresh
    # public-API build -------------------------------------------------------------------------
    ref_idx = vs.build_lbvh(vs.flag_bricks(vs.classify(v, tfs[0], dilate=True)))
    m = ref_idx.node_count
    parity = (n_bricks == ref_idx.n_bricks and height == ref_idx.height() and
              all(torch.equal(rb.tree[f][:m], ref_idx.dev[f][:m]) and
                  torch.equal(rb.tree[f][:m], rbc.tree[f][:m])
                  for f in ("lo", "hi", "left", "right", "leaf_brick")) and
              torch.equal(rb.brick_bits, rbc.brick_bits))

    # ---- e2e through the public API ---------------------------------------------------------
    luts = [tf.lut for tf in tfs]
    e_steps = args.steps  # the same TF sweep / camera orbit as the device-timed loop
    pub = TileRenderer(W, H)

    build_stream = torch.cuda.Stream()

    def e2e_step(k, j):
        # TF change on a side stream: frame k+1's classify + build_index overlap frame k's
        # render (fresh index tensors per frame, kept alive until that frame's result())
        with torch.cuda.stream(build_stream):
            tf = vs.TransferFunction(luts[j])           # host LUT -> pinned -> device
            b = vs.classify(v, tf, dilate=True)
            index = vs.build_index("lbvh", b)
        torch.cuda.current_stream().wait_stream(build_stream)
        return pub.frame_async(v, tf, index, cams[j]), (tf, b, index)  # pixels -> pinned host

    with torch.cuda.stream(st):  # frames on the high-priority stream, TF changes on build_stream
        for k in range(min(args.warmup, 3)):
            e2e_step(k, k % NSWEEP)[0].result()
        e2e_runs = []
        for _ in range(3):  # three passes over the sweep (host-side jitter): the median is reported
            torch.cuda.synchronize()
            barrier(ws)
            e0.record(torch.cuda.current_stream())
            pending = None
            for k in range(e_steps):  # frame k's readback overlaps frame k+1's TF change / render
                nxt = e2e_step(k, sweep_j(k, e_steps))
                if pending is not None:
                    fr = pending[0].result()
                pending = nxt
            fr = pending[0].result()
            e1.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            e2e_runs.append(max_over_ranks(e0.elapsed_time(e1) / e_steps, ws))
            del fr, pending
    e2e_ms = statistics.median(e2e_runs)

    # ---- the other hierarchies' TF-change rebuilds (north star: "the same rebuild is also
    # reported for the SVT k-d tree, binned k-d tree and hybrid grid"): public API, classify +
    # build_index, synchronised, median of 3 after one warm-up, sparse / medium / dense ramp
    rebuilds = {}
    vox = v.dims[0] * v.dims[1] * v.dims[2]
    nbricks = rb.cap
    ncell16 = (-(-v.dims[0] // 16)) * (-(-v.dims[1] // 16)) * (-(-v.dims[2] // 16))

    def kind_bytes(kind, st):
        """Compulsory bytes of one TF-change rebuild (SVT-free builders: no summed-volume
        tables are written, so SURVEY §8d's B_svt-kd term does not apply).  lbvh / grid take the
        warm vote (the volume already has its presence masks): 32 B per brick; the k-d kinds
        classify + dilate the volume to packed bits (N^3 read, N^3/8 written) and write 37 B
        per row; hybrid adds its 16^3 grid, binned its 13 B per 8^3 cell box."""
        m = st["node_count"]
        if kind == "lbvh":
            nb = (m + 1) // 2
            return 32 * nbricks + 16 * nb + 36 * m + 12 * nb
        if kind == "grid":
            return 32 * nbricks + ncell16
        b = vox + vox // 8 + 37 * m
        if kind == "hybrid":
            b += ncell16
        if kind.startswith("kd-binned"):
            b += 13 * nbricks
        return b

    for kind in () if args.frame_only else ("lbvh", "grid", "hybrid", "kd-shallow",
                                            "kd-binned-mls32"):
        per_t, fr_t, m_t = [], [], []
        for t in (0.6, 0.3, 0.0):
            tfk = vs.TransferFunction.ramp(t)
            times = []
            for r in range(4):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ix = vs.build_index(kind, vs.classify(v, tfk, dilate=True))
                stats = vs.report_stats(ix)
                torch.cuda.synchronize()
                if r:
                    times.append((time.perf_counter() - t0) * 1e3)
            ms = statistics.median(times)
            per_t.append(round(ms, 3))
            m_t.append(stats["node_count"])
            fr_t.append(round(kind_bytes(kind, stats) / (ms * 1e-3) / 1e9 / hbm_peak()[0], 3))
        rebuilds[kind] = {"ms": per_t, "nodes": m_t, "roofline_frac": fr_t}
        del ix
    torch.cuda.empty_cache()

    # ---- roofline of the HBM-bound kernel -------------------------------------------------
    peak, peak_kind = hbm_peak()
    alg = rb.algorithmic_bytes(n_bricks)
    achieved = alg["summary_kernel"] / (summ_ms * 1e-3) / 1e9
    # dram bytes of this kernel per launch from the ncu --set full capture of the same
    # command (bench.py --frame-only), or null when no capture is committed
    traffic, traffic_src = profile_value("ncu_k_brick_summary.json", "dram_bytes_per_launch")
    l1_by_t = {t: profile_value(f"ncu_render_t{int(t * 10):02d}.json", "l1_hit_pct")[0]
               for t in render_by_t}

    if rank != 0:
        return
    cpu = None
    if ws == 1 and not args.no_cpu:
        # bounded CPU sample: args.cpu_frames full, unscaled frames of the same workload
        of = OracleFrames(u8.cpu().numpy())
        t0 = time.perf_counter()
        runs = [of.frame(tfs[sweep_j(k, args.cpu_frames)].lut, cams[sweep_j(k, args.cpu_frames)])
                for k in range(args.cpu_frames)]
        wall = time.perf_counter() - t0
        cpu = {"value": args.cpu_frames / wall, "unit": "frames/s", "cores": of.threads,
               "kind": "port",
               "sample": f"{args.cpu_frames} full {W}x{H} frames at {n}^3 (no scaling), sweep "
                         f"TFs j={[sweep_j(k, args.cpu_frames) for k in range(args.cpu_frames)]}"
                         f": classify+flag_bricks+build_lbvh + render through that tree",
               "rebuild_ms": 1e3 * statistics.mean(r["rebuild_s"] for r in runs),
               "render_ms": 1e3 * statistics.mean(r["render_s"] for r in runs)}
        del of
    clocks = clk.summary()
    # per step (ncu launch list of this command, profiles/r02_launches_interactive_frame.csv):
    # warm rebuild k_flags_tiles<FL_PRESENCE>, k_tile_scan, k_leaves_coop, k_tree_chunk,
    # k_tree_cross | render k_segments_brick, k_integrate_segments
    launches_per_step = 5 + 2
    line = {
        "metric": METRIC,
        "value": 1e3 / ms_per_step,
        "unit": "frames/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u8+f64",
        "data": "synthetic",
        "config": {**workload_config(n, nblobs, args.steps),
                   "l2": "input 1 GiB > 126 MB L2 (no flush needed)",
                   "parallelism": (f"image row stripes x{ws} + NCCL all-gather; "
                                   "per-TF build replicated"
                                   + ("; per-volume presence pass sharded by brick x-slabs"
                                      if ws > 1 else "")),
                   "pipeline": "rebuild k+1 on a side stream || render k (two index buffers); "
                               "renders on a high-priority stream"},
        "build_ms": build_ms,
        "build": {"warm_ms": build_ms, "cold_ms": build_cold_ms,
                  "warm": "per-volume 256-bit brick halo presence masks (built once, "
                          f"{32 * rb.cap / 2**20:.0f} MiB) -> flags -> tree: what the timed loop "
                          "runs (the volume stays resident across the TF sweep)",
                  "cold": "one-pass volume summary (k_brick_summary, 1 B/voxel) -> flags -> "
                          "tree: the first TF on a volume",
                  "alg_bytes_cold": alg["rebuild"], "alg_bytes_warm": alg["rebuild_warm"],
                  "roofline_frac_cold": alg["rebuild"] / (build_cold_ms * 1e-3) / 1e9 / peak,
                  "roofline_frac_warm": alg["rebuild_warm"] / (build_ms * 1e-3) / 1e9 / peak},
        "render_ms": render_ms_t[0.3],
        "render_by_t": {
            f"{t:.1f}": {"ms": render_ms_t[t], "fps": 1e3 / render_ms_t[t],
                         "samples_per_frame": smp, "Msamples_s": smp / render_ms_t[t] / 1e3,
                         "l1_hit_pct_ncu": l1_by_t[t]}
            for t, (_, smp) in render_by_t.items()},
        "render": {"view": "Camera.orbit(dims, 30, 15, 1920, 1080) (SURVEY App. B), LBVH of "
                           "ramp(t); render_ms = t 0.3; l1_hit_pct_ncu from profiles/"
                           "<round>_ncu_render_tXX.json (ncu --set full, same view)",
                   "kernels": "k_segments_brick (LBVH brick DDA) + k_integrate_segments"},
        "ert": {"eps": ERT_EPS, "value": 1e3 / ert_step_ms, "unit": "frames/s",
                "ms_per_step": ert_step_ms,
                "render_by_t": {f"{t:.1f}": {"ms": ert_ms_t[t], "fps": 1e3 / ert_ms_t[t],
                                             "samples_per_frame": smp,
                                             "max_abs_rgba_vs_exact": err}
                                for t, (_, smp, err) in ert_by_t.items()},
                "what": "opt-in early ray termination at opacity 1 - eps (RGBA within eps of "
                        "the reference integral; north star tolerance 1e-3): the same timed "
                        "loop and per-t renders with ert_eps; samples_per_frame = samples "
                        "actually taken"},
        "summary_kernel_ms": summ_ms,
        "n_bricks": n_bricks, "lbvh_nodes": max(2 * n_bricks - 1, 0), "lbvh_height": height,
        "parity_index_vs_public_api": bool(parity),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": "k_brick_summary", "peak_source": peak_kind,
                     "alg_bytes_per_launch": alg["summary_kernel"],
                     "share_of_step": None, "share_of_cold_rebuild": summ_ms / build_cold_ms,
                     "note": "the cold rebuild's volume pass (1 B/voxel), timed in this run; the "
                             "timed warm loop runs k_flags_tiles<FL_PRESENCE> instead "
                             "(roofline_warm_vote); the frame itself is the render kernels "
                             "(issue / FP64 / L1 bound, render_by_t)"},
        "roofline_warm_vote": {"bound": "hbm", "kernel": "k_flags_tiles<FL_PRESENCE>",
                               "alg_bytes_per_launch": 32 * rb.cap,
                               "ms": vote_ms, "unit": "GB/s",
                               "achieved": 32 * rb.cap / (vote_ms * 1e-3) / 1e9,
                               "frac": 32 * rb.cap / (vote_ms * 1e-3) / 1e9 / peak,
                               "share_of_step": vote_ms / ms_per_step},
        "rebuild_roofline_frac": alg["rebuild"] / (build_cold_ms * 1e-3) / 1e9 / peak,
        "rebuild_by_kind": {"ramp_t": [0.6, 0.3, 0.0], **rebuilds,
                            "how": "public API classify+build_index, host-synchronised wall "
                                   "time, median of 3; roofline_frac = compulsory bytes (see "
                                   "kind_bytes in bench.py / DESIGN.md §3) / time / HBM peak"},
        "e2e": {"value": 1e3 / e2e_ms, "unit": "frames/s",
                "h2d_bytes_per_step": 64 + 4096 + 2048, "d2h_bytes_per_step": W * H * 4 + 16,
                "ms_per_step": e2e_ms, "passes_ms_per_step": [round(x, 4) for x in e2e_runs],
                "path": "TransferFunction->classify->build_index('lbvh') on a build stream->"
                        "TileRenderer.frame_async(...).result(); frame k+1's TF change and "
                        "frame k's readback overlap frame k's render; median of 3 passes"},
        "gpu_launches": launches_per_step * args.steps,
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def channel_tfs(nch: int, k: int = NSWEEP):
    """Per-channel tinted ramps; the sweep moves every channel's threshold together."""
    from paper_1912_09596_b200.volume import TransferFunction

    tints = [(1.0, 0.3, 0.2), (0.2, 1.0, 0.3), (0.3, 0.4, 1.0), (1.0, 0.9, 0.2)]
    out = []
    for i in range(k):
        t = 0.6 - 0.6 * i / 63
        out.append([TransferFunction.ramp(threshold=t, color_lo=(0.1, 0.1, 0.1),
                                          color_hi=tints[c]) for c in range(nch)])
    return out


def run_multi(args, rank, ws, local):
    """BASELINE.json configs[4]: 4-channel 1024^3, 1080p, row-stripe tiles + NCCL gather."""
    import torch

    import paper_1912_09596_b200 as vs
    from paper_1912_09596_b200.engine import LbvhRebuilder
    from paper_1912_09596_b200.multichannel import classify_multi, interleaved_quads
    from paper_1912_09596_b200.render import tf_device
    from paper_1912_09596_b200.synth import gen_blobs_u8
    from paper_1912_09596_b200.tiles import TileRenderer

    n, nch = args.size, args.channels
    nblobs = max(1, 25600 * n ** 3 // 1024 ** 3)
    u8s = [gen_blobs_u8((n, n, n), n=nblobs, seed=7 + c, sigma=3.0) for c in range(nch)]
    vols = [vs.Volume.from_u8(u) for u in u8s]
    interleaved_quads(vols)  # channel-interleaved trilinear gather volume, built once
    tfs = channel_tfs(nch)
    cams = cameras(vols[0].dims)
    params = torch.stack([torch.stack([tf.params() for tf in tl]) for tl in tfs])
    for tl in tfs:
        for tf in tl:
            tf_device(tf, 0.5)
    # two index buffers: frame k+1's union rebuild (side stream) overlaps frame k's render
    rbs = [LbvhRebuilder(vols, warm=True).capture()]
    idxs = [r.index() for r in rbs]
    tiles = TileRenderer(W, H)
    st = torch.cuda.Stream(priority=-1) if os.environ.get("VSB200_PRIO", "1") == "1" \
        else torch.cuda.current_stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):

        def step(k, j):
            # rebuild then render on one stream: a rebuild overlapped on a side stream takes
            # SM slots from the 118-register 4-channel integrator while it runs and costs the
            # frame 15% (tools/mc_loop_probe.py; the single-channel frame is indifferent)
            rbs[0].rebuild(params[j])
            return tiles.render_multi(vols, tfs[j], idxs[0], cams[j], checked=False)

        for k in range(args.warmup):
            step(k, k % NSWEEP)
        torch.cuda.synchronize()
        barrier(ws)
        with ClockSampler(local) as clk:
            time.sleep(0.3)
            torch.cuda.synchronize()
            barrier(ws)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            tiles.multi_flags()
            e0.record(st)
            for k in range(args.steps):
                step(k, sweep_j(k, args.steps))
            e1.record(st)
            torch.cuda.synchronize()
        if tiles.multi_flags() & 4:
            raise RuntimeError("a timed frame exceeded the segment capacity (incomplete frame)")
        ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, ws)
        samples = tiles.sample_total()
        # e2e through the public API: per-step host LUTs -> classify_multi -> build_index -> frame
        luts = [[tf.lut for tf in tl] for tl in tfs]
        e_steps = args.steps
        build_stream = torch.cuda.Stream()
        e2e_runs = []
        for _ in range(3):  # three passes over the sweep (host-side jitter): the median is reported
            torch.cuda.synchronize()
            barrier(ws)
            e0.record(st)
            pending = None
            for k in range(e_steps):  # frame k's readback overlaps frame k+1's TF change / render
                j = sweep_j(k, e_steps)
                with torch.cuda.stream(build_stream):  # TF change overlapping the previous render
                    tl = [vs.TransferFunction(l) for l in luts[j]]
                    b = classify_multi(vols, tl, dilate=True)
                    index = vs.build_index("lbvh", b)
                torch.cuda.current_stream().wait_stream(build_stream)
                nxt = (tiles.frame_multi_async(vols, tl, index, cams[j]), (tl, b, index))
                if pending is not None:
                    frame = pending[0].result()
                pending = nxt
            frame = pending[0].result()
            e1.record(st)
            torch.cuda.synchronize()
            e2e_runs.append(max_over_ranks(e0.elapsed_time(e1) / e_steps, ws))
            del frame, pending
    e2e_ms = statistics.median(e2e_runs)
    if rank != 0:
        return
    cpu = None
    if ws == 1 and not args.no_cpu:
        from oracle import oracle as O

        # one full, unscaled 4-channel frame on every host core: per-channel classification,
        # union + dilation, flag_bricks + build_lbvh, the multi-channel render through it
        hosts = [u.cpu().numpy() for u in u8s]
        threads = os.cpu_count() or 1
        O.set_threads(threads)
        j0 = NSWEEP // 3
        opaque = np.zeros((256, 4), np.float32)
        opaque[1:, 3] = 1.0
        t0 = time.perf_counter()
        union = np.zeros(hosts[0].shape, bool)
        for h_, tf in zip(hosts, tfs[j0]):
            union |= O.classify(h_, tf.lut, dilate=False)[0]
        bits, _ = O.classify(union.view(np.uint8), opaque, dilate=True)
        del union
        coords, codes = O.flag_bricks(bits, 8)
        del bits
        tree = O.build_lbvh(coords, codes, 8, hosts[0].shape)
        t1 = time.perf_counter()
        O.render_multi("lbvh", hosts, [tf.lut for tf in tfs[j0]], tree, cams[j0],
                       nthreads=threads)
        t2 = time.perf_counter()
        cpu = {"value": 1.0 / (t2 - t0), "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": f"1 full {W}x{H} {nch}-channel frame at {n}^3 (no scaling), sweep "
                         f"TF j={j0}: per-channel classify, union dilation, flag_bricks + "
                         f"build_lbvh, multi-channel render",
               "rebuild_ms": (t1 - t0) * 1e3, "render_ms": (t2 - t1) * 1e3}
    line = {
        "metric": METRIC, "value": 1e3 / ms, "unit": "frames/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8+f64",
        "data": "synthetic",
        "config": {"workload": f"{nch}-channel {n}^3 u8 blobs (seeds 7..{6 + nch}), union "
                               f"LBVH rebuild + {W}x{H} render per frame, TF sweep",
                   "frame": "rebuild+render", "channels": nch, **sweep_desc(args.steps),
                   "parallelism": f"image row stripes x{ws} + NCCL all-gather"},
        "render": {"samples_per_frame": samples},
        "e2e": {"value": 1e3 / e2e_ms, "unit": "frames/s",
                "h2d_bytes_per_step": nch * (64 + 4096 + 2048),
                "d2h_bytes_per_step": W * H * 4, "ms_per_step": e2e_ms,
                "passes_ms_per_step": [round(x, 4) for x in e2e_runs],
                "path": "TransferFunction x nch->classify_multi->build_index('lbvh') on a "
                        "build stream->TileRenderer.frame_multi_async(...).result(); median "
                        "of 3 passes"},
        # warm rebuild (one vote over the channels' presence masks + 4 tree kernels), render
        "gpu_launches": (5 + 2) * args.steps,
        "cpu_baseline": cpu, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(n: int) -> int:
    """``bench.py --gpus N`` run bare: start N ranks (one per GPU) under torch.distributed.run
    on 127.0.0.1 with this same command line; rank 0 prints the JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--cpu-frames", type=int, default=2,
                    help="full CPU oracle frames timed for cpu_baseline (rank 0, N=1)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--frame-only", action="store_true",
                    help="skip the other hierarchies' rebuild timings (profiling runs)")
    ap.add_argument("--channels", type=int, default=1,
                    help="> 1: BASELINE configs[4] multi-channel frames")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        # CPU arm: rank 0 alone, no process group (the other ranks exit without work)
        run_reference(args, int(os.environ.get("RANK", "0")),
                      int(os.environ.get("WORLD_SIZE", "1")))
        return
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # communicator init lines (rank / nranks / transport) in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    rank, ws, local = dist_setup()
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {ws}; reporting n_gpus = {ws}",
              file=sys.stderr)
    if args.channels > 1:
        run_multi(args, rank, ws, local)
    else:
        run_ours(args, rank, ws, local)
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
