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
# CPU reference (the oracle port of the reference path; test infrastructure)
# ------------------------------------------------------------------------------------------

def cpu_rebuild(u8_host: np.ndarray, lut: np.ndarray, slab: int):
    """classify(dilate) + flag_bricks + build_lbvh on x-slab [0, slab) (1 core)."""
    from oracle import oracle as O

    sub = np.ascontiguousarray(u8_host[:slab])
    t0 = time.perf_counter()
    bits, _ = O.classify(sub, lut, dilate=True)
    coords, codes = O.flag_bricks(bits, 8)
    O.build_lbvh(coords, codes, 8, sub.shape)
    return time.perf_counter() - t0


def oracle_lbvh(u8_host: np.ndarray, lut: np.ndarray):
    """The oracle's full-size LBVH for `lut` (untimed setup of the render sample)."""
    from oracle import oracle as O

    bits, _ = O.classify(u8_host, lut, dilate=True)
    coords, codes = O.flag_bricks(bits, 8)
    return O.build_lbvh(coords, codes, 8, u8_host.shape)


def cpu_render_rows(u8_host, lut, tree, cam, nrows: int, threads: int):
    """Render `nrows` middle rows of the frame through the oracle LBVH (timed)."""
    from oracle import oracle as O

    r0 = cam.height // 2 - nrows // 2
    t0 = time.perf_counter()
    _, samples = O.render("lbvh", u8_host, lut, tree, cam, rows=(r0, r0 + nrows),
                          nthreads=threads)
    return time.perf_counter() - t0, int(samples.sum())


class CpuFrame:
    """Bounded CPU sample of one interactive frame: the rebuild on an x-slab (1 core, scaled by
    n/slab) + the render of a middle row band (all cores, scaled by height/rows) through the
    oracle LBVH of the first sweep TF.  Sizes are calibrated once to a time budget."""

    def __init__(self, u8_host, lut0, cam, budget_s: float):
        self.u8 = u8_host
        self.n = u8_host.shape[0]
        self.threads = os.cpu_count() or 1
        self.tree = oracle_lbvh(u8_host, lut0)
        self.lut0 = lut0
        t = cpu_rebuild(u8_host, lut0, 16)
        self.slab = max(16, min(self.n, int(16 * (0.5 * budget_s) / max(t, 1e-3)) // 8 * 8))
        tr, _ = cpu_render_rows(u8_host, lut0, self.tree, cam, 8, self.threads)
        self.rows = max(8, min(cam.height, int(8 * (0.5 * budget_s) / max(tr, 1e-3)) // 8 * 8))

    def frame(self, lut, cam):
        rb = cpu_rebuild(self.u8, lut, self.slab)
        tr, _ = cpu_render_rows(self.u8, self.lut0, self.tree, cam, self.rows, self.threads)
        rebuild_s = rb * self.n / self.slab
        render_s = tr * cam.height / self.rows
        return {"frame_s": rebuild_s + render_s, "rebuild_s": rebuild_s, "render_s": render_s}

    def sample(self, cam):
        return (f"oracle rebuild on x-slab [0,{self.slab}) of {self.n}^3 scaled "
                f"x{self.n / self.slab:.1f} (1 core) + oracle LBVH render of {self.rows} middle "
                f"rows of {cam.width}x{cam.height} scaled x{cam.height / self.rows:.1f} "
                f"({self.threads} threads)")


def cpu_frame_estimate(u8_host, lut, cam, budget_s: float):
    cf = CpuFrame(u8_host, lut, cam, budget_s)
    est = cf.frame(lut, cam)
    est["threads"] = cf.threads
    est["sample"] = cf.sample(cam)
    return est


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
    if rank != 0:
        return
    import torch  # noqa: F401

    n = args.size
    u8d, nblobs = make_volume(n)
    u8 = u8d.cpu().numpy()
    tfs = sweep_tfs()
    cams = cameras(u8.shape)
    nsteps = args.steps + args.warmup
    budget = max(0.5, min(20.0, 120.0 / max(nsteps, 1)))
    cf = CpuFrame(u8, tfs[0].lut, cams[0], budget)
    times = []
    info = None
    for k in range(nsteps):
        est = cf.frame(tfs[k % NSWEEP].lut, cams[k % NSWEEP])
        if k >= args.warmup:
            times.append(est["frame_s"])
            info = est
    info["threads"] = cf.threads
    info["sample"] = cf.sample(cams[0]) + "; per step: the sweep TF's rebuild, orbit camera"
    frame_s = statistics.mean(times)
    value = 1.0 / frame_s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": frame_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8+f64", "data": "synthetic",
        "config": {"workload": f"interactive TF sweep on {n}^3 u8 blobs ({nblobs} blobs, sigma "
                               f"3, seed 7): LBVH rebuild + {W}x{H} render per frame",
                   "frame": "rebuild+render"},
        "build_ms": info["rebuild_s"] * 1e3, "render_ms": info["render_s"] * 1e3,
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": info["threads"],
                         "kind": "port", "sample": info["sample"]},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, ws, local):
    import torch

    import paper_1912_09596_b200 as vs
    from paper_1912_09596_b200.engine import LbvhRebuilder, tf_params_device
    from paper_1912_09596_b200.render import camera_desc, index_desc, tf_device, volume_desc
    from paper_1912_09596_b200.tiles import TileRenderer

    n = args.size
    u8, nblobs = make_volume(n)
    v = vs.Volume.from_u8(u8)
    tfs = sweep_tfs()
    cams = cameras(v.dims)
    params = tf_params_device(tfs)
    for tf in tfs:
        tf_device(tf, 0.5)  # LUT + opacity-correction tables resident for the sweep
    # two index buffers: frame k+1's rebuild (side stream) overlaps frame k's render
    rbs = [LbvhRebuilder(v).capture(), LbvhRebuilder(v).capture()]
    rb = rbs[0]
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

    def step(k):
        j, b = k % NSWEEP, k % 2
        with torch.cuda.stream(sb):
            sb.wait_event(rendered[b])        # buffer b free: frame k-2 rendered
            rbs[b].rebuild(params[j])
            built[b].record(sb)
        st.wait_event(built[b])
        with torch.cuda.stream(st):
            img = tiles.render(v, tfs[j], idxs[b], cams[j], idx_desc=ids[b], vol_desc=vd,
                               cam_desc=cds[j])
        rendered[b].record(st)
        return img

    # ---- device-resident loop (value) ------------------------------------------------------
    with torch.cuda.stream(st):
        for k in range(args.warmup):
            step(k)
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
                step(k)
            st.wait_stream(sb)
            e1.record(st)
            torch.cuda.synchronize()
            total_ms = e0.elapsed_time(e1)
            # component split (not the headline): rebuild alone, summary kernel alone, render alone
            bev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(3)]
            reps = max(10, min(args.steps, 100))
            bev[0][0].record(st)
            for k in range(reps):
                rb.rebuild(params[k % NSWEEP])
            bev[0][1].record(st)
            summ = []
            for k in range(reps):
                rb.set_tf(params[k % NSWEEP])
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                rb.launch_summary(st.cuda_stream)
                b.record(st)
                rb.launch_tree(st.cuda_stream)
                summ.append((a, b))
            rb.rebuild(params[0])
            rrep = max(3, min(args.steps, 10))
            samples = 0
            bev[1][0].record(st)
            for k in range(rrep):
                tiles.render(v, tfs[0], idx, cams[k % NSWEEP], idx_desc=index_desc(idx),
                             vol_desc=vd, cam_desc=cds[k % NSWEEP])
            bev[1][1].record(st)
            torch.cuda.synchronize()
            samples = tiles.sample_total()  # last frame's samples (all ranks)
    total_ms = max_over_ranks(total_ms, ws)
    ms_per_step = total_ms / args.steps
    build_ms = max_over_ranks(bev[0][0].elapsed_time(bev[0][1]) / reps, ws)
    render_ms = max_over_ranks(bev[1][0].elapsed_time(bev[1][1]) / rrep, ws)
    summ_ms = statistics.median([a.elapsed_time(b) for a, b in summ])
    info = rb.info.cpu().tolist()
    n_bricks, height = int(info[0]), int(info[1])

    # ---- parity spot check: the timed path's index vs a fresh public-API build ----------------
    ref_idx = vs.build_lbvh(vs.flag_bricks(vs.classify(v, tfs[0], dilate=True)))
    parity = (n_bricks == ref_idx.n_bricks and height == ref_idx.height() and
              all(torch.equal(rb.tree[f][:ref_idx.node_count], ref_idx.dev[f][:ref_idx.node_count])
                  for f in ("lo", "hi", "left", "right")))

    # ---- e2e through the public API ---------------------------------------------------------
    luts = [tf.lut for tf in tfs]
    e_steps = args.steps  # the same TF sweep / camera orbit as the device-timed loop
    pub = TileRenderer(W, H)

    build_stream = torch.cuda.Stream()

    def e2e_step(k):
        # TF change on a side stream: frame k+1's classify + build_index overlap frame k's
        # render (fresh index tensors per frame, kept alive until that frame's result())
        j = k % NSWEEP
        with torch.cuda.stream(build_stream):
            tf = vs.TransferFunction(luts[j])           # host LUT -> pinned -> device
            b = vs.classify(v, tf, dilate=True)
            index = vs.build_index("lbvh", b)
        torch.cuda.current_stream().wait_stream(build_stream)
        return pub.frame_async(v, tf, index, cams[j]), (tf, b, index)  # pixels -> pinned host

    with torch.cuda.stream(st):  # frames on the high-priority stream, TF changes on build_stream
        for k in range(min(args.warmup, 3)):
            e2e_step(k)[0].result()
        e2e_runs = []
        for _ in range(3):  # three passes over the sweep (host-side jitter): the median is reported
            torch.cuda.synchronize()
            barrier(ws)
            e0.record(torch.cuda.current_stream())
            pending = None
            for k in range(e_steps):  # frame k's readback overlaps frame k+1's TF change / render
                nxt = e2e_step(k)
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
    for kind in () if args.frame_only else ("lbvh", "grid", "hybrid", "kd-shallow",
                                            "kd-binned-mls32"):
        per_t = []
        for t in (0.6, 0.3, 0.0):
            tfk = vs.TransferFunction.ramp(t)
            times = []
            for r in range(4):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ix = vs.build_index(kind, vs.classify(v, tfk, dilate=True))
                vs.report_stats(ix)
                torch.cuda.synchronize()
                if r:
                    times.append((time.perf_counter() - t0) * 1e3)
            per_t.append(round(statistics.median(times), 3))
        rebuilds[kind] = per_t
        del ix
    torch.cuda.empty_cache()

    # ---- roofline of the HBM-bound kernel -------------------------------------------------
    peak, peak_kind = hbm_peak()
    alg = rb.algorithmic_bytes(n_bricks)
    achieved = alg["summary_kernel"] / (summ_ms * 1e-3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "r01_summary_traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    if rank != 0:
        return
    cpu = None
    if ws == 1 and not args.no_cpu:
        est = cpu_frame_estimate(u8.cpu().numpy(), tfs[0].lut, cams[0], args.cpu_budget)
        cpu = {"value": 1.0 / est["frame_s"], "unit": "frames/s", "cores": est["threads"],
               "kind": "port", "sample": est["sample"], "rebuild_ms": est["rebuild_s"] * 1e3,
               "render_ms": est["render_s"] * 1e3}
    clocks = clk.summary()
    # per step (ncu launch list, profiles/r01_launches_interactive_frame.csv): k_brick_summary,
    # k_summary_to_bitmap, 2 CUB scan kernels launched by vs_lbvh_from_bitmap (leaf ranks),
    # k_leaves_from_bitmap, k_karras, k_refit_chunked, k_brick_grid | k_segments,
    # k_integrate_segments
    launches_per_step = 8 + 2
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
        "config": {"workload": f"interactive TF sweep on {n}^3 u8 blobs ({nblobs} blobs, sigma "
                               f"3, seed 7): LBVH rebuild + {W}x{H} render per frame, 64 ramp "
                               f"TFs t=0.6..0, orbit camera el 15, dt 0.5",
                   "frame": "rebuild+render", "brick": 8,
                   "l2": "input 1 GiB > 126 MB L2 (no flush needed)",
                   "parallelism": f"image row stripes x{ws} + NCCL all-gather; build replicated",
                   "pipeline": "rebuild k+1 on a side stream || render k (two index buffers); "
                               "renders on a high-priority stream"},
        "build_ms": build_ms,
        "render_ms": render_ms,
        "render": {"fps": 1e3 / render_ms, "samples_per_frame": samples,
                   "Msamples_s": samples / render_ms / 1e3,
                   "kernels": "k_segments<LBVH brick DDA> + k_integrate_segments"},
        "summary_kernel_ms": summ_ms,
        "n_bricks": n_bricks, "lbvh_nodes": max(2 * n_bricks - 1, 0), "lbvh_height": height,
        "parity_index_vs_public_api": bool(parity),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_brick_summary", "peak_source": peak_kind,
                     "alg_bytes_per_launch": alg["summary_kernel"],
                     "share_of_step": summ_ms / ms_per_step},
        "rebuild_roofline_frac": alg["rebuild"] / (build_ms * 1e-3) / 1e9 / peak,
        "rebuild_ms_by_kind": {"ramp_t": [0.6, 0.3, 0.0], **rebuilds,
                               "how": "public API classify+build_index, host-synchronised "
                                      "wall time, median of 3"},
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
    rbs = [LbvhRebuilder(vols).capture(), LbvhRebuilder(vols).capture()]
    idxs = [r.index() for r in rbs]
    tiles = TileRenderer(W, H)
    # frames on a high-priority stream, rebuilds / TF changes on default-priority streams
    st = torch.cuda.Stream(priority=-1) if os.environ.get("VSB200_PRIO", "1") == "1" \
        else torch.cuda.current_stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        sb = torch.cuda.Stream()
        built = [torch.cuda.Event(), torch.cuda.Event()]
        rendered = [torch.cuda.Event(), torch.cuda.Event()]

        def step(k):
            j, b = k % NSWEEP, k % 2
            with torch.cuda.stream(sb):
                sb.wait_event(rendered[b])
                rbs[b].rebuild(params[j])
                built[b].record(sb)
            st.wait_event(built[b])
            img = tiles.render_multi(vols, tfs[j], idxs[b], cams[j], checked=False)
            rendered[b].record(st)
            return img

        for k in range(args.warmup):
            step(k)
        torch.cuda.synchronize()
        barrier(ws)
        with ClockSampler(local) as clk:
            time.sleep(0.3)
            torch.cuda.synchronize()
            barrier(ws)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            tiles.multi_flags()
            e0.record(st)
            sb.wait_stream(st)
            for k in range(args.steps):
                step(k)
            st.wait_stream(sb)
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
                j = k % NSWEEP
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

        hosts = [u.cpu().numpy() for u in u8s]
        t0 = time.perf_counter()
        slab = 64
        for h_, tf in zip(hosts, tfs[0]):
            O.classify(np.ascontiguousarray(h_[:slab]), tf.lut, dilate=True)
        rebuild_s = (time.perf_counter() - t0) * n / slab
        import types
        cam = cams[0]
        nrows = 4
        sub = types.SimpleNamespace(eye=cam.eye, direction=cam.direction, up=cam.up,
                                    extent=cam.extent, width=cam.width, height=nrows)
        # a band of rows through the image centre: shift the eye down to row H/2
        b = classify_multi(vols, tfs[0], dilate=True)
        index = vs.build_index("lbvh", b)
        eye, up, right, scale = cam.frame_vectors()
        shift = (H / 2.0 - nrows / 2.0) * scale
        sub.eye = tuple(np.asarray(eye) - shift * np.asarray(up))
        oidx = {"lo": index.lo, "hi": index.hi, "left": index.left, "right": index.right,
                "root": index.root, "height": index.height()}
        t0 = time.perf_counter()
        O.render_multi("lbvh", hosts, [tf.lut for tf in tfs[0]], oidx, sub)
        render_s = (time.perf_counter() - t0) * H / nrows
        cpu = {"value": 1.0 / (rebuild_s + render_s), "unit": "frames/s", "cores": 1,
               "kind": "port", "sample": f"oracle: {nch}-channel classify on x-slab [0,{slab}) "
               f"scaled x{n / slab:.0f} + multi-channel LBVH render of {nrows} centre rows "
               f"scaled x{H / nrows:.0f} (1 thread)",
               "rebuild_ms": rebuild_s * 1e3, "render_ms": render_s * 1e3}
    line = {
        "metric": METRIC, "value": 1e3 / ms, "unit": "frames/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8+f64",
        "data": "synthetic",
        "config": {"workload": f"{nch}-channel {n}^3 u8 blobs (seeds 7..{6 + nch}), union "
                               f"LBVH rebuild + {W}x{H} render per frame, TF sweep",
                   "frame": "rebuild+render", "channels": nch,
                   "parallelism": f"image row stripes x{ws} + NCCL all-gather"},
        "render": {"samples_per_frame": samples},
        "e2e": {"value": 1e3 / e2e_ms, "unit": "frames/s",
                "h2d_bytes_per_step": nch * (64 + 4096 + 2048),
                "d2h_bytes_per_step": W * H * 4, "ms_per_step": e2e_ms,
                "passes_ms_per_step": [round(x, 4) for x in e2e_runs],
                "path": "TransferFunction x nch->classify_multi->build_index('lbvh') on a "
                        "build stream->TileRenderer.frame_multi_async(...).result(); median "
                        "of 3 passes"},
        # summaries, ORs, tree (as the single-channel step), render
        "gpu_launches": (nch + (nch - 1) + 7 + 2) * args.steps,
        "cpu_baseline": cpu, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--frame-only", action="store_true",
                    help="skip the other hierarchies' rebuild timings (profiling runs)")
    ap.add_argument("--channels", type=int, default=1,
                    help="> 1: BASELINE configs[4] multi-channel frames")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, ws, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, rank, ws)
    elif args.channels > 1:
        run_multi(args, rank, ws, local)
    else:
        run_ours(args, rank, ws, local)
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
