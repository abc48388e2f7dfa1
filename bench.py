#!/usr/bin/env python
"""Benchmark: interactive transfer-function sweep on a synthetic 1024^3 u8 volume (B200).

One step = one TF-change frame: the LBVH over the volume's dilated brick classification is
rebuilt for the next TF of a sweep (BASELINE.json configs[3], the north-star target "a TF
change rebuilds the LBVH in <= 5 ms at >= 50% of HBM roofline").  The rebuild is:

    vs_classify_summary (one pass over the u8 volume) -> vs_summary_to_bitmap
    -> vs_lbvh_from_bitmap (scan, leaves, Karras, refit)

captured as one CUDA graph; the TF reaches the device as a 64-byte parameter block.

  value  frames/s with the volume and the sweep's TF blocks resident in HBM (device-timed)
  e2e    the same through the public API (TransferFunction -> classify -> build_index ->
         report_stats) with the TF uploaded from pinned host memory and the stats read back
  roofline  k_brick_summary: algorithmic bytes (N^3 read + 4 B/brick summary write) over its
         CUDA-event duration vs MEASURED_PEAKS.json hbm (else the recipe's fallback)
  cpu_baseline  the C oracle (oracle/vs_oracle.c: classify(dilate) + flag_bricks + build_lbvh,
         1 core) on an x-slab of the same volume, scaled to the full volume

Multi-GPU (--gpus N under torchrun): the build does not shard (construction is
replicated); every rank rebuilds its own replica and value sums the ranks' frames (weak).
`--impl reference` times the CPU oracle port of the reference path instead (rank 0 only).
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


def sweep_luts(k: int):
    """TF sweep of config 4: ramp thresholds 0.6 -> 0, cycled."""
    from paper_1912_09596_b200.volume import TransferFunction

    ts = [0.6 - 0.6 * i / 63 for i in range(64)]
    return [TransferFunction.ramp(threshold=ts[i % 64]) for i in range(k)]


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
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

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
# CPU baseline (oracle port of the reference path, test infrastructure)
# ------------------------------------------------------------------------------------------

def cpu_rebuild_sample(u8_host: np.ndarray, lut: np.ndarray, slab: int):
    """classify(dilate) + flag_bricks + build_lbvh on x-slab [0, slab) with the C oracle."""
    from oracle import oracle as O

    sub = np.ascontiguousarray(u8_host[:slab])
    t0 = time.perf_counter()
    bits, _ = O.classify(sub, lut, dilate=True)
    coords, codes = O.flag_bricks(bits, 8)
    O.build_lbvh(coords, codes, 8, sub.shape)
    return time.perf_counter() - t0


def cpu_baseline(u8_host, lut, budget_s: float = 20.0):
    nx = u8_host.shape[0]
    slab = min(nx, 16)
    t = cpu_rebuild_sample(u8_host, lut, slab)
    # grow the slab to ~budget_s of work (bounded sample), multiple of 8
    target = int(slab * max(1.0, budget_s / max(t, 1e-3)))
    slab2 = max(8, min(nx, (target // 8) * 8))
    if slab2 > slab:
        t = cpu_rebuild_sample(u8_host, lut, slab2)
        slab = slab2
    full_s = t * nx / slab
    return {"value": 1.0 / full_s, "unit": "frames/s", "cores": 1, "kind": "port",
            "sample": f"oracle classify(dilate)+flag_bricks+build_lbvh on x-slab "
                      f"[0,{slab}) of the {nx}^3 volume ({t:.2f} s), scaled x{nx / slab:.1f}",
            "full_rebuild_ms": full_s * 1e3}


# ------------------------------------------------------------------------------------------

def dist_setup():
    import torch
    import torch.distributed as dist

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if ws > 1 and not dist.is_initialized():
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return rank, ws, local


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def run_reference(args, rank, ws):
    if rank != 0:
        return
    import torch  # noqa: F401
    from paper_1912_09596_b200.synth import gen_blobs_u8

    n = args.size
    u8 = gen_blobs_u8((n, n, n), n=max(1, 25600 * n ** 3 // 1024 ** 3), seed=7,
                      sigma=3.0).cpu().numpy()
    luts = [tf.lut for tf in sweep_luts(max(args.steps + args.warmup, 1))]
    nsteps = args.steps + args.warmup
    # size each step's slab so the whole run stays within ~120 s
    probe = cpu_rebuild_sample(u8, luts[0], 8)
    per_step_budget = min(5.0, 120.0 / max(nsteps, 1))
    slab = max(8, min(n, int(8 * per_step_budget / max(probe, 1e-3)) // 8 * 8))
    times = []
    for k in range(nsteps):
        t = cpu_rebuild_sample(u8, luts[k], slab)
        if k >= args.warmup:
            times.append(t)
    full_s = sum(times) / len(times) * n / slab
    value = 1.0 / full_s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": full_s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"TF-sweep LBVH rebuild, {n}^3 u8 blobs (25600 per 1024^3, "
                               f"sigma 3, seed 7), ramp t=0.6..0", "frame": "rebuild"},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": 1, "kind": "port",
                         "sample": f"oracle C port, x-slab [0,{slab}) per step, scaled "
                                   f"x{n / slab:.1f}"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, ws, local):
    import torch

    import paper_1912_09596_b200 as vs
    from paper_1912_09596_b200.engine import LbvhRebuilder, tf_params_device
    from paper_1912_09596_b200.synth import gen_blobs_u8

    n = args.size
    dims = (n, n, n)
    nblobs = max(1, 25600 * n ** 3 // 1024 ** 3)
    u8 = gen_blobs_u8(dims, n=nblobs, seed=7, sigma=3.0)
    v = vs.Volume(u8)
    nsweep = 64
    tfs = sweep_luts(nsweep)
    params = tf_params_device(tfs)
    rb = LbvhRebuilder(v, with_grid=False).capture()
    st = torch.cuda.current_stream()

    # ---- device-resident loop (value) ------------------------------------------------------
    for k in range(args.warmup):
        rb.rebuild(params[k % nsweep])
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    # dominant kernel timed on its own (same stream), to apportion the step
    sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    barrier(ws)
    with ClockSampler(local) as clk:
        time.sleep(0.3)  # let the sampler start
        torch.cuda.synchronize()
        barrier(ws)
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(st)
        for k in range(args.steps):
            rb.rebuild(params[k % nsweep])
        t_end.record(st)
        torch.cuda.synchronize()
        total_ms = t_start.elapsed_time(t_end)
        # kernel-level split (not the headline): summary kernel alone vs the tree launches
        for k in range(args.steps):
            rb.set_tf(params[k % nsweep])
            sev[k][0].record(st)
            rb.launch_summary(st.cuda_stream)
            sev[k][1].record(st)
            rb.launch_tree(st.cuda_stream)
        torch.cuda.synchronize()
    total_ms = max_over_ranks(total_ms, ws)
    ms_per_step = total_ms / args.steps
    summ_ms = statistics.median([a.elapsed_time(b) for a, b in sev])
    info = rb.info.cpu().tolist()
    n_bricks, height = int(info[0]), int(info[1])

    # ---- parity spot check of the last TF against a fresh public-API build -----------------
    last_tf = tfs[(args.steps - 1) % nsweep]
    ref_idx = vs.build_lbvh(vs.flag_bricks(vs.classify(v, last_tf, dilate=True)))
    rb.rebuild(params[(args.steps - 1) % nsweep])
    snap = rb.lbvh()
    parity = (snap.n_bricks == ref_idx.n_bricks and snap.height() == ref_idx.height() and
              all(torch.equal(snap.dev[f][:snap.node_count], ref_idx.dev[f][:ref_idx.node_count])
                  for f in ("lo", "hi", "left", "right")))

    # ---- e2e through the public API ---------------------------------------------------------
    luts = [tf.lut for tf in tfs]
    e_steps = max(1, min(args.steps, 200))
    for k in range(min(args.warmup, 3)):
        vs.report_stats(vs.build_index("lbvh", vs.classify(v, vs.TransferFunction(luts[k]),
                                                            dilate=True)))
    torch.cuda.synchronize()
    barrier(ws)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(e_steps):
        tf = vs.TransferFunction(luts[k % nsweep])      # host LUT -> params -> pinned H2D
        b = vs.classify(v, tf, dilate=True)
        stats = vs.report_stats(vs.build_index("lbvh", b))  # D2H of {n, height}
    e1.record(st)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / e_steps, ws)

    # ---- roofline of the dominant kernel ----------------------------------------------------
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
    cpu = cpu_baseline(u8.cpu().numpy(), luts[0], budget_s=args.cpu_budget) \
        if (ws == 1 and not args.no_cpu) else None
    clocks = clk.summary()
    line = {
        "metric": METRIC,
        "value": ws * 1e3 / ms_per_step,
        "unit": "frames/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": f"TF-sweep LBVH rebuild, {n}^3 u8 blobs ({nblobs} blobs, sigma "
                               f"3, seed 7), 64 ramp TFs t=0.6..0 cycled", "frame": "rebuild",
                   "brick": 8, "l2": "input 1 GiB > 126 MB L2 (no flush needed)",
                   "parallelism": f"replica x{ws}"},
        "build_ms": ms_per_step,
        "summary_kernel_ms": summ_ms,
        "n_bricks_last": n_bricks, "lbvh_nodes_last": max(2 * n_bricks - 1, 0),
        "height_last": height,
        "parity_last_tf_vs_public_api": bool(parity),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "k_brick_summary", "peak_source": peak_kind,
                     "alg_bytes_per_launch": alg["summary_kernel"]},
        "rebuild_roofline_frac": alg["rebuild"] / (ms_per_step * 1e-3) / 1e9 / peak,
        "e2e": {"value": ws * 1e3 / e2e_ms, "unit": "frames/s", "h2d_bytes_per_step": 64,
                "d2h_bytes_per_step": 8, "ms_per_step": e2e_ms,
                "path": "TransferFunction->classify->build_index('lbvh')->report_stats"},
        "gpu_launches": 5 * args.steps,
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, ws, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, rank, ws)
    else:
        run_ours(args, rank, ws, local)
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
