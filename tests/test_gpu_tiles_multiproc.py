"""The tile-parallel render path end to end with 2 processes.  Each rank renders its
interleaved row stripes; the gathered, re-permuted frame and the summed sample count equal a
single-process render bit for bit.  On one GPU the ranks share it over a gloo group (NCCL
refuses two ranks on one device); with >= 2 GPUs the same check runs over NCCL, one rank per
GPU (skipped on the 1-GPU boxes)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, u8, lut, q, backend="gloo"):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1912_09596_b200 as vs
        from paper_1912_09596_b200.tiles import TileRenderer

        v = vs.Volume.from_u8(u8)
        tf = vs.TransferFunction(lut)
        idx = vs.build_index("lbvh", vs.classify(v, tf, dilate=True))
        cam = vs.Camera.orbit(v.dims, 30.0, 15.0, width=72, height=45)
        fr = TileRenderer(72, 45, stripe=4).frame(v, tf, idx, cam)
        q.put((rank, fr.pixels, fr.sample_count))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("backend", ["gloo", "nccl"])
def test_two_rank_tiles_equal_single_render(blobs64, backend):
    import torch
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if backend == "nccl" and torch.cuda.device_count() < 2:
        pytest.skip("NCCL tile gather needs 2 GPUs (gpurun boxes have 1)")
    import paper_1912_09596_b200 as vs

    u8, lut = blobs64["u8"], blobs64["ramp03_lut"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, u8, lut, q, backend))
             for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, pix, n = q.get(timeout=300)
        res[rank] = (pix, n)
    for p in procs:
        p.join(timeout=60)
    v = vs.Volume.from_u8(u8)
    tf = vs.TransferFunction(lut)
    idx = vs.build_index("lbvh", vs.classify(v, tf, dilate=True))
    full = vs.render_frame(v, tf, idx, vs.Camera.orbit(v.dims, 30.0, 15.0, width=72, height=45))
    for r in (0, 1):
        np.testing.assert_array_equal(res[r][0], full.pixels)
        assert res[r][1] == full.sample_count
