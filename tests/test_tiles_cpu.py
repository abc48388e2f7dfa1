"""Host-side logic of the multi-GPU tile split, on CPU: the stripe partition covers every
image row exactly once, and a world_size-2 gloo all-gather of per-rank stripes reassembled
with the same permutation TileRenderer uses reproduces the full frame."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1912_09596_b200.tiles import assemble, gather_permutation, stripe_rows


@pytest.mark.parametrize("height,world,stripe", [(1080, 1, 8), (1080, 2, 8), (1080, 8, 8),
                                                 (37, 3, 4), (5, 4, 1), (64, 8, 16)])
def test_partition_covers_rows(height, world, stripe):
    seen = np.concatenate([stripe_rows(height, world, p, stripe) for p in range(world)])
    assert sorted(seen.tolist()) == list(range(height))
    mx, src = gather_permutation(height, world, stripe)
    slots = np.full(world * mx, -1)
    for p in range(world):
        r = stripe_rows(height, world, p, stripe)
        slots[p * mx: p * mx + len(r)] = r
    assert (slots[src] == np.arange(height)).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, height, width, stripe, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frame = torch.arange(height * width * 4, dtype=torch.int64).reshape(height, width, 4) % 251
        rows = stripe_rows(height, world, rank, stripe)
        mx, perm = gather_permutation(height, world, stripe)
        local = torch.zeros((mx, width, 4), dtype=torch.uint8)
        local[: len(rows)] = frame[torch.from_numpy(rows)].to(torch.uint8)  # "render" own rows
        gathered = torch.empty((world * mx, width, 4), dtype=torch.uint8)
        dist.all_gather_into_tensor(gathered, local)
        out = torch.empty((height, width, 4), dtype=torch.uint8)
        assemble(gathered, torch.from_numpy(perm), out)
        q.put((rank, bool(torch.equal(out, frame.to(torch.uint8)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("height,stripe", [(1080, 8), (37, 4)])
def test_gloo_world2_gather_assembles_frame(height, stripe):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, height, 24, stripe, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}


@pytest.mark.parametrize("nbx,world", [(128, 1), (128, 2), (128, 8), (5, 3), (3, 4), (1, 2)])
def test_presence_slabs_partition(nbx, world):
    from paper_1912_09596_b200.tiles import presence_slabs

    sl = presence_slabs(nbx, world)
    assert len(sl) == world
    per = -(-nbx // world)
    covered = []
    for bx0, bx1 in sl:
        assert 0 <= bx0 <= bx1 <= nbx and bx1 - bx0 <= per
        covered += list(range(bx0, bx1))
    assert covered == list(range(nbx))


class _FakeVolume:  # what shard_presence reads of a Volume (dims; bins only on the GPU path)
    def __init__(self, dims):
        self.dims = dims


def _presence_worker(rank, world, port, dims, q):
    from paper_1912_09596_b200.tiles import shard_presence

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nbx, nby, nbz = (-(-d // 8) for d in dims)
        sw = nby * nbz * 8

        def builder(bx0, bx1, out):  # "build" this rank's slabs: word w of the array -> w % 9973
            out[: (bx1 - bx0) * sw] = torch.arange(bx0 * sw, bx1 * sw, dtype=torch.int32) % 9973

        p = shard_presence(_FakeVolume(dims), builder=builder)
        ref = torch.arange(nbx * sw, dtype=torch.int32) % 9973
        q.put((rank, bool(torch.equal(p, ref))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims", [(64, 40, 32), (72, 16, 16)])
def test_gloo_world2_sharded_presence_assembles(dims):
    """Sharded per-volume presence build (tiles.shard_presence): each rank's brick x-slabs,
    one all-gather, the full array in order on every rank (9 slabs over 2 ranks: uneven)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_presence_worker, args=(r, 2, port, dims, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res == {0: True, 1: True}
