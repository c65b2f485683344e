"""Multi-process (world_size 2-3, gloo, CPU) checks of the sharding host
logic: the interleaved block partition covers every ray exactly once, and
ShardedFrame (render_image_distributed's all-gather + unshard + counter
all-reduce) reassembles image order on every rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_13744_b200.render import RAY_BLOCK, ShardedFrame, shard_rays, unshard_index


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("n_rays,world", [(640_000, 2), (640_000, 8), (6400, 3), (4096, 2), (1, 4), (10_000, 16)])
def test_partition_covers_every_ray_once(n_rays, world):
    seen = np.zeros(n_rays, np.int64)
    for r in range(world):
        off, stride, n_local = shard_rays(n_rays, r, world)
        assert off % RAY_BLOCK == 0 and stride == world
        i = np.arange(n_local)
        g = off + (i // RAY_BLOCK) * stride * RAY_BLOCK + i % RAY_BLOCK  # == global_ray() in gf_march.cuh
        assert np.all(g < n_rays)
        seen[g] += 1
    assert np.all(seen == 1)
    # per-rank load differs by at most one block
    loads = [shard_rays(n_rays, r, world)[2] for r in range(world)]
    assert max(loads) - min(loads) <= RAY_BLOCK


def _worker(rank, world, port, n_rays, out):
    """Runs the product's ShardedFrame (the gather / unshard / counter
    all-reduce of render_image_distributed) on gloo; the "render" of each
    shard writes the global ray id of every local row (the map
    global_ray() in gf_march.cuh implements on the device)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fr = ShardedFrame(n_rays, rank, world)
    fr.local.fill_(-1.0)
    i = torch.arange(fr.n_local, dtype=torch.int64)
    g = fr.offset + (i // RAY_BLOCK) * fr.stride * RAY_BLOCK + i % RAY_BLOCK
    fr.local[: fr.n_local] = g.to(torch.float32)[:, None] * torch.tensor([1.0, 2.0, 3.0])
    fr.stats.copy_(torch.tensor([fr.n_local, 2 * fr.n_local, rank, 1]))
    img, stats = fr.gather()
    out.put((rank, img.numpy().copy(), stats.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_rays,world", [(20_000, 2), (6400, 2), (4096, 2), (13_000, 3)])
def test_gloo_sharded_frame_reassembles_image_order(n_rays, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_rays, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.arange(n_rays, dtype=np.float32)[:, None] * np.array([1.0, 2.0, 3.0], np.float32)
    for rank, img, stats in res:  # every rank holds the assembled frame and the global counters
        assert np.array_equal(img, want), rank
        assert stats == [n_rays, 2 * n_rays, sum(range(world)), world]
