"""Multi-process (world_size 2, gloo, CPU) checks of the sharding host logic:
the interleaved block partition covers every ray exactly once, and the
all-gather + unshard permutation reassembles image order."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_13744_b200.render import RAY_BLOCK, shard_rays, unshard_index


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
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    off, stride, n_local = shard_rays(n_rays, rank, world)
    n_blocks = (n_rays + RAY_BLOCK - 1) // RAY_BLOCK
    cap = ((n_blocks + world - 1) // world) * RAY_BLOCK
    buf = torch.full((cap, 3), -1.0, dtype=torch.float64)
    i = torch.arange(n_local, dtype=torch.int64)
    g = off + (i // RAY_BLOCK) * stride * RAY_BLOCK + i % RAY_BLOCK
    buf[:n_local] = g.to(torch.float64)[:, None]  # "render" = global ray id
    gathered = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf)
    stats = torch.tensor([n_local], dtype=torch.int64)
    dist.all_reduce(stats)
    if rank == 0:
        flat = torch.cat(gathered)
        img = flat[torch.from_numpy(unshard_index(n_rays, world))][:, 0]
        out.put((img.numpy(), int(stats.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_rays,world", [(20_000, 2), (6400, 2)])
def test_gloo_gather_reassembles_image_order(n_rays, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_rays, q)) for r in range(world)]
    for p in procs:
        p.start()
    img, total = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert total == n_rays
    assert np.array_equal(img, np.arange(n_rays, dtype=np.float64))
