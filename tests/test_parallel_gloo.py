"""Host logic of the slab decomposition on CPU: partitioning invariants and the
ghost-plane exchange, world_size 2 (and 3) with the gloo backend."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2006_16764_b200.parallel import exchange_planes_torch, partition_planes


def test_partition_invariants():
    for nslow, world, align in [(2049, 8, 8), (65, 2, 8), (65, 4, 8), (17, 2, 8), (513, 8, 8), (13, 3, 1)]:
        b = partition_planes(nslow, world, align)
        assert len(b) == world and b[0][0] == 0 and b[-1][1] == nslow
        for (lo, hi), (lo2, _) in zip(b, b[1:]):
            assert hi == lo2 and hi > lo and lo2 % align == 0
        sizes = [hi - lo for lo, hi in b]
        assert max(sizes) - min(sizes) <= align + 1
    with pytest.raises(ValueError):
        partition_planes(9, 4, 8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, nx, ny, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # a global block-ordered 2D vector with value = field*1e6 + node id
        N = nx * ny
        g = torch.cat([torch.arange(N, dtype=torch.float64), 1e6 + torch.arange(N, dtype=torch.float64)])
        lo, hi = partition_planes(ny, world, 1)[rank]
        local = torch.cat([g[lo * nx:hi * nx], g[N + lo * nx:N + hi * nx]])
        glo, ghi = exchange_planes_torch(local, nx)
        ok = True
        if rank > 0:
            want = torch.stack([g[(lo - 1) * nx:lo * nx], g[N + (lo - 1) * nx:N + lo * nx]])
            ok &= torch.equal(glo, want)
        else:
            ok &= glo is None
        if rank + 1 < world:
            want = torch.stack([g[hi * nx:(hi + 1) * nx], g[N + hi * nx:N + (hi + 1) * nx]])
            ok &= torch.equal(ghi, want)
        else:
            ok &= ghi is None
        # global sum of a distributed dot product equals the serial one
        part = torch.tensor([float((local * local).sum())], dtype=torch.float64)
        dist.all_reduce(part)
        ok &= abs(float(part) - float((g * g).sum())) <= 1e-9 * float((g * g).sum())
        result[rank] = 1 if ok else 0
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_plane_exchange(world):
    ctx = mp.get_context("spawn")
    result = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 7, 11, result)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert list(result) == [1] * world
