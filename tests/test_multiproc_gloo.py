"""World-size-2 (gloo, CPU) test of the (b, h) sharding used by bench.py and
the multi-GPU path: each rank computes its shard (here with the oracle, as a
stand-in for the device kernel), the shards are all-gathered, and the result
equals the unsharded computation bitwise (no data-path exchange)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_16847_b200.shard import bh_range
from workloads import Config, Pattern, make_qkv


CFG = Config("gloo_small", Pattern("global_local", 96, lo=8, hi=8, n_global=4), 2, 3, 16, "fp32", 301)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, scaling, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    BH = CFG.BH
    rng = bh_range(BH, rank, world, scaling)
    q, k, v = make_qkv(CFG, bh_range=rng)
    mine = torch.stack([torch.from_numpy(O.attention(CFG.pattern, q[i], k[i], v[i], CFG.scale, nthreads=1))
                        for i in range(len(rng))])
    gathered = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(gathered, mine)
    t = torch.tensor([float(rank)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out_q.put((torch.cat(gathered).numpy(), float(t)))
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_sharded_equals_unsharded(scaling):
    world = 2
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scaling, q_)) for r in range(world)]
    for p in procs:
        p.start()
    got, tmax = q_.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == world - 1
    from oracle import oracle as O
    total = bh_range(CFG.BH, world - 1, world, scaling).stop
    q, k, v = make_qkv(CFG, bh_range=range(total))
    ref = np.stack([O.attention(CFG.pattern, q[i], k[i], v[i], CFG.scale, nthreads=1) for i in range(total)])
    assert np.array_equal(got, ref)


def test_bh_range_partitions():
    for world in (1, 2, 4, 8):
        covered = [i for r in range(world) for i in bh_range(96, r, world, "strong")]
        assert covered == list(range(96))
        assert [len(bh_range(96, r, world, "weak")) for r in range(world)] == [96] * world
    with pytest.raises(ValueError):
        bh_range(10, 0, 4, "strong")
