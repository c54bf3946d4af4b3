"""World-size-2 (gloo, CPU) test of the multi-rank orchestration bench.py uses:
the (b, h) split of shard.bh_range, and shard.gather_and_check -- all-gather of every rank's O
shard and the bitwise comparison of every rank's first/last slices with a one-process
recomputation.  On CPU the fp64 oracle is the stand-in for the device kernel (no GPU here); the
same functions run over NCCL in bench.py --gpus N."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_16847_b200.shard import bh_range, check_slices, gather_and_check
from workloads import Config, Pattern, make_qkv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = Config("gloo_small", Pattern("global_local", 96, lo=8, hi=8, n_global=4), 2, 3, 16, "fp32", 301)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_slices(idx):
    from oracle import oracle as O
    q, k, v = make_qkv(CFG, bh_range=list(idx))
    return torch.stack([torch.from_numpy(O.attention(CFG.pattern, q[i], k[i], v[i], CFG.scale, nthreads=1))
                        for i in range(len(idx))])


def _worker(rank, world, port, scaling, corrupt, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = bh_range(CFG.BH, rank, world, scaling)
    mine = _oracle_slices(rng)
    if corrupt and rank == 1:
        mine[-1, 0, 0] += 1e-3                    # a rank whose last slice differs must be caught
    res = gather_and_check(mine, _oracle_slices)
    t = torch.tensor([float(rank)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out_q.put((res, float(t)))
    dist.destroy_process_group()


def _run(world, scaling, corrupt):
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scaling, corrupt, q_)) for r in range(world)]
    for p in procs:
        p.start()
    res, tmax = q_.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == world - 1
    return res


def test_gather_and_check_strong_split():
    res = _run(2, "strong", corrupt=False)
    assert res["bitwise_equal_to_one_device"]
    assert res["gathered_slices"] == CFG.BH
    assert res["slices_checked"] == check_slices(2, CFG.BH // 2)


def test_gather_and_check_catches_a_bad_shard():
    res = _run(2, "strong", corrupt=True)
    assert not res["bitwise_equal_to_one_device"]


def test_bh_range_partitions():
    for world in (1, 2, 4, 8):
        covered = [i for r in range(world) for i in bh_range(96, r, world, "strong")]
        assert covered == list(range(96))
        assert [len(bh_range(96, r, world, "weak")) for r in range(world)] == [96] * world
        # Mistral: 128 (b, h) units, 16 per rank at 8 GPUs (BASELINE.json configs[4])
        assert len(bh_range(128, world - 1, world, "strong")) == 128 // world
    with pytest.raises(ValueError):
        bh_range(10, 0, 4, "strong")


def test_check_slices_covers_every_rank():
    idx = check_slices(4, 12)
    for r in range(4):
        assert r * 12 in idx and r * 12 + 11 in idx
    assert check_slices(2, 1) == [0, 1]


def test_bench_refuses_knobs():
    env = dict(os.environ, SPLAT_TC_DEBUG="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "refusing" in r.stderr


def test_bench_gpus_mismatch_under_launcher():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    env.pop("SPLAT_TC_DEBUG", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr
