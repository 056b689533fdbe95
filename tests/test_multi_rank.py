"""World-size-2 gloo tests of the multi-GPU host logic, on CPU.

The data path has no collective (independent systems, §8e), so what can go
wrong across ranks is the partitioning, the seeding and the timing
reduction. Each rank solves its shard with the oracle (CPU), the shards are
gathered and compared with a single-process solve of the whole batch.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2309_08079_b200.sharding import max_over_ranks, seeds, shard_range, weak_shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shard_range_partitions_exactly():
    for batch in (1, 5, 64, 4096, 4097):
        for world in (1, 2, 3, 4, 8):
            got = []
            for r in range(world):
                a, b = shard_range(batch, world, r)
                assert 0 <= a <= b <= batch
                got.extend(range(a, b))
            assert got == list(range(batch))


def test_weak_shard_and_seeds():
    assert weak_shard(4096, 0) == (0, 4096)
    assert weak_shard(4096, 3) == (3 * 4096, 4 * 4096)
    assert seeds(100, 2, 5) == [102, 103, 104]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, batch, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist
    import pyoracle as orc
    import paper_2309_08079_b200.api as api
    from paper_2309_08079_b200.types import PcgConfig, PrecondKind
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, last = shard_range(batch, world, rank)
    kb = api.random_kkt_batch(777 + first, last - first, 7, 3, 2)  # system i <- seed 777 + i
    cfg = PcgConfig(epsilon=1e-10)
    lam = np.stack([orc.solve(kb.system(i), PrecondKind.symmetric_stair, cfg=cfg).lambda_
                    for i in range(last - first)])
    t = max_over_ranks(float(rank + 1), dist)
    gathered = [None] * world
    dist.all_gather_object(gathered, (first, last, lam))
    if rank == 0:
        np.save(os.path.join(out_dir, "t.npy"), np.array([t]))
        full = np.concatenate([g[2] for g in sorted(gathered, key=lambda g: g[0])])
        np.save(os.path.join(out_dir, "lam.npy"), full)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_batch_equals_single_process(tmp_path, orc):
    import paper_2309_08079_b200.api as api
    from paper_2309_08079_b200.types import PcgConfig, PrecondKind
    batch, world = 7, 2
    mp.spawn(_worker, args=(world, _free_port(), batch, str(tmp_path)), nprocs=world, join=True)
    lam = np.load(tmp_path / "lam.npy")
    assert float(np.load(tmp_path / "t.npy")[0]) == 2.0  # max over ranks
    kb = api.random_kkt_batch(777, batch, 7, 3, 2)
    cfg = PcgConfig(epsilon=1e-10)
    want = np.stack([orc.solve(kb.system(i), PrecondKind.symmetric_stair, cfg=cfg).lambda_
                     for i in range(batch)])
    assert np.array_equal(lam, want)


def _gpu_worker(rank, world, port, batch, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_2309_08079_b200.api as api
    from paper_2309_08079_b200.types import PcgConfig, PrecondKind
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, last = shard_range(batch, world, rank)
    # the bench's weak-scaling seeds: system i <- seed 2309 + i, on this rank's shard
    kb = api.random_kkt_batch(2309 + first, last - first, 63, 14, 7)
    lam, reps = api.solve_batched(kb, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
    t = max_over_ranks(float(rank + 1), dist)
    gathered = [None] * world
    dist.all_gather_object(gathered, (first, last, lam, list(reps.iterations)))
    if rank == 0:
        np.save(os.path.join(out_dir, "t.npy"), np.array([t]))
        g = sorted(gathered, key=lambda g: g[0])
        np.save(os.path.join(out_dir, "lam.npy"), np.concatenate([x[2] for x in g]))
        np.save(os.path.join(out_dir, "it.npy"), np.concatenate([np.array(x[3]) for x in g]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_rank_sharded_batch_on_the_device_path(tmp_path):
    """World size 2 (gloo, both ranks on the test box's GPU) through libb2p's
    solve_batched on contiguous shards: the gathered result equals the
    single-process batch bitwise (the bench's N > 1 data path)."""
    import paper_2309_08079_b200.api as api
    from paper_2309_08079_b200.types import PcgConfig, PrecondKind
    api.require_device()
    batch, world = 300, 2
    mp.spawn(_gpu_worker, args=(world, _free_port(), batch, str(tmp_path)), nprocs=world, join=True)
    kb = api.random_kkt_batch(2309, batch, 63, 14, 7)
    lam1, rep1 = api.solve_batched(kb, PrecondKind.symmetric_stair, 1, PcgConfig(epsilon=1e-8))
    assert float(np.load(tmp_path / "t.npy")[0]) == 2.0
    assert np.array_equal(np.load(tmp_path / "lam.npy"), lam1)
    assert np.array_equal(np.load(tmp_path / "it.npy"), rep1.iterations)
