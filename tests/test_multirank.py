"""Multi-process (world_size 2, gloo on CPU) coverage of the N>1 paths: ensemble sharding
+ the single diagnostics all-gather, and the bench's max-over-ranks reduction."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2408_03483_b200 import ensemble


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_partitions_members():
    for members in (1, 7, 64):
        for world in (1, 2, 3, 4, 8):
            ids = [i for r in range(world) for i in ensemble.shard(members, world, r)]
            assert ids == list(range(members))
            sizes = [len(ensemble.shard(members, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, members, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = ensemble.shard(members, world, rank)
    # stand-in member runner (the GPU runner is ensemble.run_member); record layout RECORD
    recs = [[m, 5, 1.0 + m, 3, 4, 5, 6, 7, 8, 10.0 * rank] for m in mine]
    out = ensemble.gather_records(recs, world)
    import bench

    mx = bench.allreduce_max(world, float(rank + 1), 0)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, out.tolist(), mx))


@pytest.mark.parametrize("members", [5, 64])
def test_two_rank_gather(members):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, members, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, out, mx in res:
        out = np.array(out)
        assert sorted(out[:, 0].astype(int).tolist()) == list(range(members))
        assert mx == 2.0
        # members of rank 1 carry its tag
        assert set(out[out[:, 0] >= ensemble.shard(members, 2, 1).start][:, 9]) == {10.0}
