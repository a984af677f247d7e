"""Multi-process (gloo, world_size 2, CPU) tests of the batch-sharding host logic: every rank runs
its slice of the batch (here through the oracle, since the CPU box has no GPU), the gathered
outputs equal the unsharded run, and the timing reduction is the max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_01302_b200.shard import shard_range, shard_sizes


def test_shard_ranges_cover_batch():
    for batch in range(1, 40):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(batch, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == batch
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = shard_sizes(batch, world)
            assert max(sizes) - min(sizes) <= 1 and sum(sizes) == batch


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import workloads as W
        from oracle import OracleGraph
        from paper_2011_01302_b200.shard import gather_outputs, max_over_ranks
        net = W.squeezenet(batch=batch, image=64)
        x = net.make_input()
        b, e = shard_range(batch, world, rank)
        local_net = net.with_batch(e - b)
        y = OracleGraph(local_net).run_sequential(x[b:e])[local_net.n_ops]
        full = gather_outputs(torch.from_numpy(y), world, batch)
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            ref = OracleGraph(net).run_sequential(x)[net.n_ops]
            q.put((float(np.abs(full.numpy() - ref).max()), t, tuple(full.shape)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [4, 5])
def test_sharded_run_equals_unsharded_gloo(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    err, t, shape = q.get(timeout=10)
    assert err == 0.0                      # images are independent: sharding is exact
    assert t == 2.0                        # max over ranks
    assert shape[0] == batch
