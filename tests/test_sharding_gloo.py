"""Multi-process batch sharding on CPU (gloo, world_size 2).

The B200 path shards the batch of a planned graph contiguously over ranks
(north_star piece 4; runtime.split_ranges / DevicePool.shards) and needs no
collective on the hot path.  This test runs the host-side protocol with two
gloo ranks: each rank takes its shard, runs the forward (the CPU oracle stands
in for the device program here), and an all_gather (test-only, not part of
the product path) reassembles the batch, which must equal the unsharded run.
bench.py uses the same split and a max-reduce of timings."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, queue):
    import torch
    import torch.distributed as dist
    import oracle
    from paper_1809_02697_b200 import DevicePool, build_model, model_input
    from paper_1809_02697_b200.executor import with_batch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        batch = 6
        g = build_model("resnet18", batch=batch, image=32, num_classes=10, softmax=False)
        feeds = model_input(g)
        shards = DevicePool(list(range(world)), "bf16").shards(batch)
        dev, (lo, hi) = shards[rank]
        assert dev == rank
        local = oracle.execute_reference(with_batch(g, hi - lo), {"data": feeds["data"][lo:hi]})[0]
        parts = [torch.zeros((b - a, 10)) for _, (a, b) in shards]
        dist.all_gather(parts, torch.from_numpy(local))
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)     # bench.py's max-over-ranks timing
        if rank == 0:
            full = oracle.execute_reference(g, feeds)[0]
            got = torch.cat(parts).numpy()
            queue.put((float(np.abs(got - full).max()), float(t.item())))
    finally:
        dist.destroy_process_group()


def test_two_rank_batch_sharding_matches_unsharded():
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, queue)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    err, tmax = queue.get(timeout=10)
    assert err == 0.0
    assert tmax == 2.0
