"""The batch-sharding protocol of bench.py / execute() run against the DEVICE
executor by two gloo ranks that share GPU 0 (the CPU version with the oracle
standing in for the device program is tests/test_sharding_gloo.py).

Each rank compiles the planned graph for its contiguous shard
(runtime.split_ranges, the reference's chunking rule runtime.py:129-149),
uploads its slice through pinned staging, runs the CUDA-graph forward, and a
test-only all_gather reassembles the batch.  The reassembled logits must equal
the same shard programs run in one process bit for bit (nothing but the batch
split differs), and match the CPU oracle within the bf16 bound with identical
top-1.  The ranks never wait on each other's kernels: there is no collective
on the hot path."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

BATCH, IMAGE, CLASSES = 6, 64, 10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard_logits(lo, hi, feeds):
    from paper_1809_02697_b200 import (DeviceProgram, ExecutablePlan, build_model,
                                       compile_graph)
    g = build_model("resnet18", batch=hi - lo, image=IMAGE, num_classes=CLASSES, softmax=False)
    prog = DeviceProgram(ExecutablePlan.compile(compile_graph(g, mode="bf16")), 0, "bf16")
    return prog.run({"data": np.ascontiguousarray(feeds["data"][lo:hi])})[0]


def _worker(rank, world, port, queue):
    import torch
    import torch.distributed as dist
    from paper_1809_02697_b200 import DevicePool, build_model, model_input
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        g = build_model("resnet18", batch=BATCH, image=IMAGE, num_classes=CLASSES, softmax=False)
        feeds = model_input(g, seed=4)
        shards = DevicePool([0] * world, "bf16").shards(BATCH)
        _, (lo, hi) = shards[rank]
        local = _shard_logits(lo, hi, feeds)
        parts = [torch.zeros((b - a, CLASSES)) for _, (a, b) in shards]
        dist.all_gather(parts, torch.from_numpy(local))
        if rank == 0:
            queue.put(torch.cat(parts).numpy())
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_shard_the_device_executor(cuda):
    import oracle
    from paper_1809_02697_b200 import DevicePool, build_model, model_input
    ctx = mp.get_context("spawn")
    queue = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, queue)) for r in range(2)]
    for p in procs:
        p.start()
    got = queue.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    g = build_model("resnet18", batch=BATCH, image=IMAGE, num_classes=CLASSES, softmax=False)
    feeds = model_input(g, seed=4)
    shards = DevicePool([0, 0], "bf16").shards(BATCH)
    here = np.concatenate([_shard_logits(lo, hi, feeds) for _, (lo, hi) in shards])
    assert np.array_equal(got, here)
    ref = oracle.execute_reference(g, feeds)[0]
    assert oracle.rel_err(got, ref) < 2e-2
    assert (got.argmax(1) == ref.argmax(1)).all()
