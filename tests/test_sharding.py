"""Multi-process instance sharding on CPU (gloo, world_size 2): shards are
disjoint and cover all instances, each rank merges only its shard, and the
gathered per-instance results equal a single-process merged run."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_13062_b200.sharding import gather_instance_outputs, shard_range


def test_shard_ranges_partition():
    for n in (1, 7, 8, 256):
        for w in (1, 2, 3, 8):
            seen = [i for r in range(w) for i in shard_range(n, w, r)]
            assert seen == list(range(n))
            sizes = [len(shard_range(n, w, r)) for r in range(w)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import executor as OX
    from paper_2009_13062_b200 import build_zoo, merge, model_inputs
    from paper_2009_13062_b200 import workloads as W

    ids = list(shard_range(n, world, rank))
    graph = W.build_graph("attnblock", batch=2)
    stores = [W.build_weights("attnblock", model=m) for m in ids]
    merged, mstore = merge(graph, stores)
    inputs = [model_inputs(graph, model=m) for m in ids]
    outs = OX.execute(merged.graph, mstore.tensors, merged.bind_inputs(inputs))
    got = gather_instance_outputs([torch.from_numpy(o) for o in outs], n)
    if rank == 0:
        q.put([g.numpy() for g in got])
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_merge_matches_single_process():
    n, world = 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from oracle import executor as OX
    from paper_2009_13062_b200 import build_zoo, merge, model_inputs
    graph, stores = build_zoo("attnblock", num_models=n, batch=2)
    merged, mstore = merge(graph, stores)
    inputs = [model_inputs(graph, model=m) for m in range(n)]
    want = OX.execute(merged.graph, mstore.tensors, merged.bind_inputs(inputs))
    assert len(got) == n
    for a, b in zip(got, want):
        assert a.tobytes() == b.tobytes()
