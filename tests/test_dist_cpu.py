"""Seed-sharded data parallelism on CPU (gloo, world size 2): the host-side sharding and the
head-gradient all-reduce that bench.py / train.py run over NCCL on GPUs.  The per-shard op here
is the C oracle with root_offset; concatenating the shards must reproduce the single-process
batch bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, iter_cases, load_golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_2511_13645_b200.shard import allreduce_grads, shard_batch

        res = {}
        for name, c in iter_cases(load_golden("powerlaw_cases.npz")):
            seeds = torch.as_tensor(c["seeds"])
            local, off = shard_batch(seeds, rank, world)
            out, s1, s2, _, _ = oracle.fused_2hop(c["rowptr"].astype(np.int32), c["col"].astype(np.int32), c["X"],
                                                  local.numpy(), c["k1"], c["k2"], c["base_seed"], root_offset=off)
            parts = [None] * world
            dist.all_gather_object(parts, (out, s1, s2))
            res[name] = parts
        g = {"W": torch.full((3, 2), float(rank + 1)), "b": torch.full((4,), 10.0 * (rank + 1))}
        allreduce_grads(g, average=True)
        res["grads"] = (g["W"].numpy(), g["b"].numpy())
        if rank == 0:
            outq.put(res)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shards_match_single_process(oracle_mod):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for name, c in iter_cases(load_golden("powerlaw_cases.npz")):
        out, s1, s2, _, _ = oracle_mod.fused_2hop(c["rowptr"].astype(np.int32), c["col"].astype(np.int32), c["X"],
                                                  c["seeds"], c["k1"], c["k2"], c["base_seed"])
        parts = res[name]
        assert np.concatenate([p[0] for p in parts]).tobytes() == out.tobytes(), name
        assert np.array_equal(np.concatenate([p[1] for p in parts]), s1), name
        assert np.array_equal(np.concatenate([p[2] for p in parts]), s2), name
    W, b = res["grads"]
    assert np.all(W == 1.5) and np.all(b == 15.0)


def test_shard_bounds_cover_the_batch():
    from paper_2511_13645_b200.shard import shard_bounds
    for B in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(B, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(4, 2, 2)
