"""Data-parallel training on the GPU: the product train_step / GraphTrainStep in a process group.

* world 2 over gloo, both ranks on cuda:0 (the GPU box has one GPU; NCCL refuses two ranks on one
  device): each rank runs the fused op on its shard of the global batch (root_offset = its first
  global position); the shards' s1 / s2 / out are bitwise the 1-GPU run of the global batch, and
  after the weighted all-reduce of the head gradients both ranks hold the same parameters, equal
  to a single-process run of the global batch within fp32 reduction-order tolerance
  (the caller mirrored is pkg/src/fsa/train.py:185-251);
* world 1 over NCCL with the collective forced on: the all-reduce is captured into the step's
  CUDA graph (GraphTrainStep) and the results equal the eager train_step.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from conftest import iter_cases, load_golden

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(c):
    import paper_2511_13645_b200 as fsa
    N = c["N"]
    g = fsa.CsrGraph.from_arrays(c["rowptr"], c["col"], device="cuda", num_nodes=N)
    X = torch.as_tensor(c["X"].astype(np.float32)).cuda()
    rng = np.random.default_rng(21)
    steps = [(rng.integers(0, N, size=36), rng.integers(0, 5, size=36)) for _ in range(3)]
    return fsa, g, X, steps


def _worker(rank, world, port, outq, graph_mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_13645_b200 import train
        from paper_2511_13645_b200.shard import shard_bounds
        name, c = next(iter_cases(load_golden("powerlaw_cases.npz")))
        fsa, g, X, steps = _setup(c)
        state = train.init_train_state(X.shape[1], 16, 5, base_seed=5)
        gbuf = torch.zeros_like(X)
        res = {"fwd": [], "loss": []}
        if graph_mode:
            lo, hi = shard_bounds(36, rank, world)
            gts = train.GraphTrainStep(g, X, hi - lo, (c["k1"], c["k2"]), state, root_offset=lo, global_batch=36)
        for i, (seeds, y) in enumerate(steps):
            bs = fsa.step_seed(9, i)
            if graph_mode:
                r = gts.run(torch.as_tensor(seeds[lo:hi]).cuda(), torch.as_tensor(y[lo:hi]).cuda(), bs)
                res["fwd"].append((gts.ex.out.cpu().numpy(), gts.ex.s1.cpu().numpy()))
            else:
                r = train.train_step(g, X, fsa.SeedBatch(seeds, y), (c["k1"], c["k2"]), bs, "fused", state,
                                     grad_scratch=gbuf)
                lo, hi = shard_bounds(36, rank, world)
                out, idx = fsa.fused_2hop_forward(g, X, torch.as_tensor(seeds[lo:hi]).cuda(), c["k1"], c["k2"], bs,
                                                  root_offset=lo)
                res["fwd"].append((out.cpu().numpy(), idx.s1.cpu().numpy(), idx.s2.cpu().numpy()))
            res["loss"].append(float(r.loss))
        res["params"] = {k: getattr(state, k).cpu().numpy() for k in train.PARAM_NAMES}
        res["steps"] = state.step_count
        parts = [None] * world
        torch.distributed.all_gather_object(parts, res)
        if rank == 0:
            outq.put(parts)
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.parametrize("graph_mode", [False, True], ids=["train_step", "GraphTrainStep"])
def test_gloo_world2_on_one_gpu(graph_mode):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from paper_2511_13645_b200 import train
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, graph_mode)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single-process reference run of the global batch
    name, c = next(iter_cases(load_golden("powerlaw_cases.npz")))
    fsa, g, X, steps = _setup(c)
    state = train.init_train_state(X.shape[1], 16, 5, base_seed=5)
    gbuf = torch.zeros_like(X)
    for i, (seeds, y) in enumerate(steps):
        bs = fsa.step_seed(9, i)
        out, idx = fsa.fused_2hop_forward(g, X, torch.as_tensor(seeds).cuda(), c["k1"], c["k2"], bs)
        r = train.train_step(g, X, fsa.SeedBatch(seeds, y), (c["k1"], c["k2"]), bs, "fused", state, grad_scratch=gbuf)
        got_out = np.concatenate([p["fwd"][i][0] for p in parts])
        got_s1 = np.concatenate([p["fwd"][i][1] for p in parts])
        assert got_out.tobytes() == out.cpu().numpy().tobytes(), i  # shards are bitwise the 1-GPU rows
        assert np.array_equal(got_s1, idx.s1.cpu().numpy()), i
        if not graph_mode:
            assert np.array_equal(np.concatenate([p["fwd"][i][2] for p in parts]), idx.s2.cpu().numpy()), i
        for p in parts:  # the loss is the global-batch mean on every rank
            assert abs(p["loss"][i] - float(r.loss)) <= 1e-5 * max(1.0, abs(float(r.loss))), i
    for k in train.PARAM_NAMES:
        np.testing.assert_array_equal(parts[0]["params"][k], parts[1]["params"][k])  # identical update
        np.testing.assert_allclose(parts[0]["params"][k], getattr(state, k).cpu().numpy(), rtol=1e-5, atol=1e-6)
    assert parts[0]["steps"] == parts[1]["steps"] == 3


def _nccl_worker(port, outq):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    torch.distributed.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2511_13645_b200 import train
        name, c = next(iter_cases(load_golden("powerlaw_cases.npz")))
        fsa, g, X, steps = _setup(c)
        s_graph, s_eager = (train.init_train_state(X.shape[1], 16, 5, base_seed=6) for _ in range(2))
        gts = train.GraphTrainStep(g, X, 36, (c["k1"], c["k2"]), s_graph, allreduce=True)
        gbuf = torch.zeros_like(X)
        diffs = []
        for i in range(6):
            seeds, y = steps[i % 3]
            bs = fsa.step_seed(10, i)
            rg = gts.run(torch.as_tensor(seeds).cuda(), torch.as_tensor(y).cuda(), bs)
            re = train.train_step(g, X, fsa.SeedBatch(seeds, y), (c["k1"], c["k2"]), bs, "fused", s_eager,
                                  grad_scratch=gbuf)
            torch.cuda.synchronize()
            diffs.append(max([abs(float(rg.loss) - float(re.loss))] +
                             [float((getattr(s_graph, k) - getattr(s_eager, k)).abs().max()) for k in train.PARAM_NAMES]))
        outq.put((diffs, gts.graphs[0] is not None and gts.graphs[1] is not None, s_graph.step_count))
    finally:
        torch.distributed.destroy_process_group()


def test_nccl_allreduce_captured_in_step_graph():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    diffs, captured, steps = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert captured, "both step parities captured as CUDA graphs (all-reduce inside)"
    assert max(diffs) <= 1e-6, diffs
    assert steps == 6


def test_sparse_zero_state_follows_the_buffer():
    """zero='sparse' re-zeroes only what this buffer's previous backward wrote: after a 'full'
    call, after a new buffer at a recycled address, and with the caller's ids changed in place."""
    import paper_2511_13645_b200 as fsa
    name, c = next(iter_cases(load_golden("powerlaw_cases.npz")))
    N = c["N"]
    g = fsa.CsrGraph.from_arrays(c["rowptr"], c["col"], device="cuda", num_nodes=N)
    X = torch.as_tensor(c["X"].astype(np.float32)).cuda()
    seeds = torch.as_tensor(c["seeds"]).cuda()
    _, i1 = fsa.fused_2hop_forward(g, X, seeds, c["k1"], c["k2"], 1)
    _, i2 = fsa.fused_2hop_forward(g, X, seeds.flip(0), c["k1"], c["k2"], 2)
    go = torch.randn((seeds.numel(), X.shape[1]), device="cuda")
    want2 = fsa.fused_2hop_backward(go, i2, N)
    buf = torch.zeros_like(X)
    fsa.fused_2hop_backward(go, i1, N, out=buf, zero="sparse")
    fsa.fused_2hop_backward(go, i2, N, out=buf, zero="full")   # must update the remembered rows
    fsa.fused_2hop_backward(go, i1, N, out=buf, zero="sparse")
    i1.s2.fill_(-1)  # the caller reuses its index buffer: our remembered rows are a private copy
    fsa.fused_2hop_backward(go, i2, N, out=buf, zero="sparse")
    assert torch.equal(buf, want2)
    del buf  # a new buffer, possibly at the recycled address: its first sparse call fills it fully
    buf2 = torch.empty((N, X.shape[1]), device="cuda")
    buf2.view(torch.int32).fill_(0x40400000)  # 3.0
    fsa.fused_2hop_backward(go, i2, N, out=buf2, zero="sparse")
    assert torch.equal(buf2, want2)


def test_nonfinite_step_does_not_advance_the_count():
    from paper_2511_13645_b200 import train
    state = train.init_train_state(4, 8, 3, base_seed=1)
    grads = {k: torch.ones_like(getattr(state, k)) for k in train.PARAM_NAMES}
    train.adamw_step(state, grads)
    grads["W2"][0, 0] = float("inf")
    assert not bool(train.adamw_step(state, grads))
    assert state.step_count == 1  # the reference raises before incrementing (train.py:163-170)
