"""The CUDA-graph step executor is bitwise identical to the eager operator API, step after
step (fresh neighbourhoods per base seed, persistent gradient buffer kept equal to the
reference's zero-filled-then-scattered buffer), with device inputs and with pinned host inputs
copied on its copy stream (outputs copied back the same way)."""

import numpy as np
import pytest
import torch

from conftest import iter_cases

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("use_graph,overlap,host", [(True, True, False), (False, False, False), (True, False, False),
                                                    (True, True, True)])
def test_executor_matches_eager(golden_powerlaw, use_graph, overlap, host):
    import paper_2511_13645_b200 as fsa
    from paper_2511_13645_b200.executor import Fused2HopStep

    for name, c in iter_cases(golden_powerlaw):
        g = fsa.CsrGraph.from_arrays(c["rowptr"], c["col"], device="cuda", num_nodes=c["N"])
        X = torch.as_tensor(c["X"]).cuda()
        B = 64
        ex = Fused2HopStep(g, X, B, c["k1"], c["k2"], root_offset=5, use_graph=use_graph, overlap_zero=overlap)
        rng = np.random.default_rng(3)
        h_out = [torch.empty((B, X.shape[1]), dtype=X.dtype).pin_memory() for _ in range(2)]
        for step in range(6):
            seeds = torch.as_tensor(rng.integers(0, c["N"], size=B))
            gout = torch.randn((B, X.shape[1]))
            bs = fsa.step_seed(42, step)
            if host:
                out, idx = ex.run(seeds.pin_memory(), bs, gout.pin_memory(), out_host=h_out[step % 2])
                ex.sync_copies()
            else:
                out, idx = ex.run(seeds.cuda(), bs, gout.cuda())
            ref_out, ref_idx = fsa.fused_2hop_forward(g, X, seeds.cuda(), c["k1"], c["k2"], bs, root_offset=5)
            ref_grad = fsa.fused_2hop_backward(gout.cuda(), ref_idx, c["N"])
            torch.cuda.synchronize()
            assert torch.equal(out, ref_out), (name, step)
            if host:
                assert torch.equal(h_out[step % 2], ref_out.cpu()), (name, step)
            assert torch.equal(idx.s1, ref_idx.s1) and torch.equal(idx.s2, ref_idx.s2), (name, step)
            assert torch.equal(ex.grad, ref_grad), (name, step)


@pytest.mark.parametrize("use_graph,host", [(True, False), (False, False), (True, True)])
def test_pipelined_executor_matches_eager(golden_powerlaw, use_graph, host):
    """pipeline=True: step i+1's forward runs on the caller's stream while step i's backward runs
    on the executor's backward stream.  Checked step by step (synchronised), and over a burst of
    back-to-back steps whose forwards and backwards overlap (the last two steps' outputs and the
    last step's gradient)."""
    import paper_2511_13645_b200 as fsa
    from paper_2511_13645_b200.executor import Fused2HopStep

    for name, c in iter_cases(golden_powerlaw):
        g = fsa.CsrGraph.from_arrays(c["rowptr"], c["col"], device="cuda", num_nodes=c["N"])
        X = torch.as_tensor(c["X"]).cuda()
        B = 64
        ex = Fused2HopStep(g, X, B, c["k1"], c["k2"], root_offset=3, use_graph=use_graph, pipeline=True)
        rng = np.random.default_rng(4)
        h_out = [torch.empty((B, X.shape[1]), dtype=X.dtype).pin_memory() for _ in range(2)]

        def inputs(step):
            seeds = torch.as_tensor(rng.integers(0, c["N"], size=B))
            return seeds, torch.randn((B, X.shape[1])), fsa.step_seed(7, step)

        def ref(seeds, gout, bs):
            ro, ri = fsa.fused_2hop_forward(g, X, seeds.cuda(), c["k1"], c["k2"], bs, root_offset=3)
            return ro, ri, fsa.fused_2hop_backward(gout.cuda(), ri, c["N"])

        def run(seeds, gout, bs, step):
            if host:
                return ex.run(seeds.pin_memory(), bs, gout.pin_memory(), out_host=h_out[step % 2])
            return ex.run(seeds.cuda(), bs, gout.cuda())

        for step in range(5):  # synchronised steps
            seeds, gout, bs = inputs(step)
            out, idx = run(seeds, gout, bs, step)
            ex.sync_copies()
            ro, ri, rg = ref(seeds, gout, bs)
            torch.cuda.synchronize()
            assert torch.equal(out, ro) and torch.equal(idx.s1, ri.s1) and torch.equal(idx.s2, ri.s2), (name, step)
            assert torch.equal(ex.grad, rg), (name, step)
            if host:
                assert torch.equal(h_out[step % 2], ro.cpu()), (name, step)
        burst = [inputs(5 + j) for j in range(6)]  # back to back: forwards overlap backwards
        res = [run(sd, go, bs, 5 + j) for j, (sd, go, bs) in enumerate(burst)]
        ex.sync_copies()
        torch.cuda.synchronize()
        for j in (4, 5):  # outputs stay valid until the step after next
            sd, go, bs = burst[j]
            ro, ri, rg = ref(sd, go, bs)
            torch.cuda.synchronize()
            out, idx = res[j]
            assert torch.equal(out, ro) and torch.equal(idx.s2, ri.s2) and torch.equal(idx.s1, ri.s1), (name, j)
            if j == 5:
                assert torch.equal(ex.grad, rg), name
