"""GPU SAGE training step (train.py) against the reference's own train_step (golden vectors,
tests/golden/train_steps.npz) and a numpy restatement of the reference step
(pkg/src/fsa/train.py:111-251) fed the oracle's aggregation: loss, parameters and moments must
agree to fp32 GEMM tolerance step after step; the fused feature gradient bitwise."""

import numpy as np
import pytest
import torch

from conftest import iter_cases

pytestmark = pytest.mark.gpu


def ref_step(xs, xa, y, P, M, V, t, lr=3e-3, wd=5e-4, b1=0.9, b2=0.999, eps=1e-8):
    concat = np.concatenate([xs, xa], 1)
    hid = np.maximum(concat @ P["W1"] + P["b1"], 0)
    logits = hid @ P["W2"] + P["b2"]
    B = len(y)
    sh = logits - logits.max(1, keepdims=True)
    e = np.exp(sh)
    tot = e.sum(1, keepdims=True)
    loss = float(-(sh - np.log(tot))[np.arange(B), y].mean())
    dl = e / tot
    dl[np.arange(B), y] -= 1
    dl /= B
    g = {"W2": hid.T @ dl, "b2": dl.sum(0)}
    dh = (dl @ P["W2"].T) * (hid > 0)
    g["W1"] = concat.T @ dh
    g["b1"] = dh.sum(0)
    dxa = (dh @ P["W1"].T)[:, xs.shape[1]:]
    bc1, bc2 = 1 - b1 ** t, 1 - b2 ** t
    for k in P:
        P[k] = P[k] - lr * wd * P[k]
        M[k] = M[k] * b1 + (1 - b1) * g[k]
        V[k] = V[k] * b2 + (1 - b2) * g[k] * g[k]
        P[k] = P[k] - lr * (M[k] / bc1) / (np.sqrt(V[k] / bc2) + eps)
    return loss, dxa


def test_train_step_matches_reference_math(oracle_mod, golden_powerlaw):
    import paper_2511_13645_b200 as fsa
    from paper_2511_13645_b200 import train

    name, c = next(iter_cases(golden_powerlaw))
    N, D = c["N"], c["X"].shape[1]
    X = c["X"].astype(np.float32)
    g = fsa.CsrGraph.from_arrays(c["rowptr"], c["col"], device="cuda", num_nodes=N)
    Xd = torch.as_tensor(X).cuda()
    rng = np.random.default_rng(9)
    state = train.init_train_state(D, 32, 5, base_seed=42)
    P = {k: getattr(state, k).double().cpu().numpy() for k in train.PARAM_NAMES}
    M = {k: np.zeros_like(v) for k, v in P.items()}
    V = {k: np.zeros_like(v) for k, v in P.items()}
    gbuf = torch.zeros((N, D), device="cuda")
    for step in range(4):
        seeds = rng.integers(0, N, size=48)
        y = rng.integers(0, 5, size=48)
        bs = fsa.step_seed(42, step)
        res = train.train_step(g, Xd, fsa.SeedBatch(seeds, y), (c["k1"], c["k2"]), bs, "fused", state,
                               grad_scratch=gbuf)
        out, s1, s2, _, _ = oracle_mod.fused_2hop(c["rowptr"].astype(np.int32), c["col"].astype(np.int32), X, seeds,
                                                  c["k1"], c["k2"], bs)
        loss, dxa = ref_step(X[seeds].astype(np.float64), out.astype(np.float64), y, P, M, V, step + 1)
        assert bool(res.grads_applied)
        assert abs(float(res.loss) - loss) < 1e-4 * max(1.0, abs(loss)), step
        for k in P:
            np.testing.assert_allclose(getattr(state, k).double().cpu().numpy(), P[k], rtol=1e-3, atol=1e-5)
        # the fused backward of the step's dx_agg: compare with the oracle replay of the same ids
        ref_g = oracle_mod.backward_2hop(dxa.astype(np.float32), s1, s2, N)
        np.testing.assert_allclose(gbuf.cpu().numpy(), ref_g, rtol=1e-3, atol=1e-6)


def test_nonfinite_gradient_skips_the_update():
    from paper_2511_13645_b200 import train
    state = train.init_train_state(4, 8, 3, base_seed=1)
    before = {k: getattr(state, k).clone() for k in train.PARAM_NAMES}
    grads = {k: torch.zeros_like(getattr(state, k)) for k in train.PARAM_NAMES}
    grads["b1"][0] = float("nan")
    ok = train.adamw_step(state, grads)
    assert not bool(ok)
    for k in train.PARAM_NAMES:
        assert torch.equal(getattr(state, k), before[k])


@pytest.mark.parametrize("dedup", [False, True])
def test_baseline_variant_trains_identically(golden_powerlaw, dedup):
    """train_step(variant="baseline") (the materialised comparator) gives the same losses,
    parameters and feature gradients as variant="fused", step after step (train.py:185-251)."""
    import paper_2511_13645_b200 as fsa
    from paper_2511_13645_b200 import train

    name, c = next(iter_cases(golden_powerlaw))
    N, D = c["N"], c["X"].shape[1]
    g = fsa.CsrGraph.from_arrays(c["rowptr"], c["col"], device="cuda", num_nodes=N)
    Xd = torch.as_tensor(c["X"].astype(np.float32)).cuda()
    states = [train.init_train_state(D, 32, 5, base_seed=7) for _ in range(2)]
    bufs = [torch.zeros((N, D), device="cuda") for _ in range(2)]
    rng = np.random.default_rng(4)
    for step in range(3):
        batch = fsa.SeedBatch(rng.integers(0, N, size=40), rng.integers(0, 5, size=40))
        bs = fsa.step_seed(7, step)
        rf = train.train_step(g, Xd, batch, (c["k1"], c["k2"]), bs, "fused", states[0], grad_scratch=bufs[0])
        rb = train.train_step(g, Xd, batch, (c["k1"], c["k2"]), bs, "baseline", states[1], grad_scratch=bufs[1],
                              dedup=dedup)
        assert torch.equal(rf.loss, rb.loss) and rf.sampled_pairs == rb.sampled_pairs
        assert torch.equal(bufs[0], bufs[1])
        for k in train.PARAM_NAMES:
            assert torch.equal(getattr(states[0], k), getattr(states[1], k))
    with pytest.raises(ValueError, match="variant"):
        train.train_step(g, Xd, batch, (c["k1"], c["k2"]), 1, "unfused", states[0])


@pytest.mark.parametrize("use_graph", [True, False])
def test_graph_train_step_matches_eager(golden_powerlaw, use_graph):
    """GraphTrainStep (the fused training step as CUDA graphs, device-side step count) against
    the eager train_step: same losses, parameters, sampled pairs and feature gradients."""
    import paper_2511_13645_b200 as fsa
    from paper_2511_13645_b200 import train

    name, c = next(iter_cases(golden_powerlaw))
    N, D = c["N"], c["X"].shape[1]
    g = fsa.CsrGraph.from_arrays(c["rowptr"], c["col"], device="cuda", num_nodes=N)
    Xd = torch.as_tensor(c["X"].astype(np.float32)).cuda()
    B = 40
    s_eager, s_graph = (train.init_train_state(D, 32, 5, base_seed=3) for _ in range(2))
    gbuf = torch.zeros((N, D), device="cuda")
    gts = train.GraphTrainStep(g, Xd, B, (c["k1"], c["k2"]), s_graph, use_graph=use_graph)
    rng = np.random.default_rng(8)
    for step in range(6):
        seeds = torch.as_tensor(rng.integers(0, N, size=B)).cuda()
        y = torch.as_tensor(rng.integers(0, 5, size=B)).cuda()
        bs = fsa.step_seed(3, step)
        re = train.train_step(g, Xd, fsa.SeedBatch(seeds, y), (c["k1"], c["k2"]), bs, "fused", s_eager,
                              grad_scratch=gbuf)
        rg = gts.run(seeds, y, bs)
        torch.cuda.synchronize()
        assert int(rg.sampled_pairs) == re.sampled_pairs, step
        assert abs(float(rg.loss) - float(re.loss)) <= 1e-6 * max(1.0, abs(float(re.loss))), step
        assert bool(rg.grads_applied)
        for k in train.PARAM_NAMES:
            torch.testing.assert_close(getattr(s_graph, k), getattr(s_eager, k), rtol=1e-6, atol=1e-7)
        torch.testing.assert_close(gts.feature_grad, gbuf, rtol=1e-6, atol=1e-7)
    assert s_graph.step_count == s_eager.step_count == 6


@pytest.mark.parametrize("variant", ["fused", "baseline"])
def test_train_step_matches_reference_goldens(variant):
    """Four train_step calls from init_train_state(D, 32, 5, base_seed=42) against the reference's
    own train_step run on the same batches (tests/golden/train_steps.npz, made by
    tests/golden/make_train_golden.py from pkg/src/fsa/train.py:185-251): losses, sampled pairs,
    parameters, AdamW moments and the feature-gradient buffer after every step."""
    from conftest import load_golden
    import paper_2511_13645_b200 as fsa
    from paper_2511_13645_b200 import train

    gt = load_golden("train_steps.npz")
    pl = load_golden("powerlaw_cases.npz")
    N, D, k1, k2, H, C, seed = (int(x) for x in gt["meta"])
    g = fsa.CsrGraph.from_arrays(pl["pl30_rowptr"], pl["pl30_col"], device="cuda", num_nodes=N)
    Xd = torch.as_tensor(pl["pl30_X"].astype(np.float32)).cuda()
    state = train.init_train_state(D, H, C, base_seed=seed)
    gbuf = torch.zeros((N, D), device="cuda")
    p = variant[0]
    for s in range(len(gt["seeds"])):
        batch = fsa.SeedBatch(gt["seeds"][s], gt["labels"][s])
        res = train.train_step(g, Xd, batch, (k1, k2), fsa.step_seed(seed, s), variant, state, grad_scratch=gbuf)
        assert res.sampled_pairs == int(gt[f"{p}{s}_pairs"]), s
        assert bool(res.grads_applied) == bool(gt[f"{p}{s}_applied"])
        assert abs(float(res.loss) - float(gt[f"{p}{s}_loss"])) < 1e-5, s
        for k in train.PARAM_NAMES:
            np.testing.assert_allclose(getattr(state, k).cpu().numpy(), gt[f"{p}{s}_{k}"], rtol=1e-3, atol=1e-5)
            np.testing.assert_allclose(state.m[k].cpu().numpy(), gt[f"{p}{s}_m_{k}"], rtol=1e-3, atol=1e-7)
            np.testing.assert_allclose(state.v[k].cpu().numpy(), gt[f"{p}{s}_v_{k}"], rtol=1e-3, atol=1e-9)
        gb = gbuf.cpu().numpy()
        rows = np.flatnonzero(np.any(gb != 0, axis=1))
        np.testing.assert_array_equal(rows, gt[f"{p}{s}_grow"])
        np.testing.assert_allclose(gb[rows], gt[f"{p}{s}_gval"], rtol=1e-3, atol=1e-6)
    assert state.step_count == len(gt["seeds"])


@pytest.mark.parametrize("B,D,H,C", [(1024, 100, 256, 47), (1000, 602, 256, 41), (37, 128, 64, 5)])
def test_sage_head_kernels_match_torch_fp64(B, D, H, C):
    """fsa_sage_head_fwd_bwd (the CUDA head of the training step) against the library head
    (head_forward + cross_entropy + head_backward, train.py:111-160) run in fp64."""
    from paper_2511_13645_b200 import train
    gen = torch.Generator(device="cuda").manual_seed(B + D)
    N = 5000
    X = torch.randn(N, D + 3, device="cuda", generator=gen)[:, :D]  # strided rows
    seeds = torch.randint(0, N, (B,), device="cuda", generator=gen)
    agg = torch.randn(B, D, device="cuda", generator=gen)
    labels = torch.randint(0, C, (B,), device="cuda", generator=gen)
    state = train.init_train_state(D, H, C, base_seed=3)
    state.b1.normal_(generator=gen)  # non-zero biases exercise the bias paths
    state.b2.normal_(generator=gen)
    loss, grads, dx = train.sage_head(X, seeds, agg, labels, state)
    s64 = train.init_train_state(D, H, C, base_seed=3, dtype=torch.float64)
    for n in train.PARAM_NAMES:
        getattr(s64, n).copy_(getattr(state, n))
    logits, cache = train.head_forward(X.double().index_select(0, seeds), agg.double(), s64)
    l64, dl = train.cross_entropy(logits, labels)
    g64, _, dx64 = train.head_backward(dl, cache, s64)
    torch.testing.assert_close(loss.double(), l64, rtol=1e-5, atol=1e-6)
    torch.testing.assert_close(dx.double(), dx64, rtol=1e-4, atol=1e-7)
    for n in train.PARAM_NAMES:
        torch.testing.assert_close(grads[n].double(), g64[n], rtol=1e-4, atol=1e-7)


def test_sage_head_bad_label_gives_nonfinite_update_skip():
    from paper_2511_13645_b200 import train
    B, D, H, C = 64, 16, 32, 4
    X = torch.randn(100, D, device="cuda")
    seeds = torch.arange(B, device="cuda")
    agg = torch.randn(B, D, device="cuda")
    labels = torch.zeros(B, dtype=torch.int64, device="cuda")
    labels[5] = C  # out of range
    state = train.init_train_state(D, H, C, base_seed=1)
    before = {k: getattr(state, k).clone() for k in train.PARAM_NAMES}
    loss, grads, _ = train.sage_head(X, seeds, agg, labels, state)
    assert not torch.isfinite(loss)
    assert not bool(train.adamw_step(state, grads))
    for k in train.PARAM_NAMES:
        assert torch.equal(getattr(state, k), before[k])


def test_adamw_kernel_matches_reference_update():
    """fsa_adamw_step (train.adamw_step on fp32 CUDA state) against the reference's numpy update
    (train.py:163-184) over three steps: same operation order in fp32, so bitwise."""
    from paper_2511_13645_b200 import train
    state = train.init_train_state(12, 16, 5, base_seed=4)
    rng = np.random.default_rng(9)
    P = {k: getattr(state, k).cpu().numpy().copy() for k in train.PARAM_NAMES}
    M = {k: np.zeros_like(v) for k, v in P.items()}
    V = {k: np.zeros_like(v) for k, v in P.items()}
    h = state.hyper
    for t in range(1, 4):
        G = {k: rng.standard_normal(v.shape).astype(np.float32) for k, v in P.items()}
        assert bool(train.adamw_step(state, {k: torch.from_numpy(g).cuda() for k, g in G.items()}))
        bc1, bc2 = 1.0 - h.beta1 ** t, 1.0 - h.beta2 ** t
        for k in P:
            p, m, v, g = P[k], M[k], V[k], G[k]
            p -= h.lr * h.weight_decay * p
            m *= h.beta1
            m += (1.0 - h.beta1) * g
            v *= h.beta2
            v += (1.0 - h.beta2) * (g * g)
            p -= h.lr * (m / bc1) / (np.sqrt(v / bc2) + h.eps)
    assert state.step_count == 3
    for k in P:
        np.testing.assert_array_equal(getattr(state, k).cpu().numpy(), P[k])
        np.testing.assert_array_equal(state.m[k].cpu().numpy(), M[k])
        np.testing.assert_array_equal(state.v[k].cpu().numpy(), V[k])
