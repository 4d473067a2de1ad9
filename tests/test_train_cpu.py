"""CPU checks of the training step's host-side math (no GPU): the library head path of
train.sage_head (taken for non-fp32 / CPU tensors) and the per-tensor AdamW path against the
reference's numpy formulas (pkg/src/fsa/train.py:111-184)."""

import numpy as np
import pytest
import torch


def _np_head(xs, xa, y, P):
    """train.py:111-160 in numpy float64."""
    concat = np.concatenate([xs, xa], axis=1)
    hidden = np.maximum(concat @ P["W1"] + P["b1"], 0.0)
    logits = hidden @ P["W2"] + P["b2"]
    shifted = logits - logits.max(axis=1, keepdims=True)
    e = np.exp(shifted)
    total = e.sum(axis=1, keepdims=True)
    logp = shifted - np.log(total)
    B = len(y)
    loss = -logp[np.arange(B), y].mean()
    dl = e / total
    dl[np.arange(B), y] -= 1
    dl /= B
    dW2 = hidden.T @ dl
    dh = (dl @ P["W2"].T) * (hidden > 0)
    dW1 = concat.T @ dh
    dconcat = dh @ P["W1"].T
    return loss, {"W1": dW1, "b1": dh.sum(0), "W2": dW2, "b2": dl.sum(0)}, dconcat[:, xs.shape[1]:]


@pytest.mark.parametrize("B,D,H,C", [(64, 12, 16, 5), (33, 7, 8, 3)])
def test_sage_head_library_path_matches_reference_math(B, D, H, C):
    from paper_2511_13645_b200 import train
    rng = np.random.default_rng(B)
    X = rng.standard_normal((100, D))
    seeds = rng.integers(0, 100, B)
    xa = rng.standard_normal((B, D))
    y = rng.integers(0, C, B)
    state = train.init_train_state(D, H, C, base_seed=2, dtype=torch.float64, device="cpu")
    state.b1.copy_(torch.from_numpy(rng.standard_normal(H)))
    state.b2.copy_(torch.from_numpy(rng.standard_normal(C)))
    P = {k: getattr(state, k).numpy().copy() for k in train.PARAM_NAMES}
    loss, grads, dx = train.sage_head(torch.from_numpy(X), torch.from_numpy(seeds), torch.from_numpy(xa),
                                      torch.from_numpy(y), state)
    l_ref, g_ref, dx_ref = _np_head(X[seeds], xa, y, P)
    assert abs(float(loss) - l_ref) < 1e-12
    np.testing.assert_allclose(dx.numpy(), dx_ref, rtol=1e-10, atol=1e-14)
    for k in train.PARAM_NAMES:
        np.testing.assert_allclose(grads[k].numpy(), g_ref[k], rtol=1e-10, atol=1e-14)


def test_adamw_library_path_matches_reference_update_and_skips_nonfinite():
    from paper_2511_13645_b200 import train
    state = train.init_train_state(6, 8, 3, base_seed=5, dtype=torch.float64, device="cpu")
    h = state.hyper
    rng = np.random.default_rng(1)
    P = {k: getattr(state, k).numpy().copy() for k in train.PARAM_NAMES}
    M = {k: np.zeros_like(v) for k, v in P.items()}
    V = {k: np.zeros_like(v) for k, v in P.items()}
    for t in range(1, 3):
        G = {k: rng.standard_normal(v.shape) for k, v in P.items()}
        assert bool(train.adamw_step(state, {k: torch.from_numpy(g) for k, g in G.items()}))
        bc1, bc2 = 1.0 - h.beta1 ** t, 1.0 - h.beta2 ** t
        for k in P:
            p, m, v, g = P[k], M[k], V[k], G[k]
            p -= h.lr * h.weight_decay * p
            m *= h.beta1
            m += (1.0 - h.beta1) * g
            v *= h.beta2
            v += (1.0 - h.beta2) * (g * g)
            p -= h.lr * (m / bc1) / (np.sqrt(v / bc2) + h.eps)
    for k in P:
        np.testing.assert_allclose(getattr(state, k).numpy(), P[k], rtol=1e-12, atol=1e-15)
    before = {k: getattr(state, k).clone() for k in train.PARAM_NAMES}
    bad = {k: torch.zeros_like(getattr(state, k)) for k in train.PARAM_NAMES}
    bad["W1"][0, 0] = float("inf")
    assert not bool(train.adamw_step(state, bad))
    assert state.step_count == 2  # the reference raises before incrementing (train.py:163-170)
    for k in train.PARAM_NAMES:
        assert torch.equal(getattr(state, k), before[k])
