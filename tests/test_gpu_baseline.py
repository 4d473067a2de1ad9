"""Unfused comparator: the materialised GPU pipeline is bitwise equal to
the fused op and to the oracle (reference tests/test_baseline.py:27-58: fp32 and fp64 bitwise),
forward and backward, dense and dedup, and its block holds what fusion removes."""

import numpy as np
import pytest
import torch

from conftest import iter_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fsa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2511_13645_b200 as m
    return m


def T(a, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a)).cuda()
    return t if dtype is None else t.to(dtype)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16])
@pytest.mark.parametrize("dedup", [False, True])
def test_2hop_baseline_equals_fused(fsa, oracle_mod, golden_powerlaw, dtype, dedup):
    for name, c in iter_cases(golden_powerlaw):
        g = fsa.CsrGraph.from_arrays(c["rowptr"], c["col"], device="cuda", num_nodes=c["N"])
        X = T(c["X"]).to(dtype)
        seeds = T(c["seeds"])
        out_f, idx = fsa.fused_2hop_forward(g, X, seeds, c["k1"], c["k2"], c["base_seed"])
        out_b, blk = fsa.baseline_forward(g, X, seeds, c["k1"], c["k2"], c["base_seed"], dedup=dedup)
        assert torch.equal(blk.ids1, idx.s1) and torch.equal(blk.ids2, idx.s2), name
        assert torch.equal(out_b, out_f), name
        if dtype == torch.float32:
            ref, *_ = oracle_mod.fused_2hop(c["rowptr"], c["col"], c["X"], c["seeds"], c["k1"], c["k2"],
                                            c["base_seed"])
            assert out_b.cpu().numpy().tobytes() == ref.tobytes(), name
        gout = T(c["gout2"]).to(dtype)
        assert torch.equal(fsa.baseline_backward(gout, blk, c["N"]), fsa.fused_2hop_backward(gout, idx, c["N"])), name
        T2, D = idx.s2.numel(), X.shape[1]
        if dedup:
            assert blk.gathered is None and blk.uniq_features.shape[0] == len(np.unique(c["s2"][c["s2"] >= 0]))
        else:
            assert blk.gathered.shape == (T2, D)
        assert blk.nbytes() > 0


@pytest.mark.parametrize("which", ["small", "powerlaw"])
def test_1hop_baseline_equals_golden(fsa, golden_small, golden_powerlaw, which):
    for name, c in iter_cases(golden_small if which == "small" else golden_powerlaw):
        g = fsa.CsrGraph.from_arrays(c["rowptr"], c["col"], device="cuda", num_nodes=c["N"])
        X = T(c["X"])
        seeds = T(c["seeds"])
        out_b, blk = fsa.baseline_1hop_forward(g, X, seeds, c["k1"], c["base_seed"])
        assert blk.ids1.cpu().numpy().tobytes() == c["samples"].tobytes(), name
        assert out_b.cpu().numpy().tobytes() == c["out1"].tobytes(), name
        grad = fsa.baseline_backward(T(c["gout1"]), blk, c["N"])
        assert grad.cpu().numpy().tobytes() == c["grad1"].tobytes(), name
        out2, blk2 = fsa.baseline_forward(g, X, seeds, c["k1"], c["k2"], c["base_seed"])
        assert out2.cpu().numpy().tobytes() == c["out2"].tobytes(), name
        grad2 = fsa.baseline_backward(T(c["gout2"]), blk2, c["N"])
        assert grad2.cpu().numpy().tobytes() == c["grad2"].tobytes(), name


def test_wide_rows_hub_baseline(fsa):
    """Wide bf16 rows, a hub next to many multi-hit nodes: the materialised backward goes through
    every row writer with per-slot rows."""
    rng = np.random.default_rng(5)
    n, deg, D = 3000, 40, 602
    col = np.stack([np.concatenate([[0], np.sort(rng.choice(np.arange(1, n), deg - 1, replace=False))])
                    for _ in range(n)]).astype(np.int32).ravel()
    g = fsa.CsrGraph.from_arrays(np.arange(0, n * deg + 1, deg, dtype=np.int64), col, device="cuda", num_nodes=n)
    X = torch.randn((n, D), device="cuda").to(torch.bfloat16)
    seeds = torch.from_numpy(rng.integers(0, n, 256)).cuda()
    out_f, idx = fsa.fused_2hop_forward(g, X, seeds, 15, 10, 77)
    out_b, blk = fsa.baseline_forward(g, X, seeds, 15, 10, 77)
    assert torch.equal(out_b, out_f)
    gout = torch.randn((256, D), device="cuda").to(torch.bfloat16)
    assert torch.equal(fsa.baseline_backward(gout, blk, n), fsa.fused_2hop_backward(gout, idx, n))
