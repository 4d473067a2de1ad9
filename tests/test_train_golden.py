"""Training-step goldens from the reference's own train_step (tests/golden/make_train_golden.py,
pkg/src/fsa/train.py:185-251) against the numpy restatement the GPU tests use
(test_gpu_train.ref_step) fed the C oracle's aggregation: pins the restatement on CPU."""

import numpy as np
import pytest

from conftest import load_golden


@pytest.fixture(scope="module")
def golden_train():
    return load_golden("train_steps.npz")


def test_restated_step_matches_reference_train_step(oracle_mod, golden_train):
    from test_gpu_train import ref_step
    from paper_2511_13645_b200.rng import step_seed

    gt = golden_train
    pl = load_golden("powerlaw_cases.npz")
    N, D, k1, k2, H, C, seed = (int(x) for x in gt["meta"])
    rowptr, col = pl["pl30_rowptr"].astype(np.int32), pl["pl30_col"].astype(np.int32)
    X = pl["pl30_X"].astype(np.float32)
    rng = np.random.default_rng([seed & 0xFFFFFFFF, 0x1D])  # train.py:97-100
    P = {"W1": (rng.standard_normal((2 * D, H)) * np.sqrt(2.0 / (2 * D))).astype(np.float32).astype(np.float64),
         "W2": (rng.standard_normal((H, C)) * np.sqrt(2.0 / H)).astype(np.float32).astype(np.float64),
         "b1": np.zeros(H), "b2": np.zeros(C)}
    M = {k: np.zeros_like(v) for k, v in P.items()}
    V = {k: np.zeros_like(v) for k, v in P.items()}
    for s in range(len(gt["seeds"])):
        seeds, y = gt["seeds"][s], gt["labels"][s]
        out, s1, s2, _, _ = oracle_mod.fused_2hop(rowptr, col, X, seeds, k1, k2, step_seed(seed, s))
        loss, dxa = ref_step(X[seeds].astype(np.float64), out.astype(np.float64), y, P, M, V, s + 1)
        assert abs(loss - float(gt[f"f{s}_loss"])) < 1e-5, s
        assert float(gt[f"f{s}_loss"]) == float(gt[f"b{s}_loss"])
        for k in P:
            np.testing.assert_allclose(P[k], gt[f"f{s}_{k}"], rtol=1e-3, atol=1e-5)
        g = oracle_mod.backward_2hop(dxa.astype(np.float32), s1, s2, N)
        rows = np.flatnonzero(np.any(g != 0, axis=1))
        np.testing.assert_array_equal(rows, gt[f"f{s}_grow"])
        np.testing.assert_allclose(g[rows], gt[f"f{s}_gval"], rtol=1e-3, atol=1e-6)
