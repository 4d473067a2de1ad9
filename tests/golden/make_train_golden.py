"""Generate training-step golden vectors from the REFERENCE's own train_step (build container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_train_golden.py

Runs /root/reference/pkg/src/fsa/train.py:185-251 (``train_step``, variant "fused" and
"baseline", with a persistent ``grad_scratch``) for four steps on the pl30 power-law golden graph
(tests/golden/powerlaw_cases.npz) from ``init_train_state(D, 32, 5, base_seed=42)``, and records
per step: the loss, sampled_pairs, the four head parameters and their AdamW moments after the
update, and the feature-gradient buffer (ids + rows of its nonzero rows).  The GPU test
(tests/test_gpu_train.py::test_train_step_matches_reference_goldens) replays the same batches
through paper_2511_13645_b200.train.train_step and compares.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path[:0] = [str(REF_SRC)]

from fsa import train  # noqa: E402
from fsa.bench import _step_seed  # noqa: E402
from fsa.graph import CsrGraph, SeedBatch  # noqa: E402

STEPS = 4
BATCH = 48
HIDDEN, CLASSES = 32, 5
BASE_SEED = 42


def main():
    z = np.load(OUT / "powerlaw_cases.npz")
    rowptr = z["pl30_rowptr"].astype(np.int32)
    col = z["pl30_col"].astype(np.int32)
    X = z["pl30_X"].astype(np.float32)
    N, D = X.shape
    k1, k2 = 15, 10
    g = CsrGraph(N, rowptr, col)
    rng = np.random.default_rng(9)
    seeds = rng.integers(0, N, size=(STEPS, BATCH)).astype(np.int64)
    labels = rng.integers(0, CLASSES, size=(STEPS, BATCH)).astype(np.int64)
    out = {"seeds": seeds, "labels": labels, "meta": np.array([N, D, k1, k2, HIDDEN, CLASSES, BASE_SEED])}
    for variant in ("fused", "baseline"):
        st = train.init_train_state(D, HIDDEN, CLASSES, base_seed=BASE_SEED)
        gbuf = np.zeros((N, D), dtype=np.float32)
        p = variant[0]
        for s in range(STEPS):
            res = train.train_step(g, X, SeedBatch(seeds[s], labels[s]), (k1, k2), _step_seed(BASE_SEED, s),
                                   variant, st, grad_scratch=gbuf)
            out[f"{p}{s}_loss"] = np.float64(res.loss)
            out[f"{p}{s}_pairs"] = np.int64(res.sampled_pairs)
            out[f"{p}{s}_applied"] = np.bool_(res.grads_applied)
            for name, prm in st.named_params():
                out[f"{p}{s}_{name}"] = prm.copy()
                out[f"{p}{s}_m_{name}"] = st.m[name].copy()
                out[f"{p}{s}_v_{name}"] = st.v[name].copy()
            rows = np.flatnonzero(np.any(gbuf != 0, axis=1))
            out[f"{p}{s}_grow"] = rows.astype(np.int32)
            out[f"{p}{s}_gval"] = gbuf[rows].copy()
    np.savez_compressed(OUT / "train_steps.npz", **out)
    print("wrote", OUT / "train_steps.npz", {k: out[k] for k in out if k.endswith("_loss")})


if __name__ == "__main__":
    main()
