"""Synthetic benchmark inputs generated on the GPU (harness inputs, not the operator).

``gen_power_law`` follows the reference generator's algorithm (pkg/src/fsa/graph.py:157-203):
truncated-Pareto degree draws rescaled to the target mean, configuration-model stub pairing,
self-loops dropped, symmetrised, de-duplicated, neighbour lists sorted ascending, up to six
rescaling attempts until the realised mean degree is within 8 %.  Only the random number
generator differs (torch's Philox on the device instead of numpy's PCG64 on the host), so the
graphs are statistically alike but not identical; it builds an ogbn-products-shaped graph
(2.45 M nodes, ~124 M arcs) in about a second instead of the reference's ~450 s.
Features and seed batches mirror bench.py:161-179 (standard normal features, shuffled seeds).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .graph import CsrGraph

__all__ = ["SHAPES", "GraphShape", "gen_power_law", "make_features", "seed_batches", "reference_batches"]


@dataclass(frozen=True)
class GraphShape:
    name: str
    num_nodes: int
    avg_degree: float   # realised arcs / node of the symmetrised real graph
    d_feat: int
    k1: int
    k2: int


# BASELINE.json configs
SHAPES = {
    "config1": GraphShape("config1-10k", 10_000, 20.0, 64, 10, 0),
    "arxiv": GraphShape("ogbn-arxiv-shaped", 169_343, 13.7, 128, 10, 10),
    "reddit": GraphShape("reddit-shaped", 232_965, 492.0, 602, 15, 10),
    "products": GraphShape("ogbn-products-shaped", 2_449_029, 50.5, 100, 15, 10),
    "products25": GraphShape("ogbn-products-shaped", 2_449_029, 50.5, 100, 25, 10),
}


def _build_csr(pairs: torch.Tensor, n: int) -> CsrGraph:
    src = torch.cat([pairs[:, 0], pairs[:, 1]])
    dst = torch.cat([pairs[:, 1], pairs[:, 0]])
    key = torch.unique(src * n + dst)  # sorted: rows ascending, neighbours ascending, deduped
    u = key // n
    v = key - u * n
    counts = torch.bincount(u, minlength=n)
    rowptr = torch.zeros(n + 1, dtype=torch.int64, device=pairs.device)
    rowptr[1:] = torch.cumsum(counts, 0)
    if int(rowptr[-1]) >= 2**31:
        raise ValueError("arc count must be < 2**31 for int32 offsets")
    return CsrGraph(n, rowptr.to(torch.int32), v.to(torch.int32).contiguous())


def gen_power_law(num_nodes: int, avg_degree: float, exponent: float, seed: int,
                  device="cuda") -> CsrGraph:
    if num_nodes < 2:
        raise ValueError("num_nodes must be >= 2")
    if avg_degree < 1 or avg_degree > num_nodes - 1:
        raise ValueError("avg_degree must be in [1, num_nodes - 1]")
    if exponent <= 1.0:
        raise ValueError("exponent must be > 1")
    device = torch.device(device)
    dmax = num_nodes - 1
    gen = torch.Generator(device=device)
    gen.manual_seed((seed & 0xFFFFFFFF) * 1000003 + 17)
    a1 = 1.0 - exponent
    u = torch.rand(num_nodes, generator=gen, device=device, dtype=torch.float64)
    raw = (1.0 + u * (float(dmax) ** a1 - 1.0)) ** (1.0 / a1)
    raw_mean = float(raw.mean())
    scale = 1.0
    best, best_err = None, float("inf")
    for attempt in range(6):
        scaled = raw * (avg_degree * scale / raw_mean)
        target = torch.clamp(torch.round(scaled), 1, dmax).to(torch.int64)
        stubs = torch.repeat_interleave(torch.arange(num_nodes, device=device), target)
        pg = torch.Generator(device=device)
        pg.manual_seed((seed & 0xFFFFFFFF) * 1000003 + 1 + attempt)
        stubs = stubs[torch.randperm(stubs.numel(), generator=pg, device=device)]
        if stubs.numel() % 2:
            stubs = stubs[:-1]
        pairs = stubs.view(-1, 2)
        pairs = pairs[pairs[:, 0] != pairs[:, 1]]
        del stubs
        g = _build_csr(pairs, num_nodes)
        del pairs
        realized = g.num_edges / num_nodes
        err = abs(realized - avg_degree) / avg_degree
        if err < best_err:
            best, best_err = g, err
        if err <= 0.08:
            return g
        scale = min(max(scale * avg_degree / max(realized, 0.5), 0.25), 8.0)
    return best


def make_features(num_nodes: int, d_feat: int, seed: int, dtype=torch.float32, device="cuda",
                  row_stride: int | None = None) -> torch.Tensor:
    """Standard-normal features (bench.py:161-162); optional padded row stride."""
    gen = torch.Generator(device=device)
    gen.manual_seed((seed & 0xFFFFFFFF) * 1000003 + 2)
    stride = row_stride or d_feat
    X = torch.randn(num_nodes, stride, generator=gen, device=device, dtype=torch.float32)
    return X[:, :d_feat].to(dtype) if stride == d_feat else X.to(dtype)[:, :d_feat]


def seed_batches(num_nodes: int, batch: int, seed: int, device="cuda"):
    """Shuffled seed batches, ragged tail dropped, reshuffled per epoch (bench.py:172-179)."""
    gen = torch.Generator(device=device)
    gen.manual_seed((seed & 0xFFFFFFFF) * 1000003 + 3)
    while True:
        perm = torch.randperm(num_nodes, generator=gen, device=device)
        for start in range(0, num_nodes - batch + 1, batch):
            yield perm[start:start + batch]


def reference_batches(num_nodes: int, batch: int, base_seed: int, device="cuda"):
    """The reference's own batch order, bit-exact (pkg/src/fsa/bench.py:172-179): numpy
    ``default_rng([base_seed & 0xFFFFFFFF, 3]).permutation(num_nodes)`` per epoch, ragged tail
    dropped.  The permutation is drawn on the host (numpy is the generator the contract names)
    and uploaded once per epoch; batches are int64 device views of it."""
    import numpy as np

    rng = np.random.default_rng([base_seed & 0xFFFFFFFF, 3])
    while True:
        perm = torch.from_numpy(rng.permutation(num_nodes)).to(device)
        for start in range(0, num_nodes - batch + 1, batch):
            yield perm[start:start + batch]
