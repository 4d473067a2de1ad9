"""Work and traffic accounting of one fused 2-hop step, shared by ``bench.py``
and the benchmark grid (``benchgrid``).

Algorithmic bytes are what the op must move at minimum: ids and CSR entries it reads, the
feature rows it gathers, the means it writes, and in the backward the gradient rows it reads
and writes.  Draws are the Algorithm-R iterations of every sampled chain
(pkg/src/fsa/kernels.py:63-67: ``deg - k`` draws for a node of degree ``deg > k``).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch


def alg_bytes(B: int, k1: int, k2: int, D: int, E: int, T1: int, T2: int, U2: int):
    """(forward, backward) algorithmic bytes of a 2-hop batch.  E = element size, T1 / T2 =
    valid first / second-hop slots, U2 = distinct valid second-hop nodes."""
    idx = 4 * B * k1 * (1 + k2)
    fwd = 8 * B + 8 * (B + T1) + 4 * (T1 + T2) + E * D * T2 + E * D * B + idx
    bwd = E * D * B + idx + E * D * U2
    return fwd, bwd


@dataclass(frozen=True)
class StepWork:
    T1: int
    T2: int
    U2: int
    draws: int

    def bytes(self, B: int, k1: int, k2: int, D: int, E: int) -> int:
        f, b = alg_bytes(B, k1, k2, D, E, self.T1, self.T2, self.U2)
        return f + b


def step_work(graph, seeds: torch.Tensor, s1: torch.Tensor, s2: torch.Tensor, k1: int, k2: int) -> StepWork:
    """Counts of one batch from its saved indices (device tensors; one host sync)."""
    rp = graph.rowptr.to(torch.int64)
    deg = rp[1:] - rp[:-1]
    v1 = s1[s1 >= 0].to(torch.int64)
    v2 = s2[s2 >= 0].to(torch.int64)
    draws = (deg[seeds.to(torch.int64)] - k1).clamp_min(0).sum() + (deg[v1] - k2).clamp_min(0).sum()
    vals = torch.stack([v1.new_tensor(v1.numel()), v2.new_tensor(v2.numel()),
                        v2.new_tensor(torch.unique(v2).numel()), draws]).tolist()
    return StepWork(*(int(x) for x in vals))
