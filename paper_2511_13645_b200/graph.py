"""Device-resident CSR graph and seed batch (mirror of the reference ``fsa.graph`` data model).

Reference: pkg/src/fsa/graph.py:38-105.  The operator's input contract is unchanged: int32
``rowptr[N+1]`` and ``col[E]`` with every neighbour list sorted ascending and de-duplicated
(graph.py:108-151) — Algorithm R's output depends on that order.  Here both arrays live in
HBM as torch int32 tensors; any reference-style graph object (``num_nodes``, numpy ``rowptr``
/ ``col``) is accepted too and uploaded once per (object, device).
"""

from __future__ import annotations

import os
import weakref
from dataclasses import dataclass
from typing import Optional, Union

import numpy as np
import torch

MAX_NODES = 2**31 - 1

__all__ = ["CsrGraph", "SeedBatch", "GraphFormatError", "as_device_graph", "as_seed_tensor", "save_csr_cache",
           "load_csr_cache"]

CACHE_MAGIC = b"FSA1"


class GraphFormatError(ValueError):
    """Malformed graph file (graph.py:30-31)."""


@dataclass(frozen=True, eq=False)
class CsrGraph:
    """CSR adjacency with int32 ``rowptr``/``col`` tensors (graph.py:38-85)."""

    num_nodes: int
    rowptr: torch.Tensor
    col: torch.Tensor

    @classmethod
    def from_arrays(cls, rowptr, col, device: Union[str, torch.device, None] = None,
                    num_nodes: Optional[int] = None, validate: bool = True) -> "CsrGraph":
        rp = torch.as_tensor(np.asarray(rowptr) if not torch.is_tensor(rowptr) else rowptr)
        cl = torch.as_tensor(np.asarray(col) if not torch.is_tensor(col) else col)
        if device is None:
            device = "cuda"
        rp = rp.to(device=device, dtype=torch.int32).contiguous()
        cl = cl.to(device=device, dtype=torch.int32).contiguous()
        n = int(rp.numel() - 1) if num_nodes is None else int(num_nodes)
        g = cls(num_nodes=n, rowptr=rp, col=cl)
        if validate:
            g.validate()
        return g

    @property
    def device(self) -> torch.device:
        return self.rowptr.device

    @property
    def num_edges(self) -> int:
        return int(self.col.numel())

    def degree(self, u: int) -> int:
        return int(self.rowptr[u + 1] - self.rowptr[u])

    def neighbors(self, u: int) -> torch.Tensor:
        return self.col[int(self.rowptr[u]):int(self.rowptr[u + 1])]

    def degrees(self) -> torch.Tensor:
        return (self.rowptr[1:] - self.rowptr[:-1]).to(torch.int64)

    def max_degree(self) -> int:
        return int(self.degrees().max()) if self.num_nodes > 0 else 0

    def validate(self) -> None:
        """CSR invariants of graph.py:64-85 (host-side checks, one sync)."""
        n = self.num_nodes
        if n <= 0:
            raise ValueError("graph must have at least one node")
        if n > MAX_NODES:
            raise ValueError("num_nodes must be < 2**31")
        if self.rowptr.dtype != torch.int32 or self.col.dtype != torch.int32:
            raise ValueError("rowptr and col must be int32")
        if tuple(self.rowptr.shape) != (n + 1,):
            raise ValueError(f"rowptr must have length N+1={n + 1}")
        if int(self.rowptr[0]) != 0:
            raise ValueError("rowptr[0] must be 0")
        if bool((self.rowptr[1:] < self.rowptr[:-1]).any()):
            raise ValueError("rowptr must be non-decreasing")
        if int(self.rowptr[-1]) != self.col.numel():
            raise ValueError("rowptr[N] must equal len(col)")
        if self.col.numel() and (int(self.col.min()) < 0 or int(self.col.max()) >= n):
            raise ValueError("col entries must lie in [0, N)")

    def to(self, device) -> "CsrGraph":
        return CsrGraph(self.num_nodes, self.rowptr.to(device), self.col.to(device))

    def cpu_arrays(self):
        return self.rowptr.cpu().numpy(), self.col.cpu().numpy()


@dataclass(eq=False)
class SeedBatch:
    """Mini-batch frontier: seed node ids (+ optional labels) (graph.py:88-105)."""

    seeds: torch.Tensor
    labels: Optional[torch.Tensor] = None

    def __post_init__(self):
        self.seeds = _as_int64(self.seeds)
        if self.seeds.ndim != 1 or self.seeds.numel() == 0:
            raise ValueError("seed batch must be a non-empty 1-D array")
        if self.labels is not None:
            self.labels = _as_int64(self.labels)
            if self.labels.shape != self.seeds.shape:
                raise ValueError("labels must match seeds in shape")

    def __len__(self) -> int:
        return int(self.seeds.numel())


def _as_int64(x) -> torch.Tensor:
    if torch.is_tensor(x):
        return x.to(torch.int64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.int64))


# reference-style graph objects -> device graphs (one upload per object and device)
_GRAPH_CACHE: dict = {}


def as_device_graph(graph, device: torch.device) -> CsrGraph:
    if isinstance(graph, CsrGraph):
        if graph.device != device:
            raise ValueError(f"graph lives on {graph.device}, features on {device}")
        return graph
    key = (id(graph), str(device))
    hit = _GRAPH_CACHE.get(key)
    if hit is not None:
        ref, g = hit
        if ref() is graph:
            return g
    g = CsrGraph.from_arrays(graph.rowptr, graph.col, device=device, num_nodes=graph.num_nodes,
                             validate=False)
    try:
        ref = weakref.ref(graph, lambda _r, k=key: _GRAPH_CACHE.pop(k, None))
    except TypeError:
        return g
    _GRAPH_CACHE[key] = (ref, g)
    return g


def as_seed_tensor(seeds, device: torch.device) -> torch.Tensor:
    """Seed positions as a contiguous int64 device tensor (fused.py:80-86 shape check)."""
    if isinstance(seeds, SeedBatch) or (hasattr(seeds, "seeds") and not torch.is_tensor(seeds)):
        seeds = seeds.seeds
    t = _as_int64(seeds)
    if t.ndim != 1 or t.numel() == 0:
        raise ValueError("seed batch must be a non-empty 1-D array")
    return t.to(device, non_blocking=True)


# ---- FSA1 binary CSR cache (graph.py:266-292), byte-compatible with the reference -------------
def save_csr_cache(graph, path) -> None:
    """Write the binary CSR cache: magic "FSA1", N (u64 LE), rowptr, col (i32 LE)."""
    if isinstance(graph, CsrGraph):
        rowptr, col = graph.cpu_arrays()
        n = graph.num_nodes
    else:
        rowptr, col, n = np.asarray(graph.rowptr), np.asarray(graph.col), int(graph.num_nodes)
    with open(path, "wb") as fh:
        fh.write(CACHE_MAGIC)
        fh.write(np.uint64(n).astype("<u8").tobytes())
        fh.write(np.ascontiguousarray(rowptr, dtype="<i4").tobytes())
        fh.write(np.ascontiguousarray(col, dtype="<i4").tobytes())


def load_csr_cache(path, device: Union[str, torch.device, None] = None) -> CsrGraph:
    """Read an FSA1 cache into a device graph (same checks and messages as graph.py:276-292)."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != CACHE_MAGIC:
            raise GraphFormatError(f"{path}: bad magic {magic!r}, expected {CACHE_MAGIC!r}")
        hdr = fh.read(8)
        if len(hdr) != 8:
            raise GraphFormatError(f"{path}: truncated header")
        n = int(np.frombuffer(hdr, dtype="<u8")[0])
        if n == 0 or n > MAX_NODES:
            raise GraphFormatError(f"{path}: implausible node count {n}")
        if size < 12 + 4 * (n + 1):
            raise GraphFormatError(f"{path}: truncated rowptr")
        rowptr = np.fromfile(fh, dtype="<i4", count=n + 1)
        nnz = int(rowptr[-1])
        if nnz < 0 or size < 12 + 4 * (n + 1) + 4 * nnz:
            raise GraphFormatError(f"{path}: truncated col")
        col = np.fromfile(fh, dtype="<i4", count=nnz)
    return CsrGraph.from_arrays(rowptr.astype(np.int32), col.astype(np.int32), device=device, num_nodes=n)
