"""Unfused comparator on the GPU: sample, materialise blocks, gather features, aggregate.

Mirror of the reference's ``fsa.baseline`` (pkg/src/fsa/baseline.py:1-200).
The stages use the same sampler and the same accumulation order as the fused operator.  The only
difference is that the sampled-id blocks, the gathered feature rows, the per-slot partial means
and the per-slot gradient block are materialised in HBM between stages: that traffic and memory
is precisely what fusion removes.  Outputs are bitwise equal to the fused ops.

Stages and kernels:
  sample              fused.sample_1hop / sample_2hop      (kernels.sample_1hop / sample_2hop)
  gather              fsa_gather_rows                      (kernels.gather_rows)
  partial / root mean fsa_group_mean                       (kernels.agg_1hop_block,
                                                            partials_2hop_block / _dedup,
                                                            agg_2hop_from_partials)
  backward            fsa_baseline_*_bwd                   (kernels.expand_grad, invert_targets,
                                                            scatter_from_block)

With half-precision features the partial means are kept in fp32, as the fused op keeps them in
registers, so the result is rounded once, exactly like the fused op.  ``dedup=True`` gathers one
row per distinct sampled node (torch.unique, ascending like np.unique) plus a slot remap.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple

import torch

from . import _lib
from .fused import (
    _DTYPE_CODE,
    _remember_rows,
    _check_features,
    _grad_buffer,
    _grad_inputs,
    _index_tensor,
    _pick_device,
    _set_device,
    _stream,
    _ws,
    sample_1hop,
    sample_2hop,
)
from .graph import as_device_graph

__all__ = ["MaterializedBlock", "baseline_1hop_forward", "baseline_forward", "baseline_backward"]


def _acc_dtype(dtype: torch.dtype) -> torch.dtype:
    return torch.float64 if dtype == torch.float64 else torch.float32


@dataclass
class MaterializedBlock:
    """The baseline's intermediate tensors (baseline.py:29-60): hop ids plus gathered features.

    One-hop blocks have ``ids2``/``take2`` None and ``gathered`` (B*k, D).  In dedup mode the
    dense gather is replaced by ``uniq_features`` (one row per distinct sampled node) and
    ``uniq_remap`` (flat slot -> row of uniq_features, -1 for padding)."""

    ids1: torch.Tensor
    take1: torch.Tensor
    ids2: Optional[torch.Tensor] = None
    take2: Optional[torch.Tensor] = None
    gathered: Optional[torch.Tensor] = None
    uniq_features: Optional[torch.Tensor] = None
    uniq_remap: Optional[torch.Tensor] = None

    def arrays(self) -> List[torch.Tensor]:
        return [a for a in (self.ids1, self.take1, self.ids2, self.take2, self.gathered, self.uniq_features,
                            self.uniq_remap) if a is not None]

    def nbytes(self) -> int:
        """Bytes the block keeps alive (what the fused op never materialises)."""
        return sum(a.numel() * a.element_size() for a in self.arrays())

    def valid_pairs(self) -> int:
        pairs = int(self.take1.sum())
        if self.take2 is not None:
            pairs += int(self.take2.sum())
        return pairs


def _features(graph, X):
    dev = _pick_device(graph, X)
    if not torch.is_tensor(X):
        raise ValueError("features must be a torch tensor on the GPU")
    g = as_device_graph(graph, dev)
    _check_features(g, X)
    return g, X.to(dev), dev


def _gather(X: torch.Tensor, ids: torch.Tensor, n: int, st: int) -> torch.Tensor:
    D = X.shape[1]
    out = torch.empty((n, D), dtype=X.dtype, device=X.device)
    _lib.check(_lib.load().fsa_gather_rows(X.data_ptr(), D, X.stride(0), _DTYPE_CODE[X.dtype], ids.data_ptr(), n,
                                           out.data_ptr(), D, st), "fsa_gather_rows")
    return out


def _group_mean(src: torch.Tensor, remap: Optional[torch.Tensor], take: torch.Tensor, k: int, G: int,
                out_dtype: torch.dtype, code: int, st: int) -> torch.Tensor:
    D = src.shape[1]
    out = torch.empty((G, D), dtype=out_dtype, device=src.device)
    src_acc = int(src.dtype == _acc_dtype(src.dtype) and code not in (_lib.FSA_F32, _lib.FSA_F64))
    out_acc = int(out_dtype == _acc_dtype(out_dtype) and code not in (_lib.FSA_F32, _lib.FSA_F64))
    _lib.check(_lib.load().fsa_group_mean(src.data_ptr(), src.stride(0), src_acc,
                                          remap.data_ptr() if remap is not None else None, take.data_ptr(),
                                          int(k), G, D, code, out.data_ptr(), D, out_acc, st), "fsa_group_mean")
    return out


def baseline_1hop_forward(graph, X, seeds, k: int, base_seed: int, meter=None, *, root_offset: int = 0,
                          validate: bool = True) -> Tuple[torch.Tensor, MaterializedBlock]:
    """sample -> materialise the (B*k, D) gather -> aggregate (baseline.py:63-89)."""
    g, X, dev = _features(graph, X)
    if k < 1:
        raise ValueError("fanout k must be >= 1")
    ids1, take1 = sample_1hop(g, seeds, k, base_seed, root_offset=root_offset, device=dev, validate=validate)
    B = ids1.shape[0]
    st = _stream(dev)
    code = _DTYPE_CODE[X.dtype]
    gathered = _gather(X, ids1.reshape(-1), B * k, st)
    out = _group_mean(gathered, None, take1, k, B, X.dtype, code, st)
    return out, MaterializedBlock(ids1=ids1, take1=take1, gathered=gathered)


def baseline_forward(graph, X, seeds, k1: int, k2: int, base_seed: int, meter=None, dedup: bool = False, *,
                     root_offset: int = 0, validate: bool = True) -> Tuple[torch.Tensor, MaterializedBlock]:
    """Two-hop unfused pipeline (baseline.py:92-154): sample; materialise the hop-id tensors and
    the gathered second-hop features (deduplicated across seeds when ``dedup``); compute the
    nested mean from the materialised tensors only."""
    g, X, dev = _features(graph, X)
    if k1 < 1 or k2 < 1:
        raise ValueError("fanouts must be >= 1")
    s1, s2, t1, t2 = sample_2hop(g, seeds, k1, k2, base_seed, root_offset=root_offset, device=dev,
                                 validate=validate)
    B = s1.shape[0]
    st = _stream(dev)
    code = _DTYPE_CODE[X.dtype]
    acc = _acc_dtype(X.dtype)
    flat = s2.reshape(-1)
    block = MaterializedBlock(ids1=s1, take1=t1, ids2=s2, take2=t2)
    if dedup:
        valid = flat >= 0
        uniq, inv = torch.unique(flat[valid], sorted=True, return_inverse=True)
        remap = torch.full((flat.numel(),), -1, dtype=torch.int32, device=dev)
        remap[valid] = inv.to(torch.int32)
        uniq32 = uniq.to(torch.int32)
        block.uniq_features = _gather(X, uniq32, uniq32.numel(), st)
        block.uniq_remap = remap
        partials = _group_mean(block.uniq_features, remap, t2, k2, B * k1, acc, code, st)
    else:
        block.gathered = _gather(X, flat, flat.numel(), st)
        partials = _group_mean(block.gathered, None, t2, k2, B * k1, acc, code, st)
    out = _group_mean(partials, None, t1, k1, B, X.dtype, code, st)
    return out, block


def baseline_backward(grad_out, block: MaterializedBlock, num_nodes: int, out: Optional[torch.Tensor] = None,
                      meter=None, *, zero: str = "full", validate: bool = True) -> torch.Tensor:
    """Adjoint of the materialised pipeline (baseline.py:157-194): the upstream gradient is
    expanded into a per-slot gradient block (the mirror image of the gathered features), then
    summed into the node-gradient buffer in ascending slot order per target -- bitwise the same
    result as the fused replay backward.  ``zero`` as in fused_2hop_backward ("sparse" re-zeroes
    only the rows the previous call on ``out`` wrote); ``validate=False`` skips the host-side
    index check (no host sync)."""
    dev = block.ids1.device
    g, _ = _grad_inputs(grad_out, dev)
    if block.ids1.shape[0] != g.shape[0]:
        raise ValueError("grad_out batch size does not match block")
    ids = block.ids2 if block.ids2 is not None else block.ids1
    if validate and int(ids.max()) >= num_nodes:
        raise ValueError("block index out of range")
    B, D = g.shape
    T = ids.numel()
    code = _DTYPE_CODE[g.dtype]
    d_gathered = torch.empty((T, -(-D // 8) * 8), dtype=_acc_dtype(g.dtype), device=dev)
    buf, mode = _grad_buffer(g, num_nodes, out, zero, ids.reshape(-1))
    _set_device(dev)
    st = _stream(dev)
    lib = _lib.load()
    s1 = _index_tensor(block.ids1, dev)
    if block.ids2 is not None:
        k1, k2 = int(block.ids1.shape[1]), int(block.ids2.shape[2])
        ws = _ws(_lib.FSA_OP_BWD2, B, k1, k2, num_nodes, dev, st, D, code)
        _lib.check(lib.fsa_baseline_2hop_bwd(g.data_ptr(), B, D, g.stride(0), code, s1.data_ptr(),
                                             _index_tensor(block.ids2, dev).data_ptr(), k1, k2, int(num_nodes),
                                             buf.data_ptr(), mode, d_gathered.data_ptr(), d_gathered.stride(0),
                                             ws.data_ptr(), ws.numel(), st), "fsa_baseline_2hop_bwd")
    else:
        k = int(block.ids1.shape[1])
        ws = _ws(_lib.FSA_OP_BWD1, B, k, 0, num_nodes, dev, st, D, code)
        _lib.check(lib.fsa_baseline_1hop_bwd(g.data_ptr(), B, D, g.stride(0), code, s1.data_ptr(),
                                             _index_tensor(block.take1, dev).data_ptr(), k, int(num_nodes),
                                             buf.data_ptr(), mode, d_gathered.data_ptr(), d_gathered.stride(0),
                                             ws.data_ptr(), ws.numel(), st), "fsa_baseline_1hop_bwd")
    _remember_rows(out, ids.reshape(-1))
    return buf
