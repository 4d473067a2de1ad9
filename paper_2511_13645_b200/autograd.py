"""``torch.autograd.Function`` wrappers: forward = fused sample + mean, backward = replay.

The feature matrix X is the differentiable input; the sampled ids are non-differentiable
outputs.  With ``save_indices=False`` the backward returns zeros, as the reference does when no
indices were saved (fused.py:206-207, 240-241).
"""

from __future__ import annotations

import torch

from .fused import (
    SampledIndices1,
    SampledIndices2,
    fused_1hop_backward,
    fused_1hop_forward,
    fused_2hop_backward,
    fused_2hop_forward,
)

__all__ = ["FusedSampleAgg1Hop", "FusedSampleAgg2Hop", "fused_sample_agg_1hop", "fused_sample_agg_2hop"]


class FusedSampleAgg1Hop(torch.autograd.Function):
    @staticmethod
    def forward(ctx, X, graph, seeds, k, base_seed, save_indices=True, root_offset=0):
        out, idx = fused_1hop_forward(graph, X, seeds, k, base_seed, save_indices,
                                      root_offset=root_offset, validate=False)
        ctx.num_nodes = X.shape[0]
        if idx is None:
            ctx.save_for_backward()
            ctx.has_idx = False
            empty = torch.empty(0, dtype=torch.int32, device=X.device)
            ctx.mark_non_differentiable(empty, empty)
            return out, empty, empty
        ctx.save_for_backward(idx.samples, idx.takes)
        ctx.has_idx = True
        ctx.mark_non_differentiable(idx.samples, idx.takes)
        return out, idx.samples, idx.takes

    @staticmethod
    def backward(ctx, grad_out, _g_samples=None, _g_takes=None):
        if not ctx.has_idx:
            gx = torch.zeros((ctx.num_nodes, grad_out.shape[1]), dtype=grad_out.dtype, device=grad_out.device)
        else:
            samples, takes = ctx.saved_tensors
            gx = fused_1hop_backward(grad_out.contiguous(), SampledIndices1(samples, takes),
                                     ctx.num_nodes, validate=False)
        return gx, None, None, None, None, None, None


class FusedSampleAgg2Hop(torch.autograd.Function):
    @staticmethod
    def forward(ctx, X, graph, roots, k1, k2, base_seed, save_indices=True, root_offset=0):
        out, idx = fused_2hop_forward(graph, X, roots, k1, k2, base_seed, save_indices,
                                      root_offset=root_offset, validate=False)
        ctx.num_nodes = X.shape[0]
        if idx is None:
            ctx.has_idx = False
            empty = torch.empty(0, dtype=torch.int32, device=X.device)
            ctx.mark_non_differentiable(empty)
            return out, empty, empty
        ctx.save_for_backward(idx.s1, idx.s2)
        ctx.has_idx = True
        ctx.mark_non_differentiable(idx.s1, idx.s2)
        return out, idx.s1, idx.s2

    @staticmethod
    def backward(ctx, grad_out, _g_s1=None, _g_s2=None):
        if not ctx.has_idx:
            gx = torch.zeros((ctx.num_nodes, grad_out.shape[1]), dtype=grad_out.dtype, device=grad_out.device)
        else:
            s1, s2 = ctx.saved_tensors
            gx = fused_2hop_backward(grad_out.contiguous(), SampledIndices2(s1, s2), ctx.num_nodes,
                                     validate=False)
        return gx, None, None, None, None, None, None, None


def fused_sample_agg_1hop(X, graph, seeds, k, base_seed, save_indices=True, root_offset=0):
    """Differentiable 1-hop op: returns ``(out, SampledIndices1 | None)``."""
    out, samples, takes = FusedSampleAgg1Hop.apply(X, graph, seeds, k, base_seed, save_indices, root_offset)
    return out, (SampledIndices1(samples, takes) if save_indices else None)


def fused_sample_agg_2hop(X, graph, roots, k1, k2, base_seed, save_indices=True, root_offset=0):
    """Differentiable 2-hop op: returns ``(out, SampledIndices2 | None)``."""
    out, s1, s2 = FusedSampleAgg2Hop.apply(X, graph, roots, k1, k2, base_seed, save_indices, root_offset)
    return out, (SampledIndices2(s1, s2) if save_indices else None)
