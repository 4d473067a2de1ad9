"""B200-native FuseSampleAgg: fused uniform neighbour sampling + mean aggregation (1-/2-hop)
with deterministic saved-index replay backward, as hand-written sm_100a CUDA kernels behind a
C ABI (include/fsa_b200.h).  Drop-in for the reference operator API ``fsa.fused``."""

from .autograd import (
    FusedSampleAgg1Hop,
    FusedSampleAgg2Hop,
    fused_sample_agg_1hop,
    fused_sample_agg_2hop,
)
from .baseline import MaterializedBlock, baseline_1hop_forward, baseline_backward, baseline_forward
from .fused import (
    SampledIndices1,
    SampledIndices2,
    device_errors,
    fused_1hop_backward,
    fused_1hop_forward,
    fused_2hop_backward,
    fused_2hop_forward,
    sample_1hop,
    sample_2hop,
    sample_neighbors_reservoir,
)
from .graph import CsrGraph, GraphFormatError, SeedBatch, load_csr_cache, save_csr_cache
from .rng import RngStream, derive_stream, splitmix64, step_seed, xorshift64

__all__ = [
    "MaterializedBlock",
    "baseline_1hop_forward",
    "baseline_forward",
    "baseline_backward",
    "CsrGraph",
    "SeedBatch",
    "GraphFormatError",
    "save_csr_cache",
    "load_csr_cache",
    "SampledIndices1",
    "SampledIndices2",
    "fused_1hop_forward",
    "fused_1hop_backward",
    "fused_2hop_forward",
    "fused_2hop_backward",
    "sample_1hop",
    "sample_2hop",
    "sample_neighbors_reservoir",
    "device_errors",
    "FusedSampleAgg1Hop",
    "FusedSampleAgg2Hop",
    "fused_sample_agg_1hop",
    "fused_sample_agg_2hop",
    "RngStream",
    "derive_stream",
    "splitmix64",
    "xorshift64",
    "step_seed",
]
