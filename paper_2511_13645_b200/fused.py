"""Fused neighbour sampling + mean aggregation with exact replay backward — B200 operator API.

Drop-in mirror of the reference operator layer ``fsa.fused`` (pkg/src/fsa/fused.py:40-299):
same function names, argument meaning, return types and ``ValueError`` messages.  Every call
runs the hand-written sm_100a kernels of ``libfsa_b200.so`` through the C ABI
(include/fsa_b200.h); there is no CPU path.

Inputs may be torch CUDA tensors (the fast path: nothing leaves HBM) or numpy arrays (host
mode: inputs are uploaded, results come back as numpy arrays, like the reference).
Extensions over the reference, all optional keyword arguments:
  * ``root_offset``  global batch position of ``seeds[0]`` (seed-sharded data parallelism;
                     0 reproduces the reference bit for bit),
  * ``validate``     host-side range checks before launch (one device sync); False skips them
                     (the device still flags bad inputs, see :func:`device_errors`),
  * bf16 / fp16 features (fp32 accumulation, one rounding at the end),
  * ``zero`` for the backward: "full" (reference semantics, zero-fill the whole buffer),
                     or "sparse": re-zero only the rows written by this function's previous
                     call on the same buffer when the buffer is unchanged since (checked with
                     the tensor's version counter), else a full fill.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref
from dataclasses import dataclass
from typing import Optional, Tuple, Union

import numpy as np
import torch

from . import _lib
from .graph import CsrGraph, SeedBatch, as_device_graph, as_seed_tensor
from .rng import MASK64, RngStream

__all__ = [
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
    "FEATURE_DTYPES",
]

FEATURE_DTYPES = (torch.float32, torch.float64, torch.bfloat16, torch.float16)
_DTYPE_CODE = {torch.float32: _lib.FSA_F32, torch.float64: _lib.FSA_F64,
               torch.bfloat16: _lib.FSA_BF16, torch.float16: _lib.FSA_F16}


# ---------------------------------------------------------------------------------------------
# replay index containers (fused.py:40-77)
# ---------------------------------------------------------------------------------------------
@dataclass
class SampledIndices1:
    """Per-seed sampled neighbour ids (−1 padded) and take counts."""

    samples: torch.Tensor  # int32 (B, k)
    takes: torch.Tensor    # int32 (B,)

    @property
    def fanout(self) -> int:
        return int(self.samples.shape[1])

    def valid_pairs(self) -> int:
        return int(self.takes.sum())


@dataclass
class SampledIndices2:
    """Two-hop ids: s1 (B, k1), s2 (B, k1, k2), −1 padded; counts are recomputed from −1."""

    s1: torch.Tensor
    s2: torch.Tensor

    @property
    def fanouts(self) -> Tuple[int, int]:
        return int(self.s1.shape[1]), int(self.s2.shape[2])

    def take1(self):
        return (self.s1 >= 0).sum(1).to(torch.int32) if torch.is_tensor(self.s1) else \
            (self.s1 >= 0).sum(axis=1).astype(np.int32)

    def take2(self):
        return (self.s2 >= 0).sum(2).to(torch.int32) if torch.is_tensor(self.s2) else \
            (self.s2 >= 0).sum(axis=2).astype(np.int32)

    def valid_pairs(self) -> int:
        return int((self.s1 >= 0).sum() + (self.s2 >= 0).sum())


# ---------------------------------------------------------------------------------------------
# workspace / device plumbing
# ---------------------------------------------------------------------------------------------
_tls = threading.local()


def _ws(op: int, B: int, k1: int, k2: int, N: int, device: torch.device, stream: int, D: int = 0,
        dtype_code: int = 0) -> torch.Tensor:
    """Cached, zero-initialised workspace per (device, stream, op kind)."""
    need = _lib.load().fsa_ws_bytes(op, B, k1, k2, D, dtype_code, N)
    if need == 0:
        raise ValueError("invalid workspace request")
    cache = getattr(_tls, "ws", None)
    if cache is None:
        cache = _tls.ws = {}
    # backward workspaces hold per-node counters that stay zero between calls: bound to one N
    key = (device.index, stream, op, N if op in (_lib.FSA_OP_BWD1, _lib.FSA_OP_BWD2) else 0)
    buf = cache.get(key)
    if buf is None or buf.numel() < need:
        buf = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=device)
        cache[key] = buf
    return buf


# First-hop path of the 2-hop forward (fsa_tune 6): one warp per root (k_hop1) wins while first-hop
# chains are short; the tile sampler wins on dense graphs (measured: products mean degree 50 and
# arxiv 14 -> warp per root, 3 % / 5 % faster; Reddit 492 -> tiles, 7 % faster).  Both are
# bitwise identical; FSA_HOP1 (1 / 2) pins the path for experiments.
HOP1_TILE_MEAN_DEGREE = 128.0
_hop1_set = [None]


def _select_hop1(g) -> None:
    if os.environ.get("FSA_HOP1"):
        return
    mode = 2 if g.num_edges > HOP1_TILE_MEAN_DEGREE * max(1, g.num_nodes) else 1
    if _hop1_set[0] != mode:
        _lib.check(_lib.load().fsa_tune(6, mode), "fsa_tune")
        _hop1_set[0] = mode


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _set_device(device: torch.device) -> None:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if getattr(_tls, "dev", None) != idx:
        _lib.check(_lib.load().fsa_set_device(idx), "fsa_set_device")
        _tls.dev = idx


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def device_errors(device: Union[str, torch.device, None] = None, clear: bool = True) -> int:
    """OR of the device error bits raised by the last forward/backward on this stream
    (FSA_DEVERR_* in include/fsa_b200.h).  Synchronises the stream."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    st = _stream(dev)
    flags = 0
    cache = getattr(_tls, "ws", {}) or {}
    for (idx, s, _op, _n), buf in cache.items():
        if idx == dev.index and s == st:
            f = C.c_int(0)
            _lib.check(_lib.load().fsa_read_error(buf.data_ptr(), int(clear), C.byref(f), st), "fsa_read_error")
            flags |= f.value
    return flags


# ---------------------------------------------------------------------------------------------
# validation (messages match fused.py:80-96, 121, 162, 204-214, 244-246, 282-293)
# ---------------------------------------------------------------------------------------------
def _check_features(graph, X):
    if X.ndim != 2 or X.shape[0] != graph.num_nodes:
        raise ValueError(f"features must be ({graph.num_nodes}, D), got {tuple(X.shape)}")
    if X.dtype not in FEATURE_DTYPES:
        raise ValueError(f"features must be float32, float64, bfloat16 or float16, got {X.dtype}")
    if X.stride(1) != 1 or X.stride(0) < X.shape[1]:
        raise ValueError("features must be C-contiguous (row-major)")


def _to_device_features(X, device) -> Tuple[torch.Tensor, bool]:
    if torch.is_tensor(X):
        return X, False
    arr = np.asarray(X)
    if arr.dtype not in (np.float32, np.float64):
        raise ValueError(f"features must be float32 or float64, got {arr.dtype}")
    if not arr.flags.c_contiguous:
        raise ValueError("features must be C-contiguous")
    return torch.from_numpy(arr).to(device), True


def _pick_device(graph, X) -> torch.device:
    if torch.is_tensor(X) and X.is_cuda:
        return X.device
    if isinstance(graph, CsrGraph):
        return graph.device
    if not torch.cuda.is_available():
        raise RuntimeError("FuseSampleAgg needs a CUDA device (there is no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _check_seed_range(seeds: torch.Tensor, n: int) -> None:
    lo, hi = torch.aminmax(seeds)
    if int(lo) < 0 or int(hi) >= n:
        raise ValueError(f"seed out of range for graph with {n} nodes")


def _seed_u64(base_seed: int) -> int:
    return int(base_seed) & MASK64


def _host(t: torch.Tensor):
    return t.cpu().numpy()


# ---------------------------------------------------------------------------------------------
# forward
# ---------------------------------------------------------------------------------------------
def fused_1hop_forward(graph, X, seeds, k: int, base_seed: int, save_indices: bool = True,
                       meter=None, *, root_offset: int = 0, validate: bool = True,
                       out: Optional[torch.Tensor] = None):
    """Sample up to ``k`` neighbours per seed and return their feature means (fused.py:103-143).

    Returns ``(out[B, D], SampledIndices1 | None)``.  Degree <= k takes the whole row in CSR
    order; an isolated seed gives a zero row with take 0.  ``meter`` is accepted for signature
    compatibility and ignored (device memory is tracked by torch's allocator).
    """
    device = _pick_device(graph, X)
    Xd, host_mode = _to_device_features(X, device)
    g = as_device_graph(graph, device)
    _check_features(g, Xd)
    sd = as_seed_tensor(seeds, device)
    if validate:
        _check_seed_range(sd, g.num_nodes)
    if k < 1:
        raise ValueError("fanout k must be >= 1")
    B, D = int(sd.numel()), int(Xd.shape[1])
    if out is None:
        out = torch.empty((B, D), dtype=Xd.dtype, device=device)
    samples = takes = None
    if save_indices:
        samples = torch.empty((B, k), dtype=torch.int32, device=device)
        takes = torch.empty((B,), dtype=torch.int32, device=device)
    _set_device(device)
    st = _stream(device)
    ws = _ws(_lib.FSA_OP_FWD1, B, k, 0, 0, device, st)
    lib = _lib.load()
    _lib.check(lib.fsa_fused_1hop_fwd(
        g.rowptr.data_ptr(), g.col.data_ptr(), g.num_nodes, Xd.data_ptr(), D, Xd.stride(0),
        _DTYPE_CODE[Xd.dtype], sd.data_ptr(), B, int(root_offset), int(k), _seed_u64(base_seed),
        int(bool(save_indices)), _ptr(samples), _ptr(takes), out.data_ptr(), out.stride(0),
        ws.data_ptr(), ws.numel(), st), "fsa_fused_1hop_fwd")
    idx = SampledIndices1(samples, takes) if save_indices else None
    if host_mode:
        return _host(out), (SampledIndices1(_host(samples), _host(takes)) if idx else None)
    return out, idx


def fused_2hop_forward(graph, X, roots, k1: int, k2: int, base_seed: int, save_indices: bool = True,
                       meter=None, *, root_offset: int = 0, validate: bool = True,
                       out: Optional[torch.Tensor] = None):
    """Nested two-hop sampled mean (fused.py:146-188): per root, the mean over first-hop samples
    of the mean over their second-hop samples; −1 slots are skipped and every mean divides by
    the realised count.  Returns ``(out[B, D], SampledIndices2 | None)``."""
    device = _pick_device(graph, X)
    Xd, host_mode = _to_device_features(X, device)
    g = as_device_graph(graph, device)
    _check_features(g, Xd)
    sd = as_seed_tensor(roots, device)
    if validate:
        _check_seed_range(sd, g.num_nodes)
    if k1 < 1 or k2 < 1:
        raise ValueError("fanouts must be >= 1")
    B, D = int(sd.numel()), int(Xd.shape[1])
    if out is None:
        out = torch.empty((B, D), dtype=Xd.dtype, device=device)
    s1 = s2 = t1 = t2 = None
    if save_indices:
        s1 = torch.empty((B, k1), dtype=torch.int32, device=device)
        s2 = torch.empty((B, k1, k2), dtype=torch.int32, device=device)
        t1 = torch.empty((B,), dtype=torch.int32, device=device)
        t2 = torch.empty((B, k1), dtype=torch.int32, device=device)
    _set_device(device)
    st = _stream(device)
    ws = _ws(_lib.FSA_OP_FWD2, B, k1, k2, 0, device, st)
    lib = _lib.load()
    _select_hop1(g)
    _lib.check(lib.fsa_fused_2hop_fwd(
        g.rowptr.data_ptr(), g.col.data_ptr(), g.num_nodes, Xd.data_ptr(), D, Xd.stride(0),
        _DTYPE_CODE[Xd.dtype], sd.data_ptr(), B, int(root_offset), int(k1), int(k2),
        _seed_u64(base_seed), int(bool(save_indices)), _ptr(s1), _ptr(s2), _ptr(t1), _ptr(t2),
        out.data_ptr(), out.stride(0), ws.data_ptr(), ws.numel(), st), "fsa_fused_2hop_fwd")
    idx = SampledIndices2(s1, s2) if save_indices else None
    if host_mode:
        return _host(out), (SampledIndices2(_host(s1), _host(s2)) if idx else None)
    return out, idx


def sample_1hop(graph, seeds, k: int, base_seed: int, *, root_offset: int = 0,
                device: Union[str, torch.device, None] = None, validate: bool = True):
    """Sampling only (kernels.py:87-97): returns ``(samples int32[B,k], takes int32[B])``."""
    dev = torch.device(device) if device is not None else _pick_device(graph, None)
    g = as_device_graph(graph, dev)
    sd = as_seed_tensor(seeds, dev)
    if validate:
        _check_seed_range(sd, g.num_nodes)
    if k < 1:
        raise ValueError("fanout k must be >= 1")
    B = int(sd.numel())
    samples = torch.empty((B, k), dtype=torch.int32, device=dev)
    takes = torch.empty((B,), dtype=torch.int32, device=dev)
    _set_device(dev)
    st = _stream(dev)
    ws = _ws(_lib.FSA_OP_FWD1, B, k, 0, 0, dev, st)
    _lib.check(_lib.load().fsa_fused_1hop_fwd(
        g.rowptr.data_ptr(), g.col.data_ptr(), g.num_nodes, None, 0, 0, _lib.FSA_F32,
        sd.data_ptr(), B, int(root_offset), int(k), _seed_u64(base_seed), 1,
        samples.data_ptr(), takes.data_ptr(), None, 0, ws.data_ptr(), ws.numel(), st), "sample_1hop")
    return samples, takes


def sample_2hop(graph, seeds, k1: int, k2: int, base_seed: int, *, root_offset: int = 0,
                device: Union[str, torch.device, None] = None, validate: bool = True):
    """Sampling only (kernels.py:99-120): returns ``(s1, s2, take1, take2)``."""
    dev = torch.device(device) if device is not None else _pick_device(graph, None)
    g = as_device_graph(graph, dev)
    sd = as_seed_tensor(seeds, dev)
    if validate:
        _check_seed_range(sd, g.num_nodes)
    if k1 < 1 or k2 < 1:
        raise ValueError("fanouts must be >= 1")
    B = int(sd.numel())
    s1 = torch.empty((B, k1), dtype=torch.int32, device=dev)
    s2 = torch.empty((B, k1, k2), dtype=torch.int32, device=dev)
    t1 = torch.empty((B,), dtype=torch.int32, device=dev)
    t2 = torch.empty((B, k1), dtype=torch.int32, device=dev)
    _set_device(dev)
    st = _stream(dev)
    ws = _ws(_lib.FSA_OP_FWD2, B, k1, k2, 0, dev, st)
    _select_hop1(g)
    _lib.check(_lib.load().fsa_fused_2hop_fwd(
        g.rowptr.data_ptr(), g.col.data_ptr(), g.num_nodes, None, 0, 0, _lib.FSA_F32,
        sd.data_ptr(), B, int(root_offset), int(k1), int(k2), _seed_u64(base_seed), 1,
        s1.data_ptr(), s2.data_ptr(), t1.data_ptr(), t2.data_ptr(), None, 0,
        ws.data_ptr(), ws.numel(), st), "sample_2hop")
    return s1, s2, t1, t2


# ---------------------------------------------------------------------------------------------
# backward
# ---------------------------------------------------------------------------------------------
# id(buffer) -> (weakref to the buffer, its version after our write, data_ptr, shape, a private
# copy of the ids whose rows we wrote).  The entry dies with the buffer, every backward that
# writes the buffer (whatever its zero mode) replaces it, and a torch-side modification of the
# buffer (version change) or a different tensor object forces a full fill.
_SPARSE_STATE: dict = {}


def _check_grad(grad_out):
    if grad_out.ndim != 2:
        raise ValueError("grad_out must be 2-D (B, D)")
    if grad_out.dtype not in FEATURE_DTYPES:
        raise ValueError("grad_out must be float32 or float64")


def _grad_inputs(grad_out, device):
    host_mode = not torch.is_tensor(grad_out)
    if host_mode:
        arr = np.asarray(grad_out)
        if arr.ndim != 2:
            raise ValueError("grad_out must be 2-D (B, D)")
        if arr.dtype not in (np.float32, np.float64):
            raise ValueError("grad_out must be float32 or float64")
        grad_out = torch.from_numpy(np.ascontiguousarray(arr)).to(device)
    _check_grad(grad_out)
    if grad_out.stride(1) != 1:
        grad_out = grad_out.contiguous()
    return grad_out, host_mode


def _index_tensor(a, device):
    if torch.is_tensor(a):
        return a.to(device=device, dtype=torch.int32).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32)).to(device)


def _grad_buffer(grad_out, num_nodes, out, zero, ids_flat):
    """Returns (buffer, zero_mode) honouring fused.py:290-299 semantics."""
    if out is None:
        return torch.zeros((num_nodes, grad_out.shape[1]), dtype=grad_out.dtype,
                           device=grad_out.device), 0
    if tuple(out.shape) != (num_nodes, grad_out.shape[1]) or out.dtype != grad_out.dtype \
            or not out.is_contiguous() or out.device != grad_out.device:
        raise ValueError("gradient buffer has wrong shape or dtype")
    if zero == "sparse":
        prev = _SPARSE_STATE.get(id(out))
        if prev is not None and prev[0]() is out and prev[1] == out._version and prev[2] == out.data_ptr() \
                and prev[3] == tuple(out.shape):
            rows = prev[4]
            if rows.numel():
                _lib.check(_lib.load().fsa_zero_rows(out.data_ptr(), out.shape[1], _DTYPE_CODE[out.dtype],
                                                     rows.data_ptr(), rows.numel(), _stream(out.device)),
                           "fsa_zero_rows")
            return out, 0
        return out, 1
    if zero != "full":
        raise ValueError("zero must be 'full' or 'sparse'")
    return out, 1


def _remember_rows(out, ids_flat):
    """After a backward wrote ``out``: its nonzero rows are exactly the rows of ``ids_flat``."""
    if out is None or not torch.is_tensor(out):
        return
    key = id(out)
    rows = ids_flat.clone() if ids_flat is not None else torch.empty(0, dtype=torch.int32, device=out.device)
    ref = weakref.ref(out, lambda _r, k=key: _SPARSE_STATE.pop(k, None))
    _SPARSE_STATE[key] = (ref, out._version, out.data_ptr(), tuple(out.shape), rows)


def fused_1hop_backward(grad_out, indices: Optional[SampledIndices1], num_nodes: int,
                        out: Optional[torch.Tensor] = None, meter=None, *, validate: bool = True,
                        zero: str = "full"):
    """Replay saved indices: grad[v] += grad_out[i] / max(1, take_i) (fused.py:191-222).

    Accumulation per target row follows ascending (seed, slot) order, exactly as the
    reference, so results are bitwise reproducible.  ``indices=None`` yields zeros."""
    device = grad_out.device if torch.is_tensor(grad_out) else torch.device("cuda", torch.cuda.current_device())
    g, host_mode = _grad_inputs(grad_out, device)
    if indices is None:
        buf, mode = _grad_buffer(g, num_nodes, out, "full", None)
        if mode == 1:
            buf.zero_()
        _remember_rows(None if host_mode else out, None)
        return _host(buf) if host_mode else buf
    samples = _index_tensor(indices.samples, device)
    takes = _index_tensor(indices.takes, device)
    if samples.shape[0] != g.shape[0]:
        raise ValueError("grad_out batch size does not match saved indices")
    if validate:
        if int(takes.min()) < 0:
            raise ValueError("negative take count")
        if int(samples.max()) >= num_nodes:
            raise ValueError("saved index out of range")
    B, k = int(samples.shape[0]), int(samples.shape[1])
    ids_flat = samples.reshape(-1)
    buf, mode = _grad_buffer(g, num_nodes, None if host_mode else out, zero, ids_flat)
    _set_device(device)
    st = _stream(device)
    ws = _ws(_lib.FSA_OP_BWD1, B, k, 0, num_nodes, device, st, g.shape[1], _DTYPE_CODE[g.dtype])
    _lib.check(_lib.load().fsa_fused_1hop_bwd(
        g.data_ptr(), B, g.shape[1], g.stride(0), _DTYPE_CODE[g.dtype], samples.data_ptr(),
        takes.data_ptr(), k, int(num_nodes), buf.data_ptr(), mode, None, None, None,
        ws.data_ptr(), ws.numel(), st), "fsa_fused_1hop_bwd")
    _remember_rows(None if host_mode else out, ids_flat)
    if host_mode:
        res = _host(buf)
        if out is not None:
            out[...] = res
            return out
        return res
    return buf


def fused_2hop_backward(grad_out, indices: Optional[SampledIndices2], num_nodes: int,
                        out: Optional[torch.Tensor] = None, meter=None, *, validate: bool = True,
                        zero: str = "full", touched: Optional[torch.Tensor] = None,
                        n_touched: Optional[torch.Tensor] = None,
                        grad_rows: Optional[torch.Tensor] = None):
    """Two-hop replay: grad[w] += grad_out[r] / (k1_eff(r) * k2_eff(r, j)) (fused.py:225-255).

    Effective counts come from the −1 pattern of the saved indices.  Optional sparse outputs
    (``touched`` int32[B*k1*k2], ``n_touched`` int32[1], ``grad_rows`` [B*k1*k2, D]) give the
    gradient in COO form; with ``out=False`` no dense buffer is produced at all."""
    device = grad_out.device if torch.is_tensor(grad_out) else torch.device("cuda", torch.cuda.current_device())
    g, host_mode = _grad_inputs(grad_out, device)
    dense = out is not False
    if indices is None:
        if not dense:
            return None
        buf, mode = _grad_buffer(g, num_nodes, out, "full", None)
        if mode == 1:
            buf.zero_()
        _remember_rows(None if host_mode else out, None)
        return _host(buf) if host_mode else buf
    s1 = _index_tensor(indices.s1, device)
    s2 = _index_tensor(indices.s2, device)
    if s1.shape[0] != g.shape[0]:
        raise ValueError("grad_out batch size does not match saved indices")
    if validate and int(s2.max()) >= num_nodes:
        raise ValueError("saved index out of range")
    B, k1, k2 = int(s1.shape[0]), int(s1.shape[1]), int(s2.shape[2])
    ids_flat = s2.reshape(-1)
    if dense:
        buf, mode = _grad_buffer(g, num_nodes, None if host_mode else out, zero, ids_flat)
    else:
        buf, mode = None, 0
    _set_device(device)
    st = _stream(device)
    ws = _ws(_lib.FSA_OP_BWD2, B, k1, k2, num_nodes, device, st, g.shape[1], _DTYPE_CODE[g.dtype])
    _lib.check(_lib.load().fsa_fused_2hop_bwd(
        g.data_ptr(), B, g.shape[1], g.stride(0), _DTYPE_CODE[g.dtype], s1.data_ptr(), s2.data_ptr(),
        k1, k2, int(num_nodes), _ptr(buf), mode, _ptr(touched), _ptr(n_touched), _ptr(grad_rows),
        ws.data_ptr(), ws.numel(), st), "fsa_fused_2hop_bwd")
    if dense:
        _remember_rows(None if host_mode else out, ids_flat)
    if host_mode and buf is not None:
        res = _host(buf)
        if out is not None and out is not False:
            out[...] = res
            return out
        return res
    return buf


def sample_neighbors_reservoir(graph, u: int, k: int, stream: RngStream):
    """Readable single-node Algorithm R (fused.py:258-279), evaluated on the host with the
    stream contract of :mod:`.rng`; the GPU samplers reproduce it bit for bit.  Advances
    ``stream`` like the reference."""
    n = int(graph.num_nodes)
    if u < 0 or u >= n:
        raise ValueError(f"node {u} out of range")
    if k < 1:
        raise ValueError("fanout k must be >= 1")
    if isinstance(graph, CsrGraph):
        lo, hi = int(graph.rowptr[u]), int(graph.rowptr[u + 1])
        neigh = graph.col[lo:hi].cpu().numpy()
    else:
        neigh = np.asarray(graph.col[graph.rowptr[u]:graph.rowptr[u + 1]])
    deg = len(neigh)
    if deg <= k:
        return neigh.copy(), deg
    res = neigh[:k].copy()
    for i in range(k, deg):
        j = stream.uniform_index(i + 1)
        if j < k:
            res[j] = neigh[i]
    return res, k
