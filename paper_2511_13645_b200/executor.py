"""Repeated-step executor for the fused 2-hop operator: static buffers, CUDA-graph replay.

The reference's training step calls ``fused_2hop_forward`` then ``fused_2hop_backward`` into
a persistent gradient buffer that it zero-fills every step (train.py:185-251, fused.py:290-296).
This executor does the same work per step with B200-side plumbing instead of per-call host
work:

* every buffer (seeds, base seed, out, s1/s2, take arrays, gradient, workspaces) is allocated
  once, so the whole step is captured as CUDA graphs and replayed with one launch;
* the base seed is read from device memory by the kernels (``fsa_fused_2hop_fwd_dseed``), so a
  replay samples a fresh neighbourhood per step exactly like the eager call;
* the persistent N x D gradient is kept equal to the reference's "zero-filled then scattered"
  buffer by re-zeroing only the rows written in the previous step, on a side stream that runs
  concurrently with the (latency-bound) forward; two graphs alternate s2 buffers so the side
  stream reads the previous step's ids while the forward writes the current ones;
* the replay backward's PLAN phase (per-node counts, segments: it reads only the sampled ids)
  and its row writes run as one branch beside the forward's feature gather (they never read
  its output); the term table (TERMS) is built on the re-zeroing stream.

Results are bitwise identical to the eager API (tests/test_gpu_executor.py).
"""

from __future__ import annotations

import os

from typing import Optional

import torch

from . import _lib
from .fused import _DTYPE_CODE, _select_hop1, _set_device, SampledIndices2
from .graph import CsrGraph

__all__ = ["Fused2HopStep"]


class Fused2HopStep:
    """One rank's fused 2-hop (k1, k2) forward + replay backward over batches of ``batch``
    seeds at global positions ``root_offset + [0, batch)``."""

    def __init__(self, graph: CsrGraph, X: torch.Tensor, batch: int, k1: int, k2: int, *,
                 root_offset: int = 0, use_graph: bool = True, overlap_zero: bool = True,
                 pipeline: bool = False):
        if X.ndim != 2 or X.shape[0] != graph.num_nodes or X.stride(1) != 1:
            raise ValueError(f"features must be ({graph.num_nodes}, D) row-major")
        if X.dtype not in _DTYPE_CODE:
            raise ValueError(f"unsupported feature dtype {X.dtype}")
        if k1 < 1 or k2 < 1 or batch < 1:
            raise ValueError("fanouts and batch must be >= 1")
        self.g, self.X = graph, X
        self.B, self.k1, self.k2 = int(batch), int(k1), int(k2)
        self.N, self.D = graph.num_nodes, int(X.shape[1])
        self.root_offset = int(root_offset)
        self.device = X.device
        self.dtype = X.dtype
        self.code = _DTYPE_CODE[X.dtype]
        self.use_graph, self.overlap_zero, self.pipeline = use_graph, overlap_zero, pipeline
        dev = self.device
        lib = _lib.load()
        _set_device(dev)
        B, k1, k2, D, N = self.B, self.k1, self.k2, self.D, self.N
        # per-parity inputs / output: step i+1's host->device copies overlap step i's compute
        self.seeds_p = [torch.zeros(B, dtype=torch.int64, device=dev) for _ in range(2)]
        self.base_seed_p = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(2)]
        self.grad_out_p = [torch.zeros((B, D), dtype=self.dtype, device=dev) for _ in range(2)]
        self.out_p = [torch.empty((B, D), dtype=self.dtype, device=dev) for _ in range(2)]
        self.copy = torch.cuda.Stream(device=dev)      # host -> device inputs
        self.copy_out = torch.cuda.Stream(device=dev)  # device -> host outputs
        self.done = [torch.cuda.Event() for _ in range(2)]
        self.done_used = [False, False]
        self.staged = False
        # D2H of a parity's out buffer finished: the next step of that parity (which rewrites
        # out_p[p]) waits for it
        self.out_copied = [torch.cuda.Event() for _ in range(2)]
        self.out_copied_used = [False, False]
        self.s1 = torch.empty((B, k1), dtype=torch.int32, device=dev)
        # pipelined: step i+1's forward runs while step i's backward still reads its s1
        self.s1_p = [self.s1, torch.empty_like(self.s1) if pipeline else self.s1]
        self.s2 = [torch.full((B, k1, k2), -1, dtype=torch.int32, device=dev) for _ in range(2)]
        self.t1 = torch.empty(B, dtype=torch.int32, device=dev)
        self.t2 = torch.empty((B, k1), dtype=torch.int32, device=dev)
        # persistent feature gradient, rows padded to whole 64-byte bursts: the row writers and the
        # re-zero store full bursts (no partial-burst read-modify-write); ``grad`` is the [N, D] view
        e = torch.empty((), dtype=self.dtype).element_size()
        self.gx_stride = -(-D * e // 64) * 64 // e
        self.grad_full = torch.zeros((N, self.gx_stride), dtype=self.dtype, device=dev)
        self.grad = self.grad_full[:, :D]
        self.ws_f = torch.zeros(lib.fsa_ws_bytes(_lib.FSA_OP_FWD2, B, k1, k2, 0, 0, 0), dtype=torch.uint8, device=dev)
        self.ws_b = torch.zeros(lib.fsa_ws_bytes(_lib.FSA_OP_BWD2, B, k1, k2, D, self.code, N), dtype=torch.uint8, device=dev)
        self.side = torch.cuda.Stream(device=dev)
        # the backward branch (PLAN -> ROWS) shares the SMs with the gather; it is the longer branch
        self.plan = torch.cuda.Stream(device=dev, priority=int(os.environ.get("FSA_PLAN_PRIO", "0")))
        self.parity = 0
        self.graphs = [None, None]
        self.steps_run = 0
        # pipelined steps: the forward (SAMPLE + GATHER) of step i on the caller's stream, its
        # backward on self.bwd once that forward is done, so step i+1's forward overlaps it
        self.bwd = torch.cuda.Stream(device=dev)
        self.fwd_done = [torch.cuda.Event() for _ in range(2)]
        self.graphs_b = [None, None]

    # -- raw launch sequence of one step (eager or under capture) ----------------------------
    def _launch(self, parity: int, head=None, tail=None) -> None:
        """main:   fwd SAMPLE ──┬── fwd GATHER ─────────────────────┬── (step end)
           plan:                ├── bwd PLAN ──────┬── bwd ROWS ──┘  (PLAN needs only s1/s2)
           zero:   re-zero prev rows ── bwd TERMS ─┘                 (grad_out + s1/s2)

        With ``head`` (a callable run on the main stream after the gather, which writes this
        parity's grad_out buffer from the forward output: a training step's head), TERMS runs on
        the main stream after it instead; ``tail`` runs on the main stream beside the row writes
        (a training step's optimizer update)."""
        lib = _lib.load()
        main = torch.cuda.current_stream(self.device)
        cur, prev = self.s2[parity], self.s2[1 - parity]
        seeds, base_seed = self.seeds_p[parity], self.base_seed_p[parity]
        grad_out, out = self.grad_out_p[parity], self.out_p[parity]
        zs = self.side if self.overlap_zero else main
        if self.overlap_zero:
            zs.wait_stream(main)
        with torch.cuda.stream(zs):
            _lib.check(lib.fsa_zero_rows_strided(self.grad_full.data_ptr(), self.D, self.gx_stride, self.gx_stride,
                                                 self.code, prev.data_ptr(), prev.numel(), zs.cuda_stream),
                       "fsa_zero_rows_strided")
        st = main.cuda_stream
        fwd_args = (self.g.rowptr.data_ptr(), self.g.col.data_ptr(), self.N, self.X.data_ptr(), self.D,
                    self.X.stride(0), self.code, seeds.data_ptr(), self.B, self.root_offset, self.k1, self.k2,
                    0, base_seed.data_ptr(), 1, self.s1_p[parity].data_ptr(), cur.data_ptr(), self.t1.data_ptr(),
                    self.t2.data_ptr(), out.data_ptr(), out.stride(0), self.ws_f.data_ptr(),
                    self.ws_f.numel(), st)
        bwd_args = (grad_out.data_ptr(), self.B, self.D, grad_out.stride(0), self.code,
                    self.s1_p[parity].data_ptr(), cur.data_ptr(), self.k1, self.k2, self.N, self.grad_full.data_ptr(),
                    self.gx_stride, self.gx_stride, 0, self.ws_b.data_ptr(), self.ws_b.numel())
        _select_hop1(self.g)  # baked into the captured graph
        _lib.check(lib.fsa_fused_2hop_fwd_phase(*fwd_args, _lib.FSA_FWD_SAMPLE), "fwd SAMPLE")
        if not self.overlap_zero:
            _lib.check(lib.fsa_fused_2hop_bwd_phase_rows(*bwd_args, st, _lib.FSA_BWD_PLAN), "bwd PLAN")
            _lib.check(lib.fsa_fused_2hop_fwd_phase(*fwd_args, _lib.FSA_FWD_GATHER), "fwd GATHER")
            if head is not None:
                head(out, grad_out)
            _lib.check(lib.fsa_fused_2hop_bwd_phase_rows(*bwd_args, st, _lib.FSA_BWD_TERMS), "bwd TERMS")
            _lib.check(lib.fsa_fused_2hop_bwd_phase_rows(*bwd_args, st, _lib.FSA_BWD_ROWS), "bwd ROWS")
            if tail is not None:
                tail()
            return
        # the backward does not read the gather's output: PLAN -> ROWS run as one branch beside it
        ps = self.plan
        if head is None:
            zs.wait_stream(main)  # TERMS after the re-zeroing, on the same side stream
            _lib.check(lib.fsa_fused_2hop_bwd_phase_rows(*bwd_args, zs.cuda_stream, _lib.FSA_BWD_TERMS), "bwd TERMS")
        ps.wait_stream(main)
        _lib.check(lib.fsa_fused_2hop_bwd_phase_rows(*bwd_args, ps.cuda_stream, _lib.FSA_BWD_PLAN), "bwd PLAN")
        _lib.check(lib.fsa_fused_2hop_fwd_phase(*fwd_args, _lib.FSA_FWD_GATHER), "fwd GATHER")
        if head is not None:
            head(out, grad_out)
            _lib.check(lib.fsa_fused_2hop_bwd_phase_rows(*bwd_args, st, _lib.FSA_BWD_TERMS), "bwd TERMS")
            ps.wait_stream(main)
        ps.wait_stream(zs)  # term table written, previous rows zeroed
        _lib.check(lib.fsa_fused_2hop_bwd_phase_rows(*bwd_args, ps.cuda_stream, _lib.FSA_BWD_ROWS), "bwd ROWS")
        if tail is not None:
            tail()
        main.wait_stream(ps)

    # -- pipelined steps: forward and backward as separate launch sequences ---------------------
    def _args(self, parity: int, st: int):
        cur = self.s2[parity]
        seeds, base_seed = self.seeds_p[parity], self.base_seed_p[parity]
        grad_out, out = self.grad_out_p[parity], self.out_p[parity]
        fwd_args = (self.g.rowptr.data_ptr(), self.g.col.data_ptr(), self.N, self.X.data_ptr(), self.D,
                    self.X.stride(0), self.code, seeds.data_ptr(), self.B, self.root_offset, self.k1, self.k2,
                    0, base_seed.data_ptr(), 1, self.s1_p[parity].data_ptr(), cur.data_ptr(), self.t1.data_ptr(),
                    self.t2.data_ptr(), out.data_ptr(), out.stride(0), self.ws_f.data_ptr(),
                    self.ws_f.numel(), st)
        bwd_args = (grad_out.data_ptr(), self.B, self.D, grad_out.stride(0), self.code,
                    self.s1_p[parity].data_ptr(), cur.data_ptr(), self.k1, self.k2, self.N, self.grad_full.data_ptr(),
                    self.gx_stride, self.gx_stride, 0, self.ws_b.data_ptr(), self.ws_b.numel())
        return fwd_args, bwd_args

    def _launch_fwd(self, parity: int) -> None:
        """Pipelined step, forward: SAMPLE -> GATHER on the current stream."""
        lib = _lib.load()
        fwd_args, _ = self._args(parity, torch.cuda.current_stream(self.device).cuda_stream)
        _select_hop1(self.g)  # baked into the captured graph
        _lib.check(lib.fsa_fused_2hop_fwd_phase(*fwd_args, _lib.FSA_FWD_SAMPLE), "fwd SAMPLE")
        _lib.check(lib.fsa_fused_2hop_fwd_phase(*fwd_args, _lib.FSA_FWD_GATHER), "fwd GATHER")

    def _launch_bwd(self, parity: int) -> None:
        """Pipelined step, backward (after its forward): the previous step's rows re-zeroed, then
           zero:  re-zero prev rows ── TERMS ─┐
           plan:  PLAN ───────────────────────┴── ROWS ── (joined back to the current stream)"""
        lib = _lib.load()
        base = torch.cuda.current_stream(self.device)
        _, bwd_args = self._args(parity, base.cuda_stream)
        prev = self.s2[1 - parity]
        zs, ps = self.side, self.plan
        zs.wait_stream(base)
        ps.wait_stream(base)
        with torch.cuda.stream(zs):
            _lib.check(lib.fsa_zero_rows_strided(self.grad_full.data_ptr(), self.D, self.gx_stride, self.gx_stride,
                                                 self.code, prev.data_ptr(), prev.numel(), zs.cuda_stream),
                       "fsa_zero_rows_strided")
        _lib.check(lib.fsa_fused_2hop_bwd_phase_rows(*bwd_args, zs.cuda_stream, _lib.FSA_BWD_TERMS), "bwd TERMS")
        _lib.check(lib.fsa_fused_2hop_bwd_phase_rows(*bwd_args, ps.cuda_stream, _lib.FSA_BWD_PLAN), "bwd PLAN")
        ps.wait_stream(zs)
        _lib.check(lib.fsa_fused_2hop_bwd_phase_rows(*bwd_args, ps.cuda_stream, _lib.FSA_BWD_ROWS), "bwd ROWS")
        base.wait_stream(ps)

    def _capture_fn(self, fn, parity: int) -> torch.cuda.CUDAGraph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn(parity)
        return g

    def _launch_pipelined(self, p: int, main) -> None:
        """Step i's forward on ``main``; its backward on self.bwd after that forward.  The caller
        made ``main`` wait for step i-2's backward (which read this parity's s1 / s2)."""
        if self.use_graph and self.steps_run >= 2:
            if self.graphs[p] is None:
                self.graphs[p] = self._capture_fn(self._launch_fwd, p)
                self.graphs_b[p] = self._capture_fn(self._launch_bwd, p)
            self.graphs[p].replay()
        else:
            self._launch_fwd(p)
        self.fwd_done[p].record(main)
        self.bwd.wait_event(self.fwd_done[p])
        with torch.cuda.stream(self.bwd):
            if self.use_graph and self.steps_run >= 2:
                self.graphs_b[p].replay()
            else:
                self._launch_bwd(p)

    def _capture(self, parity: int, head=None, tail=None) -> torch.cuda.CUDAGraph:
        # warm the launch path once outside capture (device init, function attributes)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._launch(parity, head, tail)
        return g

    @property
    def out(self) -> torch.Tensor:
        """Output of the most recent step."""
        return self.out_p[1 - self.parity]

    def set_grad_out(self, grad_out: torch.Tensor) -> None:
        """Fill both grad_out buffers (steps run with ``grad_out=None`` then reuse it)."""
        for g in self.grad_out_p:
            g.copy_(grad_out)

    def run(self, seeds: Optional[torch.Tensor], base_seed: int, grad_out: Optional[torch.Tensor] = None,
            out_host: Optional[torch.Tensor] = None):
        """One step.  ``seeds`` (int64 [B]) and ``grad_out`` ([B, D]) may be device tensors or
        pinned host tensors; host inputs are copied on a copy stream into this step's buffers
        (two sets, alternating), so the copies overlap the previous step's compute.  Pass
        ``grad_out=None`` to reuse what the buffer holds.  With ``out_host`` (pinned, [B, D]) the
        step's output is copied back on the copy stream after the step.  ``grad_out=None`` reuses
        the content of this parity's buffer (see set_grad_out).  Returns
        ``(out, SampledIndices2)`` views of static buffers, valid until the step after next."""
        if not self.staged:
            self.stage(seeds, base_seed, grad_out)
        elif seeds is not None or grad_out is not None:
            raise ValueError("inputs were staged already: call run(None, base_seed)")
        return self.launch(out_host)

    def stage(self, seeds: Optional[torch.Tensor], base_seed: int, grad_out: Optional[torch.Tensor] = None) -> None:
        """Copy the next step's inputs into its buffers on the copy stream (host or device
        tensors), which waits only for the step that last read those buffers and for work queued
        on the caller's stream when an input is a device tensor.  ``run`` does this itself;
        calling it ahead of ``launch`` lets the copies overlap whatever the caller queues in
        between."""
        if self.staged:
            raise ValueError("a staged step has not been launched yet")
        p = self.parity
        main = torch.cuda.current_stream(self.device)
        if self.done_used[p]:
            self.copy.wait_event(self.done[p])
        dev_in = [t for t in (seeds, grad_out) if t is not None and t.is_cuda]
        if dev_in:  # device inputs may come from work on the caller's stream
            self.copy.wait_stream(main)
        b = int(base_seed) & 0xFFFFFFFFFFFFFFFF
        with torch.cuda.stream(self.copy):
            if seeds is not None:
                self.seeds_p[p].copy_(seeds, non_blocking=True)
            if grad_out is not None:
                self.grad_out_p[p].copy_(grad_out, non_blocking=True)
            self.base_seed_p[p].fill_(b - (1 << 64) if b >= (1 << 63) else b)  # same 64 bits, int64 storage
        for t in dev_in:  # the caller may free them while the copy is pending
            t.record_stream(self.copy)
        self.staged = True

    def launch(self, out_host: Optional[torch.Tensor] = None):
        """Run the staged step on the current stream (see ``run``)."""
        if not self.staged:
            raise ValueError("no staged inputs: call stage() first (or run())")
        self.staged = False
        p = self.parity
        main = torch.cuda.current_stream(self.device)
        main.wait_stream(self.copy)
        if self.out_copied_used[p]:  # the previous D2H of out_p[p] must finish before it is rewritten
            main.wait_event(self.out_copied[p])
            self.out_copied_used[p] = False
        if self.pipeline:
            if self.done_used[p]:  # step i-2's backward read this parity's s1 / s2
                main.wait_event(self.done[p])
            self._launch_pipelined(p, main)
            self.done[p].record(self.bwd)  # the whole step: its backward follows its forward
            self.done_used[p] = True
            if out_host is not None:
                self.copy_out.wait_event(self.fwd_done[p])
                with torch.cuda.stream(self.copy_out):
                    out_host.copy_(self.out_p[p], non_blocking=True)
                self.out_copied[p].record(self.copy_out)
                self.out_copied_used[p] = True
            self.steps_run += 1
            self.parity = 1 - p
            return self.out_p[p], SampledIndices2(self.s1_p[p], self.s2[p])
        if self.use_graph:
            if self.steps_run < 2:  # first use of each parity runs eagerly (init, attributes)
                self._launch(p)
            else:
                if self.graphs[p] is None:
                    self.graphs[p] = self._capture(p)
                self.graphs[p].replay()
        else:
            self._launch(p)
        self.done[p].record(main)
        self.done_used[p] = True
        if out_host is not None:  # on its own stream: the next step's input copies do not queue behind it
            self.copy_out.wait_event(self.done[p])
            with torch.cuda.stream(self.copy_out):
                out_host.copy_(self.out_p[p], non_blocking=True)
            self.out_copied[p].record(self.copy_out)
            self.out_copied_used[p] = True
        self.steps_run += 1
        self.parity = 1 - p
        return self.out_p[p], SampledIndices2(self.s1_p[p], self.s2[p])

    def sync_copies(self) -> None:
        """Make the current stream wait for the copy streams (pending D2H of outputs) and, when
        pipelined, for the backward stream (the feature gradient of the last step)."""
        cur = torch.cuda.current_stream(self.device)
        cur.wait_stream(self.copy)
        cur.wait_stream(self.copy_out)
        if self.pipeline:
            cur.wait_stream(self.bwd)

    def kernel_times(self, seeds_list, base_seeds, flush=None) -> dict:
        """Per-kernel device time inside the captured step graph: {name: (ms per launch, launches
        per step)}.  A dedicated graph is captured with event-record nodes around every kernel
        (fsa_profile), replayed once per (seeds, base_seed) pair, each optionally preceded by
        ``flush()`` (an L2 flush), and discarded."""
        _lib.profile(True)
        try:
            g = self._capture(self.parity)
            tot: dict = {}
            for seeds, bs in zip(seeds_list, base_seeds):
                self.seeds_p[self.parity].copy_(seeds, non_blocking=True)
                b = int(bs) & 0xFFFFFFFFFFFFFFFF
                self.base_seed_p[self.parity].fill_(b - (1 << 64) if b >= (1 << 63) else b)
                if flush is not None:
                    flush()
                g.replay()
                torch.cuda.synchronize(self.device)
                for k, (ms, n) in _lib.profile_read().items():
                    t, c = tot.get(k, (0.0, 0))
                    tot[k] = (t + ms, n)
            del g
        finally:
            _lib.profile(False)
        steps = max(1, len(base_seeds))
        return {k: (t / steps / n, n) for k, (t, n) in tot.items()}

    TRACE_NAMES = ("k_plan_roots", "k_sample1", "k_plan_hop2", "k_sample2", "k_gather2", "k_zero_rows",
                   "k_bwd_count", "k_bwd_single", "k_bwd_scatter", "k_bwd_multi", "k_bwd_big", "k_bwd_reserve",
                   "k_final2", "k_bwd_terms", "k_hop1")

    def kernel_spans(self, seeds_list, base_seeds, flush=None) -> dict:
        """Per-kernel device time of the normal step graph, from the library's per-block
        %globaltimer trace (fsa_trace): {name: (ms per launch, launches per step)}, where a
        kernel's time is its first block's start to its last block's end, averaged over one
        replay per (seeds, base_seed) pair (each optionally preceded by ``flush()``).  Unlike
        event-record nodes, the trace adds no nodes to the graph."""
        import ctypes as C
        lib = _lib.load()
        ns, nb = C.c_int(0), C.c_int(0)
        _lib.check(lib.fsa_trace_geometry(C.byref(ns), C.byref(nb)), "fsa_trace_geometry")
        buf = torch.empty((ns.value, nb.value, 2), dtype=torch.int64, device=self.device)
        tot: dict = {}
        n = 0
        try:
            for seeds, bs in zip(seeds_list, base_seeds):
                buf[..., 0] = torch.iinfo(torch.int64).max
                buf[..., 1] = 0
                _lib.check(lib.fsa_trace(buf.data_ptr()), "fsa_trace")
                if flush is not None:
                    flush()
                self.run(seeds, bs)
                torch.cuda.synchronize(self.device)
                _lib.check(lib.fsa_trace(None), "fsa_trace")
                t = buf.cpu()
                used = t[..., 1] > 0
                for slot in range(min(ns.value, len(self.TRACE_NAMES))):
                    u = used[slot]
                    if bool(u.any()):
                        span = float(t[slot, u, 1].max() - t[slot, u, 0].min()) / 1e6
                        tot[self.TRACE_NAMES[slot]] = tot.get(self.TRACE_NAMES[slot], 0.0) + span
                n += 1
        finally:
            lib.fsa_trace(None)
        return {k: (v / max(1, n), 1) for k, v in tot.items()}

