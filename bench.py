#!/usr/bin/env python
"""bench.py — seeds/s and achieved HBM GB/s of the fused 2-hop (15,10) sample + mean-aggregation
forward + replay backward on an ogbn-products-shaped synthetic power-law graph (BASELINE.json).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config products]
                    [--alpha 3.0] [--no-alt] [--profile]

A step = one forward (fused_2hop_forward, save_indices=True) + one replay backward
(fused_2hop_backward into a persistent N x D gradient buffer, re-zeroed sparsely) over one
batch of B=1024 seeds per GPU.  Multi-GPU: one process per GPU (``--gpus N`` re-launches itself
under torch.distributed.run when WORLD_SIZE is unset), seeds sharded by global batch position
(root_offset), graph + features replicated, no collective on the data path -> weak scaling
(headline); strong scaling (global B=1024) and the config-5 training step (products 25-10, SAGE
head, NCCL all-reduce of the head gradients captured in the step graph) are reported beside it.
Timing: W warm-up steps, then K steps each bracketed by CUDA events on the operator's stream,
L2 flushed (512 MiB read) before every step outside the events, barrier + synchronize around
the timed region, max over ranks.  Before timing, two batches of the executor step (one eager,
one CUDA-graph replay) are checked against the CPU oracle ("parity").

Also reported (one JSON line on rank 0): e2e through the public API with pinned host inputs,
the dominant kernel's roofline (library CUDA-event timing + algorithmic bytes), the CPU
oracle baseline on the host cores, clocks sampled during the timed region, and the same
measurement at power-law exponent 2.1 (the reference default; sampler-bound) under "alt".
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "seeds/s and achieved HBM GB/s, fused 2-hop sample+mean-agg fwd+bwd (15-10)"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["fused", "reference"], default="fused")
    p.add_argument("--config", default="products", choices=["products", "products25", "reddit", "arxiv"])
    p.add_argument("--alpha", type=float, default=3.0)
    p.add_argument("--batch", type=int, default=1024, help="seeds per GPU")
    p.add_argument("--dtype", default=None, choices=[None, "fp32", "bf16"])
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--batch-stream", default="reference", choices=["reference", "device"],
                   help="seed batches: the reference's numpy permutation stream (bench.py:172-179, bit-exact) "
                        "or a torch device randperm")
    p.add_argument("--no-alt", action="store_true", help="skip the alpha=2.1 side measurement")
    p.add_argument("--no-unfused", action="store_true", help="skip the unfused-comparator measurement")
    p.add_argument("--no-train", action="store_true", help="skip the SAGE training-step measurement")
    p.add_argument("--no-parity", action="store_true", help="skip the oracle check of two batches")
    p.add_argument("--no-strong", action="store_true", help="skip the strong-scaling (global B) measurement")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--profile", action="store_true", help="print the per-kernel table to stderr")
    p.add_argument("--eager", action="store_true", help="no CUDA graphs for the device-resident measurement")
    p.add_argument("--pipeline", action="store_true",
                   help="time pipelined back-to-back steps (executor pipeline=True: step i+1's forward beside "
                        "step i's backward) instead of single steps with an L2 flush before each")
    p.add_argument("--flush", default="read", choices=["read", "write", "none"],
                   help="L2 flush between timed steps: read 512 MiB (evicts, leaves L2 clean), write "
                        "512 MiB (evicts, leaves L2 dirty: its write-back lands in the timed step), none")
    return p.parse_args()


# ----------------------------------------------------------------------------------------------
# environment
# ----------------------------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region.

    Polls NVML in-process every 2 ms (a ctypes call, so the GIL is released while the driver
    answers); the first sample is taken before the timed region starts and at least one more
    after it ends, so a short region still carries samples. Falls back to ``nvidia-smi -lms``
    when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.stop = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
            h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        return pynvml, h

    def _poll(self):
        nv, h = self.nvml
        bits = {"hw_slowdown": nv.nvmlClocksThrottleReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksThrottleReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksThrottleReasonSwPowerCap}
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while True:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((float(sm), float(mx), {k for k, b in bits.items() if r & b}))
            except Exception:
                pass
            if self.stop.wait(0.002):
                return

    def __enter__(self):
        try:
            self.nvml = self._nvml_handle()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.samples and time.time() - t0 < 2.0:
                time.sleep(0.001)
            self.samples.clear()  # keep only samples taken from here on (the timed region)
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.15)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.nvml is not None:
            n = len(self.samples)
            t0 = time.time()
            while len(self.samples) <= n and time.time() - t0 < 0.5:  # one sample at the region's end
                time.sleep(0.001)
            self.stop.set()
            self.thread.join(timeout=2)
            return
        if self.proc is not None:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for s, m, rs in self.samples:
            sm.append(s)
            mx = m
            reasons |= rs
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def _capture_order(path):
    """(round, session) of a profiles/rNN[sM]_ncu_traffic.json name, compared numerically."""
    import re
    m = re.match(r"r(\d+)(?:_?s(\d+))?_", path.name)
    return (int(m.group(1)), int(m.group(2) or 0)) if m else (-1, -1)


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of ``kernel`` from the latest
    committed ncu --set full capture summary (profiles/r*_ncu_traffic.json), or None."""
    files = sorted((ROOT / "profiles").glob("r*_ncu_traffic.json"), key=_capture_order)
    if not files:
        return None, None
    try:
        d = json.loads(files[-1].read_text())
        k = d["kernels"][kernel]
        return k["dram_read_bytes"] + k["dram_write_bytes"], files[-1].name
    except (KeyError, ValueError):
        return None, files[-1].name


def row_ceiling(kind):
    """Practical ceiling of this path's access pattern at the products shape (153,600 random
    400-byte rows, 2.45 M-row table, L2 flushed, kernel-only %globaltimer span) from the committed
    probe run profiles/r02_row_ceiling.jsonl (tools/tma_gather_probe.cu): best register-load
    read, or the write of whole 64-byte bursts (the padded gradient rows)."""
    p = ROOT / "profiles" / "r02_row_ceiling.jsonl"
    try:
        rows = [json.loads(ln) for ln in p.read_text().splitlines() if ln.strip()]
    except OSError:
        return None
    if kind == "read":
        c = [r for r in rows if r["variant"].startswith("ldg")]
    else:
        c = [r for r in rows if r["variant"] == "write_rows" and r["p1"] == r["p2"] == 448]
    if not c:
        return None
    best = max(c, key=lambda r: r["gbs"])
    return {"gbs": best["gbs"], "probe": best, "source": str(p.relative_to(ROOT))}


def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


# ----------------------------------------------------------------------------------------------
# workload
# ----------------------------------------------------------------------------------------------
def make_inputs(shape, alpha, seed, device, dtype):
    import torch
    from paper_2511_13645_b200 import synth

    g = synth.gen_power_law(shape.num_nodes, shape.avg_degree, alpha, seed, device=device)
    row_stride = shape.d_feat
    elem = 2 if dtype == torch.bfloat16 else 4
    if (shape.d_feat * elem) % 16:
        row_stride = ((shape.d_feat * elem + 15) // 16) * 16 // elem  # 16-byte aligned rows
    X = synth.make_features(shape.num_nodes, shape.d_feat, seed, dtype=dtype, device=device,
                            row_stride=row_stride)
    return g, X


def alg_bytes(B, k1, k2, D, E, T1, T2, U2):
    """SURVEY.md §8d algorithmic bytes per batch (fwd, bwd): paper_2511_13645_b200.metrics."""
    from paper_2511_13645_b200.metrics import alg_bytes as ab
    return ab(B, k1, k2, D, E, T1, T2, U2)


def kernel_alg_bytes(name, B, k1, k2, D, E, T1, T2, U2, singles):
    """Algorithmic bytes per launch of the HBM-heavy kernels."""
    if name == "k_gather2":  # ids + feature rows + out
        return E * D * T2 + E * D * B + 4 * B * k1 * k2 + 4 * B * k1 + 4 * T2
    if name == "k_bwd_single":
        return E * D * singles + 4 * B * k1 * k2 + 4 * U2
    if name == "k_bwd_multi":
        return E * D * (U2 - singles) + 4 * (T2 - singles)
    if name == "k_bwd_terms":  # grad_out rows + the fp32 term table (G = B*k1 rows) + denominators
        return E * D * B + 4 * D * B * k1 + 4 * B * k1
    if name == "k_zero_rows":
        return E * D * T2 + 4 * B * k1 * k2
    return None


class Runner:
    """One rank's fused 2-hop fwd+bwd step loop on its shard of the global batch.

    ``mode`` "weak": ``args.batch`` seeds per rank (global batch = batch x world); "strong":
    the global batch is ``args.batch`` and each rank takes its contiguous shard.  ``inputs``
    (graph, X) reuses another runner's device inputs; ``k1`` overrides the shape's fanout."""

    def __init__(self, args, shape, alpha, device, world, rank, mode="weak", inputs=None, k1=None):
        import torch
        import paper_2511_13645_b200 as fsa
        from paper_2511_13645_b200 import synth
        from paper_2511_13645_b200.shard import shard_bounds

        self.torch, self.fsa = torch, fsa
        self.args, self.shape, self.alpha = args, shape, alpha
        self.device, self.world, self.rank, self.mode = device, world, rank, mode
        dtype = torch.bfloat16 if (args.dtype == "bf16" or (args.dtype is None and args.config == "reddit")) \
            else torch.float32
        self.dtype = dtype
        self.E = 2 if dtype == torch.bfloat16 else 4
        t0 = time.time()
        self.g, self.X = inputs if inputs is not None else make_inputs(shape, alpha, args.seed, device, dtype)
        torch.cuda.synchronize(device)
        self.gen_s = time.time() - t0
        self.N, self.D = shape.num_nodes, shape.d_feat
        self.k1, self.k2 = (k1 or shape.k1), shape.k2
        if mode == "weak":
            self.global_B = args.batch * world
            lo, hi = rank * args.batch, (rank + 1) * args.batch
        else:
            self.global_B = args.batch
            lo, hi = shard_bounds(args.batch, rank, world)
        self.B, self.root_offset = hi - lo, lo
        nsteps = max(args.warmup + args.steps, 64) + 8  # the e2e / per-call legs cycle through them
        stream = synth.reference_batches if args.batch_stream == "reference" else synth.seed_batches
        gb = stream(self.N, self.global_B, args.seed, device=device)
        self.global_batches = [next(gb) for _ in range(nsteps)]
        self.batches = [b[lo:hi].contiguous() for b in self.global_batches]
        self.base_seeds = [fsa.step_seed(args.seed, i) for i in range(nsteps)]
        gen = torch.Generator(device=device)
        gen.manual_seed(args.seed + 7)
        self.gout = torch.randn((self.B, self.D), generator=gen, device=device).to(dtype)
        self.gbuf = torch.zeros((self.N, self.D), dtype=dtype, device=device)
        self.flush_buf = torch.ones(512 << 20 >> 3, dtype=torch.int64, device=device)
        self.flush_sink = torch.zeros(1, dtype=torch.int64, device=device)
        from paper_2511_13645_b200.executor import Fused2HopStep
        self.ex = Fused2HopStep(self.g, self.X, self.B, self.k1, self.k2, root_offset=self.root_offset,
                                use_graph=not args.eager, pipeline=args.pipeline)
        self.ex.set_grad_out(self.gout)
        self.ex_lat = None  # non-pipelined executor for the single-step latency (made on demand)
        self.idx = None

    def parity(self, n_batches=2):
        """The executor's step against the CPU oracle (test infrastructure, outside every timed
        region) on this rank's shard: steps 0..3 run (the first use of each parity is eager, then
        each parity's graph is captured and replayed), batches 0 (eager) and 3 (graph replay) are
        compared: s1 / s2 bitwise, out and the feature gradient bitwise in fp32 (bf16: equal to
        the single rounding of the fp32 oracle on the same bf16 inputs, within 1e-2)."""
        torch = self.torch
        from oracle import oracle
        oracle.set_threads(os.cpu_count() or 1)
        rp, col = self.g.cpu_arrays()
        Xh = self.X.float().contiguous().cpu().numpy()
        gh = self.gout.float().cpu().numpy()
        checked, bitwise, worst = 0, True, 0.0
        want_steps = {0, 3} if n_batches >= 2 else {0}
        for i in range(4):
            out, idx = self.ex.run(self.batches[i], self.base_seeds[i], self.gout)
            if i not in want_steps:
                continue
            torch.cuda.synchronize(self.device)
            o_out, s1, s2, _, _ = oracle.fused_2hop(rp, col, Xh, self.batches[i].cpu().numpy(), self.k1, self.k2,
                                                    self.base_seeds[i], root_offset=self.root_offset)
            o_grad = oracle.backward_2hop(gh, s1, s2, self.N)
            ok_idx = np.array_equal(idx.s1.cpu().numpy(), s1) and np.array_equal(idx.s2.cpu().numpy(), s2)
            if self.dtype == torch.float32:
                ok_val = out.cpu().numpy().tobytes() == o_out.tobytes() and \
                    self.ex.grad.cpu().numpy().tobytes() == o_grad.tobytes()
            else:
                ok_val = torch.equal(out, torch.from_numpy(o_out).to(self.device).to(self.dtype)) and \
                    torch.equal(self.ex.grad, torch.from_numpy(o_grad).to(self.device).to(self.dtype))
            for a, b in ((out, o_out), (self.ex.grad, o_grad)):
                d = float((a.float() - torch.from_numpy(b).to(self.device)).abs().max())
                worst = max(worst, d / max(1.0, float(np.abs(b).max())))
            bitwise = bitwise and ok_idx and ok_val
            checked += 1
        torch.cuda.synchronize(self.device)
        return {"checked_batches": checked, "bitwise": bool(bitwise), "max_rel_err": worst,
                "what": "executor step (eager + CUDA-graph replay) vs the CPU oracle: s1/s2, out, feature grad",
                "rank": self.rank, "root_offset": self.root_offset}

    def flush_l2(self):
        """Evict L2 (126 MB) before a timed step, outside its events: a 512 MiB read (default)
        leaves L2 clean; a 512 MiB write leaves it full of dirty lines whose write-back then
        competes with the step for HBM bandwidth."""
        mode = self.args.flush
        if mode == "read":
            torch = self.torch
            torch.sum(self.flush_buf, dim=0, keepdim=True, out=self.flush_sink)
        elif mode == "write":
            self.flush_buf.fill_(1)

    def step(self, i):
        nb = len(self.batches)
        out, idx = self.ex.run(self.batches[i % nb], self.base_seeds[i % nb])
        self.idx, self.last_i = idx, i % nb
        return out

    def stage(self, i):
        """Step i's inputs (device-resident batch, base seed) into the executor's buffers, on its
        copy stream; ``launch`` then runs the step."""
        nb = len(self.batches)
        self.ex.stage(self.batches[i % nb], self.base_seeds[i % nb])
        self.last_i = i % nb

    def launch(self):
        out, idx = self.ex.launch()
        self.idx = idx
        return out

    def eager_step(self, i):
        """The same step through the public operator API (per-kernel profiling, launch counts)."""
        fsa = self.fsa
        nb = len(self.batches)
        out, idx = fsa.fused_2hop_forward(self.g, self.X, self.batches[i % nb], self.k1, self.k2, self.base_seeds[i % nb],
                                          validate=False, root_offset=self.root_offset)
        fsa.fused_2hop_backward(self.gout, idx, self.N, out=self.gbuf, validate=False, zero="sparse")
        return out

    def timed(self, steps, warmup, flush=True):
        if self.ex.pipeline:
            return self.timed_pipelined(steps, warmup)
        return self.timed_steps(steps, warmup, flush)

    def timed_pipelined(self, steps, warmup):
        """Throughput of K back-to-back pipelined steps (step i+1's forward overlaps step i's
        backward): one pair of CUDA events around all K steps, the end event after the backward
        stream has joined.  No L2 flush (the inputs, 1.5 GB, exceed the 126 MB L2); the host
        enqueues behind a spin kernel, so the events hold device work only."""
        torch = self.torch
        warmup = max(warmup, 4)
        for i in range(warmup):
            self.step(i)
        self.ex.sync_copies()
        torch.cuda.synchronize(self.device)
        from paper_2511_13645_b200 import _lib
        l0 = _lib.launch_count()
        self.eager_step(0)
        torch.cuda.synchronize(self.device)
        per_step = _lib.launch_count() - l0
        if self.world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(self.device)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_wall = time.perf_counter()
        torch.cuda._sleep(40_000_000 * max(1, steps // 50))  # the host enqueues every step meanwhile
        a.record()
        for j in range(steps):
            self.stage(warmup + j)
            self.launch()
        self.ex.sync_copies()  # joins the backward stream
        b.record()
        torch.cuda.synchronize(self.device)
        wall = time.perf_counter() - t_wall
        if self.world > 1:
            torch.distributed.barrier()
        ms = a.elapsed_time(b) / steps
        return [ms] * steps, per_step * steps, wall

    def latency(self, steps, warmup):
        """Device time of one step alone (non-pipelined executor, L2 flushed before each step)."""
        if self.ex_lat is None:
            from paper_2511_13645_b200.executor import Fused2HopStep
            self.ex_lat = Fused2HopStep(self.g, self.X, self.B, self.k1, self.k2, root_offset=self.root_offset,
                                        use_graph=not self.args.eager)
            self.ex_lat.set_grad_out(self.gout)
        ex, self.ex = self.ex, self.ex_lat
        try:
            ms, _, _ = self.timed_steps(steps, warmup, True)
        finally:
            self.ex = ex
        return ms

    def timed_steps(self, steps, warmup, flush=True):
        torch = self.torch
        # at least 4 untimed steps whatever W is: the executor runs each of its two parities
        # eagerly once, then captures each parity's graph, and no capture may fall in the
        # timed region
        warmup = max(warmup, 4)
        for i in range(warmup):
            self.step(i)
        torch.cuda.synchronize(self.device)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        from paper_2511_13645_b200 import _lib
        l0 = _lib.launch_count()
        self.eager_step(0)
        torch.cuda.synchronize(self.device)
        per_step = _lib.launch_count() - l0  # kernels one step launches (graph replays launch the same)
        if self.world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(self.device)
        t_wall = time.perf_counter()
        # The host enqueues a chunk of steps while the stream is parked behind a spin kernel, so
        # each step's events time the device only: without it, the ~0.1 ms per step the host
        # needs to submit a step (flush, input copies, graph launch) shows up inside the events
        # whenever the device runs ahead of it.  The spin is outside every step's events.
        chunk = 50
        for j in range(steps):
            if j % chunk == 0:
                torch.cuda._sleep(40_000_000)  # ~20 ms at 1.9 GHz: more than a chunk's host time
            self.stage(warmup + j)  # inputs resident before the step's events (copy stream)
            if flush:
                self.flush_l2()
            a, b = evs[j]
            a.record()
            self.launch()
            b.record()
        torch.cuda.synchronize(self.device)
        wall = time.perf_counter() - t_wall
        if self.world > 1:
            torch.distributed.barrier()
        launches = per_step * steps
        ms = [a.elapsed_time(b) for a, b in evs]
        return ms, launches, wall

    def stats(self):
        torch = self.torch
        s1, s2 = self.idx.s1, self.idx.s2
        T1 = int((s1 >= 0).sum())
        v = s2[s2 >= 0]
        T2 = int(v.numel())
        uniq, counts = torch.unique(v, return_counts=True)
        U2 = int(uniq.numel())
        singles = int((counts == 1).sum())
        return T1, T2, U2, singles

    def draws(self):
        """Algorithm-R draws of the last batch: sum over sampled nodes of max(0, deg - k)."""
        torch = self.torch
        rp = self.g.rowptr.to(torch.int64)
        deg = rp[1:] - rp[:-1]
        seeds = self.batches[self.last_i]
        s1 = self.idx.s1[self.idx.s1 >= 0].to(torch.int64)
        return int((deg[seeds] - self.k1).clamp_min(0).sum() + (deg[s1] - self.k2).clamp_min(0).sum())

    def profile(self, steps=20):
        from paper_2511_13645_b200 import _lib
        torch = self.torch
        if not self.args.eager:  # per-kernel spans inside the captured step graph (globaltimer trace)
            n = min(steps, len(self.batches))
            return self.ex.kernel_spans(self.batches[:n], self.base_seeds[:n], flush=self.flush_l2)
        torch.cuda.synchronize(self.device)
        _lib.profile(True)
        for j in range(steps):
            self.flush_l2()
            # park the stream behind a ~1 ms spin so the step's launches queue up and the
            # per-kernel events measure back-to-back device time, not host launch gaps
            torch.cuda._sleep(2_000_000)
            self.eager_step(j)
        torch.cuda.synchronize(self.device)
        prof = _lib.profile_read()
        _lib.profile(False)
        return {k: (ms / n, n / steps) for k, (ms, n) in prof.items()}

    def e2e(self, steps, warmup):
        """End to end through the public step API (executor.Fused2HopStep.run) with pinned host
        inputs: H2D of the step's seeds and grad_out, the fused fwd + replay bwd, D2H of out."""
        torch = self.torch
        h_seeds = [b.cpu().pin_memory() for b in self.batches]
        h_gout = self.gout.cpu().pin_memory()
        h_out = [torch.empty((self.B, self.D), dtype=self.dtype).pin_memory() for _ in range(2)]
        nb = len(h_seeds)

        def one(i):  # H2D of this step's inputs and D2H of its output ride the executor's copy stream
            self.ex.run(h_seeds[i % nb], self.base_seeds[i % nb], h_gout, out_host=h_out[i % 2])

        for i in range(warmup):
            one(i)
        self.ex.sync_copies()
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            torch.distributed.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for j in range(steps):
            one(warmup + j)
        self.ex.sync_copies()  # the last D2H is inside the timed region
        b.record()
        torch.cuda.synchronize(self.device)
        ms = a.elapsed_time(b) / steps
        return ms, 8 * self.B + self.E * self.B * self.D, self.E * self.B * self.D

    def e2e_eager(self, steps, warmup):
        """Same through the per-call operator API (fused_2hop_forward / fused_2hop_backward)."""
        torch, fsa = self.torch, self.fsa
        h_seeds = [b.cpu().pin_memory() for b in self.batches]
        h_gout = self.gout.cpu().pin_memory()
        h_out = torch.empty((self.B, self.D), dtype=self.dtype).pin_memory()
        nb = len(h_seeds)

        def one(i):
            seeds = h_seeds[i % nb].to(self.device, non_blocking=True)
            gout = h_gout.to(self.device, non_blocking=True)
            out, idx = fsa.fused_2hop_forward(self.g, self.X, seeds, self.k1, self.k2, self.base_seeds[i % nb],
                                              validate=False, root_offset=self.root_offset)
            fsa.fused_2hop_backward(gout, idx, self.N, out=self.gbuf, validate=False, zero="sparse")
            h_out.copy_(out, non_blocking=True)

        for i in range(warmup):
            one(i)
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            torch.distributed.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for j in range(steps):
            one(warmup + j)
        b.record()
        torch.cuda.synchronize(self.device)
        ms = a.elapsed_time(b) / steps
        return ms, 8 * self.B + self.E * self.B * self.D, self.E * self.B * self.D


    def train(self, steps, warmup, graph_mode, hidden=256, classes=47):
        """SAGE training step (head H=256, C=47, AdamW) around the fused
        op: GraphTrainStep (CUDA graphs; with world > 1 the head-gradient all-reduce is captured in
        the step graph) or the eager train_step (handed the GLOBAL batch: it shards it itself and
        all-reduces).  Device-resident seeds/labels.  Returns ms per step, max over ranks."""
        torch, fsa = self.torch, self.fsa
        from paper_2511_13645_b200 import train as tr
        state = tr.init_train_state(self.D, hidden, classes, 42, dtype=torch.float32, device=self.device)
        gen = torch.Generator(device=self.device)
        gen.manual_seed(7)
        labels = torch.randint(0, classes, (self.N,), generator=gen, device=self.device)
        X = self.X
        if graph_mode:
            gts = tr.GraphTrainStep(self.g, X, self.B, (self.k1, self.k2), state, root_offset=self.root_offset,
                                    global_batch=self.global_B)
        gbuf = torch.zeros((self.N, self.D), dtype=X.dtype, device=self.device)
        nb = len(self.batches)

        def one(i):
            j = i % nb
            if graph_mode:
                gts.run(self.batches[j], labels[self.batches[j]], self.base_seeds[j])
            else:
                gseeds = self.global_batches[j]
                tr.train_step(self.g, X, fsa.SeedBatch(gseeds, labels[gseeds]), (self.k1, self.k2),
                              self.base_seeds[j], "fused", state, grad_scratch=gbuf)

        for i in range(warmup):
            one(i)
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(self.device)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for j in range(steps):
            one(warmup + j)
        b.record()
        torch.cuda.synchronize(self.device)
        ms = a.elapsed_time(b) / steps
        if self.world > 1:
            torch.distributed.barrier()
        return max_over_ranks(ms, self.world, self.device)

    def per_call(self, steps, warmup, impl):
        """Device time of one fwd+bwd through the per-call API with device-resident inputs:
        impl "fused" (fused_2hop_forward/backward) or "unfused" / "unfused_dedup" (the
        materialised comparator, baseline.py).  Both re-zero the gradient sparsely.  Returns
        (ms per step, bytes the unfused block and gradient block materialise per step)."""
        torch, fsa = self.torch, self.fsa
        extra = [0]

        def one(i):
            seeds = self.batches[i % len(self.batches)]
            if impl == "fused":
                _, idx = fsa.fused_2hop_forward(self.g, self.X, seeds, self.k1, self.k2,
                                                self.base_seeds[i % len(self.base_seeds)],
                                                validate=False, root_offset=self.root_offset)
                fsa.fused_2hop_backward(self.gout, idx, self.N, out=self.gbuf, validate=False, zero="sparse")
            else:
                _, blk = fsa.baseline_forward(self.g, self.X, seeds, self.k1, self.k2,
                                              self.base_seeds[i % len(self.base_seeds)],
                                              dedup=impl == "unfused_dedup", validate=False,
                                              root_offset=self.root_offset)
                fsa.baseline_backward(self.gout, blk, self.N, out=self.gbuf, zero="sparse", validate=False)
                acc = 8 if self.dtype == torch.float64 else 4
                extra[0] = blk.nbytes() + blk.ids2.numel() * (-(-self.D // 8) * 8) * acc  # + gradient block

        for i in range(warmup):
            one(i)
        torch.cuda.synchronize(self.device)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for j in range(steps):
            one(warmup + j)
        b.record()
        torch.cuda.synchronize(self.device)
        return a.elapsed_time(b) / steps, extra[0]


def max_over_ranks(x, world, device):
    if world == 1:
        return x
    import torch
    on_dev = torch.distributed.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=device if on_dev else "cpu")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------------------------
# CPU oracle baseline (test infrastructure: oracle/ is only the checker / CPU timer here)
# ----------------------------------------------------------------------------------------------
def cpu_oracle_time(runner, budget_s, max_steps=None, threads=None):
    from oracle import oracle

    threads = threads or os.cpu_count()
    oracle.set_threads(threads)
    rp, col = runner.g.cpu_arrays()
    X = runner.X.float().contiguous().cpu().numpy() if runner.dtype != runner.torch.float32 else \
        runner.X.contiguous().cpu().numpy()
    gout = runner.gout.float().cpu().numpy()
    gbuf = np.zeros((runner.N, runner.D), np.float32)
    times = []
    t_start = time.perf_counter()
    i = 0
    while True:
        seeds = runner.batches[i % len(runner.batches)].cpu().numpy()
        t0 = time.perf_counter()
        out, s1, s2, _, _ = oracle.fused_2hop(rp, col, X, seeds, runner.k1, runner.k2, runner.base_seeds[i],
                                              root_offset=runner.root_offset)
        oracle.backward_2hop(gout, s1, s2, runner.N, out=gbuf)
        times.append(time.perf_counter() - t0)
        i += 1
        if (time.perf_counter() - t_start) >= budget_s or (max_steps and i >= max_steps):
            break
    return times, threads


def draw_peak(device):
    """The sampler's integer roofline: whole-GPU draws/s of k_sample's draw loop in isolation
    (fsa_bench_draws; tools/bench_draws.py), at the moduli the alpha=2.1 draws run at (the
    fraction-test path, m >= 16,384), best of the one- and two-stream forms of the loop."""
    import torch
    from paper_2511_13645_b200 import _lib

    lib = _lib.load()
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    lanes, n = sms * 8 * 256, 4096
    out = torch.zeros(2, dtype=torch.int64, device=device)
    st = torch.cuda.current_stream(device)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = {}
    for mode, name in ((1, "frac"), (3, "frac x2")):
        ms = []
        for _ in range(4):
            a.record(st)
            _lib.check(lib.fsa_bench_draws(mode, n, 200000, 15, lanes, out.data_ptr(), st.cuda_stream), "draws")
            b.record(st)
            torch.cuda.synchronize(device)
            ms.append(a.elapsed_time(b))
        best[name] = lanes * n / (min(ms[1:]) * 1e-3)
    name = max(best, key=best.get)
    return best[name], {"loop": name, "lanes": lanes, "draws_per_lane": n, "m0": 200000,
                        "all": {k: round(v, 1) for k, v in best.items()}}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ----------------------------------------------------------------------------------------------
def run_fused(args):
    import torch
    for knob, env in ((1, "FSA_SEG_DIV"), (2, "FSA_GATHER_PREFETCH"), (3, "FSA_ZERO_CTAS"), (4, "FSA_COUNT_CTAS"),
                      (5, "FSA_MULTI_CTAS"), (6, "FSA_HOP1")):  # experiment knobs (fsa_tune)
        if os.environ.get(env):
            from paper_2511_13645_b200 import _lib
            _lib.check(_lib.load().fsa_tune(knob, int(os.environ[env])), env)
    from paper_2511_13645_b200 import synth

    world, rank, local = dist_env()
    # one process per GPU over NCCL; FSA_DIST_BACKEND=gloo lets a 1-GPU box exercise the
    # multi-rank path (ranks then share cuda:0, which NCCL refuses) - a functional check only
    backend = os.environ.get("FSA_DIST_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    gpu = local % max(1, ndev) if backend != "nccl" else local
    if world > 1:
        torch.cuda.set_device(gpu)
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            torch.distributed.init_process_group(backend)
    device = torch.device("cuda", gpu)
    torch.cuda.set_device(device)
    shape = synth.SHAPES[args.config]

    def measure(alpha, full=True):
        r = Runner(args, shape, alpha, device, world, rank)
        parity = None
        if full and rank == 0 and not args.no_parity:
            parity = r.parity()
        if world > 1:
            torch.distributed.barrier()
        with ClockSampler(gpu) as clk:
            ms, launches, wall = r.timed(args.steps, args.warmup)
        mean_ms = statistics.mean(ms)
        ms_max = max_over_ranks(mean_ms, world, device)
        T1, T2, U2, singles = r.stats()
        res = {"runner": r, "ms": ms_max, "ms_local": mean_ms, "launches": launches, "clocks": clk.summary(),
               "T1": T1, "T2": T2, "U2": U2, "singles": singles, "draws": r.draws(), "gen_s": r.gen_s,
               "p50": statistics.median(ms), "wall": wall, "parity": parity}
        if full and r.ex.pipeline:  # one step alone, L2 flushed: the latency the pipeline overlaps
            lat = max_over_ranks(statistics.mean(r.latency(max(20, args.steps // 2), args.warmup)), world, device)
            res["latency"] = lat
        if full:
            res["prof"] = r.profile()
            res["e2e"] = r.e2e(max(20, args.steps // 2), 3)
            res["e2e_eager"] = r.e2e_eager(max(20, args.steps // 2), 3)
            if not args.no_train and r.dtype == torch.float32:
                res["train"] = {m: r.train(max(20, args.steps // 4), 5, m == "graph") for m in ("graph", "eager")}
            if not args.no_unfused:
                res["per_call"] = {impl: r.per_call(max(20, args.steps // 4), 3, impl)
                                   for impl in ("fused", "unfused", "unfused_dedup")}
        return res

    main = measure(args.alpha)
    r = main["runner"]
    strong = None
    if world > 1 and not args.no_strong:  # the same op step with the global batch fixed at args.batch
        rs = Runner(args, shape, args.alpha, device, world, rank, mode="strong", inputs=(r.g, r.X))
        ms_s, _, _ = rs.timed(max(20, args.steps // 2), args.warmup)
        ms_s = max_over_ranks(statistics.mean(ms_s), world, device)
        strong = {"global_batch": rs.global_B, "batch_per_gpu": [rs.B, "rank 0"], "ms_per_step": round(ms_s, 5),
                  "value": round(rs.global_B / (ms_s / 1e3), 1), "unit": "seeds/s"}
        del rs
    elif world == 1:
        strong = {"global_batch": r.global_B, "batch_per_gpu": r.B, "ms_per_step": round(main["ms"], 5),
                  "value": round(r.global_B / (main["ms"] / 1e3), 1), "unit": "seeds/s",
                  "note": "N=1: the strong-scaling workload is the headline workload"}
    config5 = None
    if not args.no_train and args.config in ("products", "products25") and r.dtype == torch.float32:
        # BASELINE.json config 5: products 25-10 SAGE training step, seed-sharded, NCCL all-reduce of
        # the head gradients (captured in the step's CUDA graph); same graph and features
        config5 = {"workload": "ogbn-products-shaped 2-hop (25,10) SAGE-mean training step (fused op fwd+bwd, "
                               "head H=256 C=47, cross-entropy, AdamW), GraphTrainStep",
                   "collective": "one all-reduce of the head gradients + loss per step (254 KB fp32), "
                                 + ("NCCL, captured in the step graph" if world > 1 and backend == "nccl"
                                    else "none at N=1" if world == 1 else f"{backend}, eager step"),
                   "unit": "seeds/s"}
        for mode in (("weak", "strong") if world > 1 else ("weak",)):
            r5 = Runner(args, synth.SHAPES["products25"], args.alpha, device, world, rank, mode=mode,
                        inputs=(r.g, r.X), k1=25)
            ms5 = r5.train(max(20, args.steps // 4), 5, True)
            config5[mode] = {"global_batch": r5.global_B, "ms_per_step": round(ms5, 5),
                             "value": round(r5.global_B / (ms5 / 1e3), 1)}
            del r5
    B, k1, k2, D, E = r.B, r.k1, r.k2, r.D, r.E
    fwd_b, bwd_b = alg_bytes(B, k1, k2, D, E, main["T1"], main["T2"], main["U2"])
    step_bytes = fwd_b + bwd_b
    seeds_s = world * B / (main["ms"] / 1e3)
    peak, peak_kind = measured_peak_hbm()

    # roofline of the dominant HBM kernel (the largest time share among the kernels that move
    # algorithmic bytes; the samplers are integer-issue bound and reported as draws/s)
    prof = main["prof"]
    hbm_k = [k for k in prof if k != "k_zero_rows" and kernel_alg_bytes(k, B, k1, k2, D, E, 1, 1, 1, 0)]
    dom = max(hbm_k, key=lambda k: prof[k][0] * prof[k][1])
    top = max(prof, key=lambda k: prof[k][0] * prof[k][1])
    dom_ms = prof[dom][0]
    kb = kernel_alg_bytes(dom, B, k1, k2, D, E, main["T1"], main["T2"], main["U2"], main["singles"])
    achieved = kb / (dom_ms / 1e3) / 1e9 if kb else None
    # the committed capture is of the products alpha=3 step (tools/profile_step.py defaults)
    traffic, traffic_src = ncu_traffic(dom) if (args.config == "products" and args.alpha == 3.0
                                                and E == 4) else (None, None)
    ceil_kind = {"k_gather2": "read", "k_bwd_single": "write"}.get(dom)
    ceiling = row_ceiling(ceil_kind) if (ceil_kind and args.config in ("products", "products25")
                                         and E == 4) else None
    if ceiling and achieved:
        ceiling["frac"] = achieved / ceiling["gbs"]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "random_row_ceiling": ceiling,
                "traffic": traffic,
                "traffic_source": traffic_src, "alg_bytes_per_launch": kb,
                "peak_kind": peak_kind, "kernel_ms": dom_ms,
                "share_of_step": prof[dom][0] * prof[dom][1] / main["ms_local"],
                "timing": "per-block %globaltimer trace of a graph replay after an L2 flush "
                          "(first block start to last block end)",
                "top_kernel": {"name": top, "ms": prof[top][0], "bound": "integer issue (sampler)"
                               if "sample" in top else "hbm/latency"}}
    kernels = {k: {"ms": round(v[0], 5), "per_step": v[1],
                   "alg_bytes": kernel_alg_bytes(k, B, k1, k2, D, E, main["T1"], main["T2"], main["U2"],
                                                 main["singles"])} for k, v in sorted(prof.items())}
    for k, v in kernels.items():
        if v["alg_bytes"]:
            v["gbs"] = round(v["alg_bytes"] / (v["ms"] / 1e3) / 1e9, 1)

    e2e_ms, h2d, d2h = main["e2e"]
    e2e_ms = max_over_ranks(e2e_ms, world, device)
    e2e_eager_ms = max_over_ranks(main["e2e_eager"][0], world, device)
    line = {
        "metric": METRIC,
        "value": round(seeds_s, 1),
        "unit": "seeds/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(main["ms"], 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16" if r.dtype == torch.bfloat16 else "fp32",
        "data": "synthetic (GPU power-law generator, graph.py:157 algorithm; standard-normal features; seed "
                + ("batches = the reference's _batch_stream, bench.py:172-179)" if args.batch_stream == "reference"
                   else "batches from a device randperm)"),
        "config": {
            "workload": f"{shape.name} 2-hop ({k1},{k2}) fused sample+mean fwd+bwd, B={B}/GPU",
            "num_nodes": r.N, "arcs": r.g.num_edges, "max_degree": r.g.max_degree(), "alpha": args.alpha,
            "avg_degree_target": shape.avg_degree, "d_feat": D, "batch_per_gpu": B, "global_batch": B * world,
            "fanouts": [k1, k2], "parallelism": f"seed-sharded dp{world} (root_offset), no data-path collective",
            "l2": ("no flush between pipelined steps: inputs (1.5 GB CSR + features, random rows) are larger "
                   "than L2; the single-step latency leg flushes L2 before every step"
                   if r.ex.pipeline else
                   {"read": "flushed before every timed step by a 512 MiB read outside the step's CUDA events "
                            "(evicts L2, leaves it clean); inputs (1.5 GB CSR + features) are larger than L2",
                    "write": "flushed before every timed step by a 512 MiB write outside the step's CUDA events",
                    "none": "no flush; inputs (1.5 GB CSR + features, random rows) are larger than L2"}[args.flush]),
            "step_timing": ("K steps back to back through the pipelined executor (step i+1's forward overlaps "
                            "step i's backward), one pair of CUDA events around all K on the caller's stream after "
                            "the backward stream joins; value = K x B / that time; the host enqueues behind a "
                            "spin kernel" if r.ex.pipeline else
                            "CUDA events around each step on its stream; the step's inputs are staged into the "
                            "executor's buffers (copy stream) before its events; the host enqueues 50 steps at a "
                            "time behind a spin kernel, so the events time device work, not host submission"),
            "grad_buffer": "persistent N x D, sparse re-zero of the previous step's rows (fsa_zero_rows) "
                           "on a side stream overlapped with the forward",
            "execution": "eager" if args.eager else "CUDA graph per step (executor.Fused2HopStep)",
            "graph_gen_s": round(main["gen_s"], 2),
        },
        "hbm": {"alg_bytes_per_step": step_bytes, "fwd_bytes": fwd_b, "bwd_bytes": bwd_b,
                "achieved_gbs": round(step_bytes / (main["ms"] / 1e3) / 1e9, 1),
                "frac_of_peak": round(step_bytes / (main["ms"] / 1e3) / 1e9 / peak, 4), "peak_gbs": peak,
                "peak_kind": peak_kind, "frac_of_8tbs_nominal": round(step_bytes / (main["ms"] / 1e3) / 8e12, 4),
                "T1": main["T1"], "T2": main["T2"], "U2": main["U2"]},
        "draws_per_step": main["draws"],
        "draws_per_s": round(main["draws"] / (main["ms"] / 1e3), 1),
        "roofline": roofline,
        "kernels": kernels,
        "clocks": main["clocks"],
        "gpu_launches": main["launches"],
        "launches_per_step": main["launches"] / args.steps,
        "e2e": {"value": round(world * B / (e2e_ms / 1e3), 1), "unit": "seeds/s", "ms_per_step": round(e2e_ms, 5),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "public step API (executor.Fused2HopStep.run, CUDA graph) with pinned host seeds + "
                        "grad_out copied H2D and out copied D2H every step",
                "per_call_api": {"value": round(world * B / (e2e_eager_ms / 1e3), 1),
                                 "ms_per_step": round(e2e_eager_ms, 5),
                                 "path": "fused_2hop_forward + fused_2hop_backward(zero='sparse') per call"}},
        "p50_ms": round(main["p50"], 5),
    }
    if "latency" in main:
        line["step_latency"] = {"ms": round(main["latency"], 5),
                                "timing": "one step alone through the non-pipelined executor, L2 flushed by a 512 "
                                          "MiB read before each step, per-step CUDA events (device work only)"}
    if main["parity"] is not None:
        line["parity"] = main["parity"]
    if strong is not None:
        line["strong_scaling"] = strong
    if config5 is not None:
        line["config5_train"] = config5
    if "train" in main:  # the caller of the hot path: the SAGE training step around the fused op
        tr_ms = main["train"]
        line["train_step"] = {
            "path": "SAGE head H=256, C=47, cross-entropy, AdamW around the fused op; device-resident batches",
            "graph": {"ms_per_step": round(tr_ms["graph"], 5), "value": round(world * B / (tr_ms["graph"] / 1e3), 1)},
            "eager": {"ms_per_step": round(tr_ms["eager"], 5), "value": round(world * B / (tr_ms["eager"] / 1e3), 1)},
            "unit": "seeds/s"}
    if "per_call" in main:  # the paper's comparison: fused vs the materialised pipeline, same API level
        pc = main["per_call"]
        fused_ms = pc["fused"][0]
        line["unfused_comparator"] = {
            "path": "per-call API, device-resident inputs, sparse gradient re-zero: fused_2hop_forward/backward "
                    "vs baseline_forward/backward (materialised blocks, baseline.py)",
            "fused": {"ms_per_step": round(fused_ms, 5), "value": round(world * B / (fused_ms / 1e3), 1)},
            **{impl: {"ms_per_step": round(pc[impl][0], 5), "value": round(world * B / (pc[impl][0] / 1e3), 1),
                      "speedup_of_fused": round(pc[impl][0] / fused_ms, 3),
                      "materialised_bytes_per_step": pc[impl][1]} for impl in ("unfused", "unfused_dedup")},
            "unit": "seeds/s"}
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU baseline is an N=1 figure
        times, threads = cpu_oracle_time(r, args.cpu_seconds, max_steps=30)
        cpu_ms = statistics.median(times) * 1e3
        line["cpu_baseline"] = {"value": round(B / (cpu_ms / 1e3), 2), "unit": "seeds/s", "cores": threads,
                                "kind": "port", "ms_per_step": round(cpu_ms, 2),
                                "sample": f"{len(times)} steps of the same workload (B={B}), fwd+bwd incl. the "
                                          f"reference's N x D zero-fill, OpenMP {threads} threads, {cpu_model()}"}
    del main, r
    torch.cuda.empty_cache()
    if not args.no_alt and args.alpha != 2.1:
        alt = measure(2.1, full=False)
        ra = alt["runner"]
        fb, bb = alg_bytes(B, k1, k2, D, E, alt["T1"], alt["T2"], alt["U2"])
        line["alt"] = {"alpha": 2.1, "value": round(world * B / (alt["ms"] / 1e3), 1), "unit": "seeds/s",
                       "ms_per_step": round(alt["ms"], 4), "draws_per_step": alt["draws"],
                       "draws_per_s": round(alt["draws"] / (alt["ms"] / 1e3), 1),
                       "hbm_gbs": round((fb + bb) / (alt["ms"] / 1e3) / 1e9, 1),
                       "arcs": ra.g.num_edges, "max_degree": ra.g.max_degree(), "clocks": alt["clocks"]}
        # second roofline: the sampler is integer-issue bound at alpha=2.1
        aprof = ra.profile(steps=5)
        samp = {k: v for k, v in aprof.items() if k.startswith("k_sample") or k == "k_hop1"}
        samp_ms = sum(v[0] * v[1] for v in samp.values())
        peak_d, peak_info = draw_peak(device)
        ach_d = alt["draws"] / (samp_ms / 1e3) if samp_ms else None
        line["alt"]["roofline"] = {
            "bound": "int", "kernels": sorted(samp), "sampler_ms": round(samp_ms, 5),
            "share_of_step": round(samp_ms / alt["ms_local"], 4),
            "achieved_draws_s": round(ach_d, 1) if ach_d else None, "peak_draws_s": round(peak_d, 1),
            "frac": round(ach_d / peak_d, 4) if ach_d else None, "unit": "draws/s",
            "peak_kind": "measured: k_sample's draw loop on every resident warp (fsa_bench_draws)",
            "peak_detail": peak_info,
            "kernels_ms": {k: round(v[0], 5) for k, v in sorted(aprof.items())}}
        if rank == 0 and world == 1 and not args.no_cpu:  # the CPU baseline is an N=1 figure
            times, threads = cpu_oracle_time(ra, args.cpu_seconds, max_steps=10)
            line["alt"]["cpu_baseline"] = {"value": round(B / statistics.median(times), 2), "unit": "seeds/s",
                                           "cores": threads, "kind": "port",
                                           "sample": f"{len(times)} steps (B={B})"}
        del alt, ra
    if args.profile and rank == 0:
        print(json.dumps(kernels, indent=1), file=sys.stderr)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def run_reference(args):
    """Reference arm: the CPU restatement of the reference algorithm (oracle/, the reference is a
    Python/numba package with no C sources to build) on all host cores, rank 0 only."""
    world, rank, local = dist_env()
    if rank != 0:
        return
    import torch
    from paper_2511_13645_b200 import synth

    shape = synth.SHAPES[args.config]
    device = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
    r = Runner.__new__(Runner)
    r.torch, r.args, r.shape, r.device = torch, args, shape, device
    r.dtype = torch.float32
    r.g, r.X = make_inputs(shape, args.alpha, args.seed, device, torch.float32)
    r.N, r.D, r.B, r.k1, r.k2 = shape.num_nodes, shape.d_feat, args.batch, shape.k1, shape.k2
    r.root_offset = 0
    stream = synth.reference_batches if args.batch_stream == "reference" else synth.seed_batches
    gb = stream(r.N, r.B, args.seed, device=device)
    r.batches = [next(gb) for _ in range(args.warmup + args.steps)]
    import paper_2511_13645_b200 as fsa
    r.base_seeds = [fsa.step_seed(args.seed, i) for i in range(len(r.batches))]
    gen = torch.Generator(device=device)
    gen.manual_seed(args.seed + 7)
    r.gout = torch.randn((r.B, r.D), generator=gen, device=device)
    # warm-up steps untimed, then K bounded steps
    cpu_oracle_time(r, 0.0, max_steps=max(1, args.warmup))
    times, threads = cpu_oracle_time(r, 1e9, max_steps=args.steps)
    ms = statistics.mean(times) * 1e3
    v = r.B / (ms / 1e3)
    line = {"metric": METRIC, "impl": "reference", "value": round(v, 2), "unit": "seeds/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic (GPU power-law generator); reference algorithm timed on the host CPU",
            "config": {"workload": f"{shape.name} 2-hop ({r.k1},{r.k2}) fused sample+mean fwd+bwd, B={r.B}",
                       "num_nodes": r.N, "arcs": r.g.num_edges, "alpha": args.alpha, "d_feat": r.D},
            "cpu_baseline": {"value": round(v, 2), "unit": "seeds/s", "cores": threads, "kind": "port",
                             "sample": f"{args.steps} steps of B={r.B} seeds (fwd + bwd incl. N x D zero-fill), "
                                       f"{cpu_model()}"},
            "e2e": {"value": round(v, 2), "unit": "seeds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def relaunch_ranks(args) -> int:
    """``--gpus N`` (N > 1) without a torchrun environment: re-run this script as N ranks, one
    process per GPU, under torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    import socket
    if os.environ.get("FSA_DIST_BACKEND", "nccl") == "nccl":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has {have} "
                  "(FSA_DIST_BACKEND=gloo shares one GPU for a functional check)", file=sys.stderr)
            return 2
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if args.impl == "fused" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_fused(args)


if __name__ == "__main__":
    main()
