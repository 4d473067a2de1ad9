"""The sampler's integer roofline (second roofline): the draw loop of k_sample
(xorshift64 step + exact `x mod (i+1)` test, kernels.py:63-67) in isolation.

  * cycles per draw of one warp (latency of the dependent chain, 1 or 32 lanes), and
  * draws/s of the whole GPU: the same loop on every resident warp (148 SMs x 32 warps), timed
    with CUDA events; this is the peak the α=2.1 sampler is measured against (bench.py `alt`).

Prints one JSON line per measurement; --json writes them as a list.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2511_13645_b200 import _lib  # noqa: E402

MODES = ["barrett", "frac", "barrett x2", "frac x2"]


def peak_draws(lib, mode, m0, n=4096, k=10, reps=5):
    """Whole-GPU draws/s of the draw loop: every SM filled with 256-thread CTAs (8 per SM)."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    lanes = sms * 8 * 256
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(reps + 1):
        a.record(st)
        _lib.check(lib.fsa_bench_draws(mode, n, m0, k, lanes, out.data_ptr(), st.cuda_stream), "bench")
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    return lanes * n / (best * 1e-3), lanes, best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    lib = _lib.load()
    rows = []
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    for mode, m0 in ((0, 16), (0, 4096), (1, 20000), (1, 200000), (2, 4096), (3, 200000)):
        r = {"mode": MODES[mode], "m0": m0}
        for lanes in (1, 32):
            n = 4096
            for _ in range(2):
                _lib.check(lib.fsa_bench_draws(mode, n, m0, 10, lanes, out.data_ptr(),
                                               torch.cuda.current_stream().cuda_stream), "bench")
                torch.cuda.synchronize()
            r[f"cycles_per_draw_{lanes}lane"] = round(int(out[0]) / n, 2)
        dps, lanes, ms = peak_draws(lib, mode, m0)
        r.update(gpu_draws_per_s=dps, gpu_lanes=lanes, gpu_ms=round(ms, 4))
        rows.append(r)
        print(json.dumps(r), flush=True)
    if args.json:
        Path(args.json).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
