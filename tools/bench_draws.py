"""Cycles per draw of the sampler's inner loop (fsa_bench_draws hook): one warp, one or 32 lanes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2511_13645_b200 import _lib  # noqa: E402

lib = _lib.load()
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for mode, m0 in ((0, 16), (0, 4096), (1, 20000), (1, 200000), (2, 4096), (3, 200000)):
    for lanes in (1, 32):
        n = 4096
        for rep in range(2):
            _lib.check(lib.fsa_bench_draws(mode, n, m0, 10, lanes, out.data_ptr(), torch.cuda.current_stream().cuda_stream), "bench")
            torch.cuda.synchronize()
        name = ["barrett", "frac", "barrett x2", "frac x2"][mode]
        print(f"mode {name} m0 {m0} lanes {lanes}: {int(out[0]) / n:.1f} cycles/draw")
