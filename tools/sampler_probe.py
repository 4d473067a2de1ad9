"""Where a sampler tile's time goes: builds (or reuses) tools/libfsa_b200_sdbg.so, the library
compiled with -DFSA_SDBG, runs CUDA-graph steps of the products shape through it, and prints
the mean clock64 cycles per tile of each k_sample sub-phase (layout, tile setup, jump-ahead,
draws, next-tile atomic) for both hops, plus the per-kernel timeline spans.

    python tools/sampler_probe.py [--alpha 3.0] [--config products]
"""
import argparse
import ctypes as C
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

DBG = ROOT / "tools" / "libfsa_b200_sdbg.so"
PHASES = ["layout", "setup", "jump", "draws", "next"]
HOP1_PHASES = ["root", "run", "finish", "prologue", "lane run"]  # k_hop1 (2-hop forward)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--alpha", type=float, default=3.0)
    p.add_argument("--config", default="products")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--rebuild", action="store_true")
    p.add_argument("--no-overlap-zero", action="store_true")
    a = p.parse_args()
    if a.rebuild or not DBG.exists():
        from paper_2511_13645_b200._build import NVCC_FLAGS, SOURCES, nvcc_path
        subprocess.run([nvcc_path(), *NVCC_FLAGS, "-DFSA_SDBG", "-o", str(DBG), *map(str, SOURCES)], check=True)
    from paper_2511_13645_b200 import _lib, synth
    _lib._LIB = _lib.load(str(DBG))
    import paper_2511_13645_b200 as fsa
    from paper_2511_13645_b200.executor import Fused2HopStep

    lib = _lib._LIB
    sh = synth.SHAPES[a.config]
    dev = torch.device("cuda", 0)
    g = synth.gen_power_law(sh.num_nodes, sh.avg_degree, a.alpha, 42, device=dev)
    X = synth.make_features(sh.num_nodes, sh.d_feat, 42, device=dev)
    batches = synth.reference_batches(sh.num_nodes, 1024, 42, device=dev)
    ex = Fused2HopStep(g, X, 1024, sh.k1, sh.k2, overlap_zero=not a.no_overlap_zero)
    gout = torch.randn((1024, sh.d_feat), device=dev)
    ns, nb = C.c_int(0), C.c_int(0)
    _lib.check(lib.fsa_trace_geometry(C.byref(ns), C.byref(nb)), "geometry")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for i in range(3):  # warm-up (captures the graphs)
        ex.run(next(batches), fsa.step_seed(42, i), gout)
    torch.cuda.synchronize()
    for rep in range(a.reps):
        buf = torch.zeros((ns.value, nb.value, 2), dtype=torch.int64, device=dev)
        buf[:16, :, 0] = 2**62  # kernel slots: block start = atomicMin
        flush.add_(1)
        torch.cuda.synchronize()
        _lib.check(lib.fsa_trace(buf.data_ptr()), "trace")
        ex.run(next(batches), fsa.step_seed(42, 10 + rep), gout)
        torch.cuda.synchronize()
        _lib.check(lib.fsa_trace(None), "trace")
        t = buf.cpu().numpy()
        t0 = min(t[sl, :, 0][t[sl, :, 1] > 0].min() for sl in range(15) if (t[sl, :, 1] > 0).any())
        print(f"--- rep {rep}")
        for slot, name in ((14, "hop1"), (3, "sample2")):
            st, en = t[slot, :, 0], t[slot, :, 1]
            used = en > 0
            d = (en[used] - st[used]) / 1e3
            print(f"{name}: start {(st[used].min() - t0) / 1e3:.1f} span {(en[used].max() - st[used].min()) / 1e3:.1f} us, "
                  f"blocks {used.sum()}, dur p50 {np.median(d):.1f} max {d.max():.1f}")
        for hop in (0, 1):
            row = []
            for ph, pname in enumerate(PHASES if hop else HOP1_PHASES):
                s = t[16 + 5 * hop + ph]
                cyc, cnt = s[:, 0].sum(), s[:, 1].sum()
                row.append(f"{pname} {cyc / max(cnt, 1):8.0f} cyc x {cnt:6d}")
            print(("k_hop1: " if hop == 0 else "hop2:   ") + " | ".join(row))


if __name__ == "__main__":
    main()
