"""Per-kernel, per-block timeline of one fused 2-hop step (globaltimer trace, fsa_trace).

    python tools/timeline.py [--alpha 3.0] [--config products] [--eager]

Prints, per kernel slot: start / end relative to the step's first block, the block count, and
block-duration percentiles, so the critical path (which kernel, which straggler block) is
visible.  Runs on one GPU; the numbers are from a CUDA-graph replay after an L2 flush."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_13645_b200 as fsa  # noqa: E402
from paper_2511_13645_b200 import _lib, synth  # noqa: E402
from paper_2511_13645_b200.executor import Fused2HopStep  # noqa: E402

NAMES = ["plan_roots", "sample1", "plan_hop2", "sample2", "gather", "zero_rows", "bwd_count", "bwd_single",
         "bwd_scatter", "bwd_multi", "bwd_big", "bwd_reserve", "final2", "bwd_terms", "hop1"]


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--alpha", type=float, default=3.0)
    p.add_argument("--config", default="products")
    p.add_argument("--eager", action="store_true")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--dtype", default=None, choices=["f32", "bf16"], help="default: bf16 for reddit, else f32")
    a = p.parse_args()
    bf16 = a.dtype == "bf16" or (a.dtype is None and a.config == "reddit")
    sh = synth.SHAPES[a.config]
    dev = torch.device("cuda", 0)
    g = synth.gen_power_law(sh.num_nodes, sh.avg_degree, a.alpha, 42, device=dev)
    X = synth.make_features(sh.num_nodes, sh.d_feat, 42, device=dev)
    if bf16:  # 16-byte row stride, as bench.py does
        stride = -(-sh.d_feat * 2 // 16) * 16 // 2
        X = synth.make_features(sh.num_nodes, sh.d_feat, 42, dtype=torch.bfloat16, device=dev, row_stride=stride)
    batches = synth.seed_batches(sh.num_nodes, 1024, 42, device=dev)
    ex = Fused2HopStep(g, X, 1024, sh.k1, sh.k2, use_graph=not a.eager)
    ex.set_grad_out(torch.randn((1024, sh.d_feat), device=dev).to(X.dtype))
    flush = torch.ones(512 << 20 >> 3, dtype=torch.int64, device=dev)
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    for i in range(6):
        ex.run(next(batches), fsa.step_seed(42, i))
    torch.cuda.synchronize()
    ns, nb = _lib.C.c_int(0), _lib.C.c_int(0)
    _lib.check(_lib.load().fsa_trace_geometry(_lib.C.byref(ns), _lib.C.byref(nb)), "geom")
    S, NB = ns.value, nb.value
    buf = torch.empty((S, NB, 2), dtype=torch.int64, device=dev)
    for rep in range(a.reps):
        buf[..., 0] = torch.iinfo(torch.int64).max
        buf[..., 1] = 0
        _lib.check(_lib.load().fsa_trace(buf.data_ptr()), "trace")
        torch.sum(flush, dim=0, keepdim=True, out=sink)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        ex.run(next(batches), fsa.step_seed(42, 100 + rep))
        ev[1].record()
        torch.cuda.synchronize()
        _lib.check(_lib.load().fsa_trace(None), "trace off")
        t = buf.cpu().numpy()
        s2 = ex.s2[1 - ex.parity].reshape(-1)
        s2 = s2[s2 >= 0]
        _, cnts = torch.unique(s2, return_counts=True)
        cn = cnts.cpu().numpy()
        print(f"slots {s2.numel()} distinct {len(cn)} multi {int((cn > 1).sum())} big(>32) {int((cn > 32).sum())} "
              f"max count {int(cn.max())} top5 {sorted(cn.tolist())[-5:]}")
        used = t[..., 1] > 0
        t0 = t[..., 0][used].min()
        print(f"--- rep {rep}: step {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us (events)")
        for sl in range(S):
            u = used[sl]
            if not u.any():
                continue
            st = (t[sl, u, 0] - t0) / 1e3
            en = (t[sl, u, 1] - t0) / 1e3
            du = en - st
            last = int(np.argmax(en))
            print(f"{NAMES[sl] if sl < len(NAMES) else sl:12s} start {st.min():7.1f} end {en.max():7.1f} "
                  f"span {en.max() - st.min():6.1f} | blocks {u.sum():5d} dur p50 {np.median(du):6.1f} "
                  f"p90 {np.percentile(du, 90):6.1f} max {du.max():6.1f} | last block #{np.flatnonzero(u)[last]} "
                  f"start {st[last]:6.1f}")


if __name__ == "__main__":
    main()
