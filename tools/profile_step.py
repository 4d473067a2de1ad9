"""A few eager fused 2-hop fwd+bwd steps on a products-shaped graph, for ncu captures:

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file launches.csv \
        python tools/profile_step.py --alpha 3.0 --steps 3
    ncu --set full --clock-control none --import-source on -k regex:k_gather2 -s 2 -c 1 -o prof \
        python tools/profile_step.py --alpha 3.0 --steps 3
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2511_13645_b200 as fsa  # noqa: E402
from paper_2511_13645_b200 import synth  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--alpha", type=float, default=3.0)
    p.add_argument("--config", default="products")
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--batch", type=int, default=1024)
    p.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    p.add_argument("--stats", action="store_true", help="print the hit-count histogram of one step")
    a = p.parse_args()
    dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
    sh = synth.SHAPES[a.config]
    dev = torch.device("cuda", 0)
    g = synth.gen_power_law(sh.num_nodes, sh.avg_degree, a.alpha, 42, device=dev)
    X = synth.make_features(sh.num_nodes, sh.d_feat, 42, device=dev).to(dt)
    batches = synth.seed_batches(sh.num_nodes, a.batch, 42, device=dev)
    gout = torch.randn((a.batch, sh.d_feat), device=dev).to(dt)
    gbuf = torch.zeros((sh.num_nodes, sh.d_feat), device=dev, dtype=dt)
    torch.cuda.synchronize()
    for i in range(a.steps):
        out, idx = fsa.fused_2hop_forward(g, X, next(batches), sh.k1, sh.k2, fsa.step_seed(42, i), validate=False)
        fsa.fused_2hop_backward(gout, idx, sh.num_nodes, out=gbuf, validate=False, zero="sparse")
        if a.stats and i == 0:
            ids = idx.s2.reshape(-1)
            cnt = torch.bincount(ids[ids >= 0].long(), minlength=sh.num_nodes)
            h = torch.bincount(cnt.clamp(max=40))
            print("slots", int((ids >= 0).sum()), "nodes", int((cnt > 0).sum()), "single", int(h[1]),
                  "multi<=32", int(h[2:33].sum()), "slots in multi", int((torch.arange(41, device=dev)[2:33] * h[2:33]).sum()),
                  "big", int(h[33:].sum()), "hist", h[:12].tolist())
            from paper_2511_13645_b200 import fused as _f
            for key, buf in _f._tls.ws.items():
                if key[2] == 4:  # FSA_OP_BWD2: header {err, multi_cursor, n_small, n_big}
                    print("bwd header", buf[:16].view(torch.int32).tolist())
    torch.cuda.synchronize()
    print("done", a.alpha, g.num_edges)


if __name__ == "__main__":
    main()
