"""Repeat the wide-row high-collision backward many times in one process and compare every
result with the first one and with the oracle: a concurrency bug in the row writers shows up
as a rare mismatch (run on a GPU box: python tools/stress_bwd.py [reps])."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_13645_b200 as fsa  # noqa: E402
import oracle as orc  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    bad = 0
    for D, dtype in ((602, torch.bfloat16), (300, torch.float32), (100, torch.float32)):
        rng = np.random.default_rng(D)
        n, deg = 3000, 40
        col = np.stack([np.concatenate([[0], np.sort(rng.choice(np.arange(1, n), deg - 1, replace=False))])
                        for _ in range(n)]).astype(np.int32).ravel()
        rowptr = np.arange(0, n * deg + 1, deg, dtype=np.int64)
        g = fsa.CsrGraph.from_arrays(rowptr, col, device="cuda", num_nodes=n)
        X = torch.from_numpy(rng.standard_normal((n, D)).astype(np.float32)).cuda().to(dtype)
        seeds = torch.from_numpy(rng.integers(0, n, 256).astype(np.int64)).cuda()
        _, idx = fsa.fused_2hop_forward(g, X, seeds, 15, 10, 987654321)
        gout = torch.from_numpy(rng.standard_normal((256, D)).astype(np.float32)).cuda().to(dtype)
        ref = orc.backward_2hop(gout.float().cpu().numpy(), idx.s1.cpu().numpy(), idx.s2.cpu().numpy(), n)
        ref = torch.from_numpy(ref).cuda().to(dtype)
        hub = int(torch.bincount(idx.s2[idx.s2 >= 0].long()).max())
        nb = 0
        T2 = idx.s2.numel()
        touched = torch.empty(T2, dtype=torch.int32, device="cuda")
        nt = torch.empty(1, dtype=torch.int32, device="cuda")
        rows = torch.empty((T2, D), device="cuda", dtype=dtype)
        for i in range(reps):
            coo = i % 2 == 1  # alternate the dense-only and dense + COO writers
            gr = fsa.fused_2hop_backward(gout, idx, n, touched=touched if coo else None,
                                         n_touched=nt if coo else None, grad_rows=rows if coo else None)
            if coo:
                k = int(nt)
                if not torch.equal(rows[:k], ref[touched[:k].long()]):
                    print(f"D={D} rep {i}: COO rows differ", flush=True)
                    nb += 1
            if not torch.equal(gr, ref):
                nb += 1
                rows = (gr != ref).any(1).nonzero().flatten()[:5].tolist()
                if nb <= 3:
                    print(f"D={D} {dtype} rep {i}: mismatch rows {rows}", flush=True)
        print(f"D={D} {dtype}: {nb}/{reps} mismatching runs (hub hits {hub})", flush=True)
        bad += nb
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
