"""How much do two independent step streams overlap?  Two executors (separate buffers and
gradients) replay their step graphs on two CUDA streams at once; the combined seeds/s against one
executor alone bounds what pipelining consecutive steps (sampling of step i+1 beside the gather
and backward of step i) could gain.

    python tools/concurrency_probe.py [--config products] [--steps 200]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2511_13645_b200 as fsa  # noqa: E402
from paper_2511_13645_b200 import synth  # noqa: E402
from paper_2511_13645_b200.executor import Fused2HopStep  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="products")
    p.add_argument("--alpha", type=float, default=3.0)
    p.add_argument("--steps", type=int, default=200)
    a = p.parse_args()
    sh = synth.SHAPES[a.config]
    dev = torch.device("cuda", 0)
    dt = torch.bfloat16 if a.config == "reddit" else torch.float32
    g = synth.gen_power_law(sh.num_nodes, sh.avg_degree, a.alpha, 42, device=dev)
    X = synth.make_features(sh.num_nodes, sh.d_feat, 42, device=dev).to(dt)
    B = 1024
    batches = synth.seed_batches(sh.num_nodes, B, 42, device=dev)
    seeds = [next(batches) for _ in range(64)]
    exs = [Fused2HopStep(g, X, B, sh.k1, sh.k2) for _ in range(2)]
    gout = torch.randn((B, sh.d_feat), device=dev).to(dt)
    for ex in exs:
        ex.set_grad_out(gout)
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]

    def run(n_ex, steps):
        for i in range(4):  # warm: eager first uses, graph capture
            for e in range(n_ex):
                with torch.cuda.stream(streams[e]):
                    exs[e].run(seeds[i % 64], fsa.step_seed(42, i))
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for s in streams[:n_ex]:
            s.wait_event(t0)
        for i in range(steps):
            for e in range(n_ex):
                with torch.cuda.stream(streams[e]):
                    exs[e].run(seeds[i % 64], fsa.step_seed(42, 100 + i))
        for s in streams[:n_ex]:
            torch.cuda.current_stream().wait_stream(s)
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
        return n_ex * steps * B / (ms / 1e3), ms / steps

    one, ms1 = run(1, a.steps)
    two, ms2 = run(2, a.steps)
    print(f"{a.config}: one stream {one / 1e6:.2f} M seeds/s ({ms1 * 1e3:.1f} us/step); two streams "
          f"{two / 1e6:.2f} M seeds/s ({ms2 * 1e3:.1f} us per pair of steps); ratio {two / one:.2f}")


if __name__ == "__main__":
    main()
