"""Eager train_step (the reference-facing call): host enqueue time vs device time, and the
host-side profile of one call (cProfile), products 15-10 at alpha 3."""
import cProfile
import pstats
import sys
import time
sys.path.insert(0, "/root/repo")
import torch  # noqa: E402
import paper_2511_13645_b200 as fsa  # noqa: E402
from paper_2511_13645_b200 import synth, train as tr  # noqa: E402

sh = synth.SHAPES["products"]
dev = torch.device("cuda", 0)
g = synth.gen_power_law(sh.num_nodes, sh.avg_degree, 3.0, 42, device=dev)
X = synth.make_features(sh.num_nodes, sh.d_feat, 42, device=dev)
bt = synth.seed_batches(sh.num_nodes, 1024, 42, device=dev)
batches = [next(bt) for _ in range(16)]
labels = torch.randint(0, 47, (sh.num_nodes,), device=dev)
lab = [labels[b] for b in batches]
state = tr.init_train_state(sh.d_feat, 256, 47, 42, device=dev)
gbuf = torch.zeros((sh.num_nodes, sh.d_feat), device=dev)


def one(i):
    tr.train_step(g, X, fsa.SeedBatch(batches[i % 16], lab[i % 16]), (sh.k1, sh.k2), fsa.step_seed(42, i), "fused",
                  state, grad_scratch=gbuf)


for i in range(5):
    one(i)
torch.cuda.synchronize()
n = 50
t = time.perf_counter()
for i in range(n):
    one(i)
th = (time.perf_counter() - t) / n * 1e3
torch.cuda.synchronize()
tw = (time.perf_counter() - t) / n * 1e3
print(f"host enqueue {th:.3f} ms/step, wall {tw:.3f} ms/step")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(400_000_000)
a.record()
for i in range(n):
    one(i)
b.record()
torch.cuda.synchronize()
print(f"device only (behind a spin): {a.elapsed_time(b) / n:.3f} ms/step")
pr = cProfile.Profile()
pr.enable()
for i in range(20):
    one(i)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
