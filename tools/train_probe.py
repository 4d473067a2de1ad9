"""Where the SAGE training step's time goes (GraphTrainStep, products 15-10 at alpha 3):
back-to-back host-enqueued steps vs the same steps parked behind a spin kernel (device time
only), the host's enqueue time per step, and a torch.profiler kernel table of graph replays."""
import sys
import time

sys.path.insert(0, "/root/repo")
import torch  # noqa: E402
import paper_2511_13645_b200 as fsa  # noqa: E402
from paper_2511_13645_b200 import synth, train as tr  # noqa: E402

sh = synth.SHAPES[sys.argv[1] if len(sys.argv) > 1 else "products"]
dev = torch.device("cuda", 0)
g = synth.gen_power_law(sh.num_nodes, sh.avg_degree, 3.0, 42, device=dev)
X = synth.make_features(sh.num_nodes, sh.d_feat, 42, device=dev)
bt = synth.seed_batches(sh.num_nodes, 1024, 42, device=dev)
batches = [next(bt) for _ in range(32)]
labels = torch.randint(0, 47, (sh.num_nodes,), device=dev)
lab = [labels[b] for b in batches]
state = tr.init_train_state(sh.d_feat, 256, 47, 42, device=dev)
gts = tr.GraphTrainStep(g, X, 1024, (sh.k1, sh.k2), state)


def one(i):
    gts.run(batches[i % 32], lab[i % 32], fsa.step_seed(42, i))


for i in range(6):
    one(i)
torch.cuda.synchronize()
n = 100
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t = time.perf_counter()
a.record()
for i in range(n):
    one(i)
b.record()
th = (time.perf_counter() - t) / n * 1e3
torch.cuda.synchronize()
print(f"back-to-back: {a.elapsed_time(b) / n:.4f} ms/step (host enqueue {th:.4f} ms/step)")
torch.cuda._sleep(200_000_000)
a.record()
for i in range(n):
    one(i)
b.record()
torch.cuda.synchronize()
print(f"behind a spin: {a.elapsed_time(b) / n:.4f} ms/step (device only)")

from torch.profiler import profile, ProfilerActivity  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(10):
        one(i)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=60))

# the head alone (no concurrent backward PLAN kernels): sage_head on this step's shapes
out = torch.randn(1024, sh.d_feat, device=dev)
gagg = torch.empty_like(out)
for _ in range(3):
    tr.sage_head(X, batches[0], out, lab[0], state, grad_agg=gagg)
torch.cuda.synchronize()
a.record()
for _ in range(50):
    tr.sage_head(X, batches[0], out, lab[0], state, grad_agg=gagg)
b.record()
torch.cuda.synchronize()
print(f"sage_head alone: {a.elapsed_time(b) / 50 * 1e3:.1f} us per call (host-bound if close to the enqueue time)")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        tr.sage_head(X, batches[0], out, lab[0], state, grad_agg=gagg)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12, max_name_column_width=60))
