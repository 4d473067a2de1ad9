"""Kernel start/end times of one GraphTrainStep replay (torch.profiler device events), to see
the step's critical path: products 15-10, alpha 3."""
import sys
sys.path.insert(0, "/root/repo")
import torch  # noqa: E402
import paper_2511_13645_b200 as fsa  # noqa: E402
from paper_2511_13645_b200 import synth, train as tr  # noqa: E402
from torch.profiler import profile, ProfilerActivity  # noqa: E402

sh = synth.SHAPES["products"]
dev = torch.device("cuda", 0)
g = synth.gen_power_law(sh.num_nodes, sh.avg_degree, 3.0, 42, device=dev)
X = synth.make_features(sh.num_nodes, sh.d_feat, 42, device=dev)
bt = synth.seed_batches(sh.num_nodes, 1024, 42, device=dev)
batches = [next(bt) for _ in range(8)]
labels = torch.randint(0, 47, (sh.num_nodes,), device=dev)
lab = [labels[b] for b in batches]
state = tr.init_train_state(sh.d_feat, 256, 47, 42, device=dev)
gts = tr.GraphTrainStep(g, X, 1024, (sh.k1, sh.k2), state)
for i in range(6):
    gts.run(batches[i % 8], lab[i % 8], fsa.step_seed(42, i))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    torch.cuda._sleep(20_000_000)
    for i in range(3):
        gts.run(batches[i % 8], lab[i % 8], fsa.step_seed(42, 6 + i))
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "sleep" not in e.name]
ev.sort(key=lambda e: e.time_range.start)
# the last step: everything after the 2nd-to-last hop1 start
starts = [e.time_range.start for e in ev if e.name.startswith("(anonymous namespace)::k_hop1")]
t0 = starts[-1]
for e in ev:
    if e.time_range.start >= t0:
        print(f"{e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f} {e.time_range.end - e.time_range.start:6.1f}  {e.name[:90]}")
