import sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2511_13645_b200 as fsa
from paper_2511_13645_b200 import synth
from paper_2511_13645_b200.executor import Fused2HopStep
sh = synth.SHAPES['products']
dev = torch.device('cuda', 0)
g = synth.gen_power_law(sh.num_nodes, sh.avg_degree, 3.0, 42, device=dev)
X = synth.make_features(sh.num_nodes, sh.d_feat, 42, device=dev)
bt = synth.seed_batches(sh.num_nodes, 1024, 42, device=dev)
ex = Fused2HopStep(g, X, 1024, 15, 10)
hs = [next(bt).cpu().pin_memory() for _ in range(64)]
hg = torch.randn(1024, 100).pin_memory()
ho = [torch.empty(1024, 100).pin_memory() for _ in range(2)]
for i in range(6): ex.run(hs[i], fsa.step_seed(42, i), hg, out_host=ho[i % 2])
torch.cuda.synchronize()
for label, kw in [("full", dict(grad=True, out=True)), ("seeds only", dict(grad=False, out=False)), ("seeds+out", dict(grad=False, out=True))]:
    t = time.perf_counter()
    for i in range(50):
        ex.run(hs[i], fsa.step_seed(42, i), hg if kw['grad'] else None, out_host=ho[i % 2] if kw['out'] else None)
    th = (time.perf_counter() - t) / 50 * 1e6
    ex.sync_copies(); torch.cuda.synchronize()
    t2 = (time.perf_counter() - t) / 50 * 1e6
    print(f"{label}: host enqueue {th:.1f} us/step, wall {t2:.1f} us/step")
t = time.perf_counter()
for i in range(50):
    ex.run(None, fsa.step_seed(42, i))
th = (time.perf_counter() - t) / 50 * 1e6
torch.cuda.synchronize(); t2 = (time.perf_counter() - t) / 50 * 1e6
print(f"device-resident: host enqueue {th:.1f} us/step, wall {t2:.1f} us/step")
