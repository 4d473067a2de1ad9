"""Per-phase times of k_head_rows (instrumented build: FSA_LIB=tools/ab/lib_trace.so, built with
-DHEAD_TRACE): concat load, hidden, ReLU, logits, softmax, dhidden, d_x_agg, stores."""
import ctypes as C
import os
import sys
sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2511_13645_b200 import train as tr, _lib  # noqa: E402
dev = torch.device("cuda", 0)
N, D, B = 2449029, 100, 1024
X = torch.randn(N, D, device=dev)
seeds = torch.randint(0, N, (B,), device=dev)
out = torch.randn(B, D, device=dev)
labels = torch.randint(0, 47, (B,), device=dev)
state = tr.init_train_state(D, 256, 47, 42, device=dev)
g = torch.empty_like(out)
for _ in range(5):
    tr.sage_head(X, seeds, out, labels, state, grad_agg=g)
torch.cuda.synchronize()
lib = _lib.load()
nb = 256
buf = (C.c_ulonglong * (9 * nb))()
assert lib.fsa_head_trace_read(buf, nb) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(nb, 9).astype(np.int64)
t0 = t[:, 0].min()
names = ["load", "hidden", "relu", "logits", "softmax", "dhidden", "dx", "stores"]
d = np.diff(t, axis=1) / 1e3
print("span us", (t[:, 8].max() - t0) / 1e3, "start spread us", (t[:, 0].max() - t0) / 1e3)
for i, n in enumerate(names):
    print(f"{n:8s} p50 {np.median(d[:, i]):6.2f} max {d[:, i].max():6.2f} us")
