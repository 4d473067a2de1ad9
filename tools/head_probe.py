"""sage_head alone on the products head shapes (B=1024, D=100, H=256, C=47), for ncu."""
import sys
sys.path.insert(0, "/root/repo")
import torch  # noqa: E402
from paper_2511_13645_b200 import train as tr  # noqa: E402
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
print("ok")
