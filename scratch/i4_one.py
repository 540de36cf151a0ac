"""One W4 gate_up linear (28672 x 4096, batch B) for ncu captures."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
B = int(os.environ.get("B", "16")); BITS = int(os.environ.get("BITS", "4"))
n, k = 28672, 4096
w = ((torch.rand(n, k, device="cuda") * 2 - 1) * 0.02).to(torch.bfloat16)
q = rq.quantize_pack(w, BITS, 128 if BITS == 4 else 4096)
x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
ws = rq.Workspace(device="cuda")
for _ in range(5):
    rq.linear(x, q, workspace=ws, check=False)
torch.cuda.synchronize()
