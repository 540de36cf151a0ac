"""One large W4 linear (405B ffn_up, 106496 x 16384, batch B) for ncu sampling captures."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
B = int(os.environ.get("B", "16"))
n, k = 106496, 16384
w = ((torch.rand(n, k, device="cuda") * 2 - 1) * 0.02).to(torch.bfloat16)
q = rq.quantize_pack(w, 4, 128)
del w
x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
ws = rq.Workspace(device="cuda")
for _ in range(3):
    rq.linear(x, q, workspace=ws, check=False)
torch.cuda.synchronize()
