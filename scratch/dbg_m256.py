import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
n, k = int(os.environ.get("N", "28672")), 4096
m = int(os.environ.get("M", "256")); path = int(os.environ.get("P", "0"))
q = rq.quantize_pack((torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16), 4, 128)
a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
ws = rq.Workspace(device="cuda")
for i in range(3):
    t = time.time(); out = rq.linear(a, q, path=path, workspace=ws); torch.cuda.synchronize(); print(m, path, i, f"{(time.time()-t)*1e3:.2f} ms", flush=True)
