"""One Llama-3.1-8B layer's 4 linears at batch B (for ncu); eager, no graph."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
B = int(os.environ.get("B", "16")); bits = int(os.environ.get("BITS", "4")); reps = int(os.environ.get("REPS", "3"))
shapes = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
qs = []
for name, n, k in shapes:
    w = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    g = 128 if bits == 4 else 1 << (k - 1).bit_length()
    qs.append(rq.quantize_pack(w, bits, g, ragged=k % g != 0))
x = torch.empty(B, 4096, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
h = torch.empty(B, 14336, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
ws = rq.Workspace(device="cuda")
torch.cuda.synchronize()
for r in range(reps):
    for (name, n, k), q in zip(shapes, qs):
        rq.linear(x if k == 4096 else h, q, workspace=ws)
torch.cuda.synchronize()
# event timing per linear (after warmup), median of 20
import statistics
if os.environ.get("NOTIME"): sys.exit(0)
for (name, n, k), q in zip(shapes, qs):
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): rq.linear(x if k == 4096 else h, q, workspace=ws)
        e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 20)
    t = statistics.median(ts)
    byts = q.weight_bytes
    print(f"{name} {n}x{k} B={B}: {t*1e3:.1f} us  {byts/t/1e6:.0f} GB/s", flush=True)
