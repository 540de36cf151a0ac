"""One Llama-3.1-8B layer's 4 linears at batch B: per-linear device time under a
CUDA graph (20 launches per replay, weights rotated over >L2 copies)."""
import os, sys, statistics, torch
sys.path.insert(0, os.environ.get("PKGROOT", os.getcwd()))
import paper_2505_15909_b200 as rq
B = int(os.environ.get("B", "16")); bits = int(os.environ.get("BITS", "4")); reps = int(os.environ.get("REPS", "3"))
shapes = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
only = os.environ.get("ONLY")
if only: shapes = [s for s in shapes if s[0] in only.split(",")]
ncopy = int(os.environ.get("NCOPY", "4"))
qs = []
for name, n, k in shapes:
    g = 128 if bits == 4 else 1 << (k - 1).bit_length()
    cp = []
    for i in range(ncopy):
        w = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
        cp.append(rq.quantize_pack(w, bits, g, ragged=k % g != 0))
        del w
    qs.append(cp)
x = torch.empty(B, 4096, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
h = torch.empty(B, 14336, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
ws = rq.Workspace(device="cuda")
st = torch.cuda.Stream()
outs = {n: torch.empty(B, n, device="cuda", dtype=torch.bfloat16) for _, n, _ in shapes}
torch.cuda.synchronize()
with torch.cuda.stream(st):
    for r in range(reps):
        for (name, n, k), cp in zip(shapes, qs):
            rq.linear(x if k == 4096 else h, cp[r % ncopy], out=outs[n], workspace=ws, stream=st)
st.synchronize()
if os.environ.get("NOTIME"): sys.exit(0)
tot = 0
for (name, n, k), cp in zip(shapes, qs):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(20):
            rq.linear(x if k == 4096 else h, cp[i % ncopy], out=outs[n], workspace=ws, stream=st)
    ts = []
    for _ in range(7):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            e0.record(st); g.replay(); e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 20)
    t = statistics.median(ts[2:])
    tot += t
    print(f"{name} {n}x{k} B={B} W{bits}: {t*1e3:.2f} us  {cp[0].weight_bytes/t/1e6:.0f} GB/s", flush=True)
print(f"layer B={B} W{bits}: {tot*1e3:.2f} us")
