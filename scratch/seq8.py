"""ffn_up W8 per-channel (28672 x 4096) at batch B: per-launch time with planes (rq.linear) vs
precomputed (linear_planes), 20 launches over 4 weight copies in a CUDA graph."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
B = int(os.environ.get("B", "16")); BITS = int(os.environ.get("BITS", "8"))
n, k = 28672, 4096
g = int(os.environ.get("G", "128" if BITS == 4 else "4096"))
qs = [rq.quantize_pack(((torch.rand(n, k, device="cuda") * 2 - 1) * 0.02).to(torch.bfloat16), BITS, g) for _ in range(4)]
x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
out = torch.empty(B, n, device="cuda", dtype=torch.bfloat16)
pl = rq.act_planes(x, rq.Planes(B, k, "cuda"))
ws = rq.Workspace(device="cuda")
st = torch.cuda.Stream()
def run(mode):
    for i in range(20):
        if mode == "linear":
            rq.linear(x, qs[i % 4], out=out, workspace=ws, stream=st, pdl=True, check=False)
        else:
            rq.linear_planes(pl, qs[i % 4], out, workspace=ws, stream=st, pdl=True)
for mode in ("linear", "planes_precomputed"):
    with torch.cuda.stream(st):
        run(mode)
    st.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        run(mode)
    with torch.cuda.stream(st):
        for _ in range(3):
            gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(10):
            gr.replay()
        e1.record(st)
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 200
    print(f"W{BITS} B={B} {mode:18s}: {us:6.2f} us per launch, {qs[0].weight_bytes / us / 1e3:7.1f} GB/s", flush=True)
