"""Per-launch time of each Llama-3.1-8B linear (W4 g128 / W8 per-channel) at batch B through rq.linear,
20 launches over 4 weight copies in a CUDA graph."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
B = int(os.environ.get("B", "16")); BITS = int(os.environ.get("BITS", "4"))
st = torch.cuda.Stream()
ws = rq.Workspace(device="cuda")
res = []
SHAPES = {"8b": [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)],
          # one TP=8 rank's shards of Llama-3.1-405B / the 70B at TP = 1
          "405b_tp8": [("qkv", 2304, 16384), ("o", 16384, 2048), ("gate_up", 13312, 16384), ("down", 16384, 6656)],
          "70b": [("qkv", 10240, 8192), ("o", 8192, 8192), ("gate_up", 57344, 8192), ("down", 8192, 28672)]}
for name, n, k in SHAPES[os.environ.get("MODEL", "8b")]:
    g = 128 if BITS == 4 or os.environ.get("W8G128") else 1 << (k - 1).bit_length()
    NAT = os.environ.get("NATIVE") == "1" or None
    qs = [rq.quantize_pack(((torch.rand(n, k, device="cuda") * 2 - 1) * 0.02).to(torch.bfloat16), BITS, g, k % g != 0, native=NAT) for _ in range(4)]
    x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    out = torch.empty(B, n, device="cuda", dtype=torch.bfloat16)
    def run():
        for i in range(20):
            rq.linear(x, qs[i % 4], out=out, workspace=ws, stream=st, pdl=True, check=False)
    with torch.cuda.stream(st):
        run()
    st.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        run()
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
    res.append(f"{name} {us:.2f}us {qs[0].weight_bytes / us / 1e3:.0f}GB/s")
print(f"{os.environ.get('TAG','')} W{BITS} B={B}: " + " | ".join(res), flush=True)
