"""Dequant-first (tcgen05 hi/lo GEMM) vs torch bf16 matmul (cuBLAS) at prefill sizes."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
for m, n, k in [(1024, 4096, 4096), (4096, 4096, 4096), (4096, 28672, 4096), (2048, 4096, 14336)]:
    w = ((torch.rand(n, k, device="cuda") * 2 - 1) * 0.02).to(torch.bfloat16)
    q = rq.quantize_pack(w, 4, 128)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    ws = rq.Workspace(device="cuda")
    def ours():
        rq.linear(a, q, out=out, path=rq.PATH_DEQUANT_FIRST, workspace=ws, check=False)
    def ref():
        torch.matmul(a, w.t(), out=out)
    res = []
    for name, f in (("dequant_first", ours), ("torch_bf16_mm", ref)):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record(); e1.synchronize()
        us = e0.elapsed_time(e1) * 100
        res.append(f"{name} {us:.1f}us {2 * m * n * k / us / 1e6:.0f} TF/s(1x)")
    print(f"m={m} n={n} k={k}: " + " | ".join(res), flush=True)
