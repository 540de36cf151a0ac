"""Quantize-and-pack kernels on the 8B gate_up (profiling driver for ncu)."""
import sys, torch
sys.path.insert(0, '.')
import paper_2505_15909_b200 as rq
n, k = 28672, 4096
w = ((torch.rand(n, k, device="cuda") * 2 - 1) * 0.02).to(torch.bfloat16)
for it in range(3):
    q4 = rq.quantize_pack(w, 4, 128)
    q8 = rq.quantize_pack(w, 8, 4096)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for bits, g in ((4, 128), (8, 4096)):
    e0.record()
    for it in range(10):
        rq.quantize_pack(w, bits, g, check=False)
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 100
    nb = n * k * 2 + n * k * bits // 8 + n * (k // g) * 2
    print(f"W{bits}: {us:.1f} us per quantize_pack, {nb / us / 1e3:.0f} GB/s")
