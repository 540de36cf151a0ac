"""The drop-in (reference-exact, f32) gemm_fused path on the device: kernel-interleaved W4 g128
codes and f32 reference-order scales, f32 activations, through rtnq_dev_linear (PATH_FUSED)."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
for n, k in [(6144, 4096), (28672, 4096), (4096, 14336)]:
    w = ((torch.rand(n, k, device="cuda") * 2 - 1) * 0.02).to(torch.bfloat16)
    q = rq.quantize_pack(w, 4, 128, native=True, kernel=True, scales_f32=True)
    for m in (1, 16):
        a = torch.empty(m, k, device="cuda").uniform_(-1, 1)
        out = torch.empty(m, n, device="cuda")
        args = (a, rq.F32, m, k, q.codes_kernel, rq.layout(rq.KERNEL_INTERLEAVED), 4, n, 128, 0,
                q.scales_f32, rq.F32, rq.SCALES_REF, out, rq.F32)
        rq.linear_raw(*args, path=rq.PATH_FUSED)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            rq.linear_raw(*args, path=rq.PATH_FUSED)
        e1.record(); e1.synchronize()
        us = e0.elapsed_time(e1) * 200
        wb = n * k // 2 + n * (k // 128) * 4
        print(f"exact gemm_fused n={n} k={k} m={m}: {us:.1f} us, {wb / us / 1e3:.1f} GB/s of weights", flush=True)
