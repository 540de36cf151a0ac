"""Correctness at the full 405B ffn_up shape (W8 per-channel and W4 g128), batch 16: the fused
int8 path against an f64 reference built from the dequantized weights."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
n, k, m = 106496, 16384, 16
torch.manual_seed(0)
for bits in (8, 4):
    w = ((torch.rand(n, k, device="cuda") * 2 - 1) * 0.02).to(torch.bfloat16)
    g = 16384 if bits == 8 else 128
    q = rq.quantize_pack(w, bits, g, ragged=bits == 8, scales_f16=True, row_major=True)
    del w
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    y = rq.linear(x, q, out_dtype=torch.float32)
    wd = rq.dequantize(q.codes_row_major, rq.layout(rq.ROW_MAJOR), bits, n, k, g, q.scales_f16, rq.F16, rq.SCALES_REF)  # the f16 scales the kernels use
    ref = torch.zeros(m, n, dtype=torch.float64, device="cuda")
    for i in range(0, n, 8192):
        ref[:, i:i + 8192] = x.double() @ wd[i:i + 8192].double().t()
    err = ((y.double() - ref).norm() / ref.norm()).item()
    print(f"W{bits} {n}x{k} m={m}: rel Frobenius error {err:.3e}", flush=True)
    del q, wd, ref, y
    torch.cuda.empty_cache()
