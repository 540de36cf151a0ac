import sys, os, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import paper_2505_15909_b200 as rq
n, k = 520, 1024
for m in (64, 65, 80, 128, 16, 17, 33):
    w = ((torch.rand(n, k, device="cuda") * 2 - 1) * 0.05).to(torch.bfloat16)
    q = rq.quantize_pack(w, 4, 128)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    out = rq.linear(a, q, out_dtype=torch.float32)
    wd = rq.dequantize(q.codes, rq.layout(rq.NATIVE_I4), 4, n, k, 128, q.scales, rq.F16, rq.SCALES_NATIVE, torch.float32)
    ref = a.double() @ wd.double().t()
    err = ((out.double() - ref).norm(dim=1) / ref.norm(dim=1)).cpu().numpy()
    bad = np.nonzero(err > 1e-5)[0]
    print(m, "max err", err.max(), "bad rows", bad[:10], len(bad))
