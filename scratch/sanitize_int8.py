"""Small W4 / W8 linears through every int8-kernel path (stream-K, cluster split-K with DSMEM
push, in-GEMM planes, planes kernel, token chunks) for compute-sanitizer runs."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
torch.manual_seed(0)
cases = [(4, 128, 2048, 4096, 16),   # W4 stream-K, in-GEMM planes (units >= 2048)
         (4, 128, 512, 1024, 16),    # W4 cluster split-K, planes kernel
         (4, 128, 384, 1024, 70),    # W4 token chunks (64 + 6)
         (4, 128, 1000, 2048, 1),    # W4 batch 1
         (8, 1024, 2048, 1024, 16),  # W8 per-channel stream-K
         (8, 2048, 512, 2048, 5)]    # W8 cluster split-K
for bits, g, n, k, m in cases:
    w = ((torch.rand(n, k, device="cuda") * 2 - 1) * 0.05).to(torch.bfloat16)
    q = rq.quantize_pack(w, bits, g, ragged=k % g != 0)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    ws = rq.Workspace(device="cuda")
    o1 = rq.linear(a, q, out_dtype=torch.float32, workspace=ws)
    o2 = rq.linear(a, q, out_dtype=torch.float32, workspace=ws)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    print("ok", bits, n, k, m, flush=True)
