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

# round 2 paths: W8 group-128 on the group kernel, two epilogue warpgroups (m >= 16), the tcgen05
# dequant-first GEMM, the drop-in group-parallel exact kernel, peer-memory row split + reduce
for bits, g, n, k, m in [(8, 128, 512, 1024, 16), (4, 128, 1024, 2048, 32)]:
    w = ((torch.rand(n, k, device="cuda") * 2 - 1) * 0.05).to(torch.bfloat16)
    q = rq.quantize_pack(w, bits, g)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    ws = rq.Workspace(device="cuda")
    o1 = rq.linear(a, q, out_dtype=torch.float32, workspace=ws)
    o2 = rq.linear(a, q, out_dtype=torch.float32, workspace=ws)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    print("ok group kernel", bits, n, k, m, flush=True)
w = ((torch.rand(200, 1000, device="cuda") * 2 - 1) * 0.05).to(torch.bfloat16)
q = rq.quantize_pack(w, 4, 128, ragged=True)
a = torch.empty(130, 1000, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
rq.linear(a, q, out_dtype=torch.bfloat16, path=rq.PATH_DEQUANT_FIRST)
torch.cuda.synchronize()
print("ok dense_tc", flush=True)
import numpy as np
wn = (np.random.default_rng(0).standard_normal((40, 2048)) * 0.05).astype(np.float32)
data, sc = rq.quantize_tensor(wn, 4, 128)
klay = rq.layout(rq.KERNEL_INTERLEAVED)
kern = rq.reshuffle(data, rq.layout(), klay, 4, 40, 2048)
rq.gemm_fused(np.ones((3, 2048), np.float32), kern, klay, 4, 40, 128, sc)
print("ok exact ki16", flush=True)
from paper_2505_15909_b200.peer import PeerGroup, slot_cap
qs = [rq.quantize_pack(((torch.rand(256, 1024, device="cuda") * 2 - 1) * 0.05).to(torch.bfloat16), 4, 128)
      for _ in range(2)]
groups = PeerGroup.single_process(2, slot_cap(16 * 256))
for rnd in range(3):
    xs = [torch.empty(5, 1024, device="cuda").uniform_(-1, 1).to(torch.bfloat16) for _ in range(2)]
    for r in range(2):
        groups[r].linear(qs[r], a=xs[r])
    outs = [torch.empty(5, 256, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    for r in range(2):
        groups[r].reduce(outs[r])
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
print("ok peer", flush=True)
