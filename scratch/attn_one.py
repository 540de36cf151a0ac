"""One decode_attention launch (B, CTX from env) for ncu."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
B = int(os.environ.get("B", "16")); ctx = int(os.environ.get("CTX", "256")); hq, hkv, d = 32, 8, 128
bf = dict(dtype=torch.bfloat16, device="cuda")
qkv = torch.randn(B, (hq + 2 * hkv) * d, **bf); kc = torch.randn(B, ctx + 1, hkv, d, **bf); vc = torch.randn_like(kc)
att = torch.empty(B, hq * d, **bf)
for _ in range(3):
    rq.decode_attention(qkv, kc, vc, att, hq, hkv, ctx)
torch.cuda.synchronize()
