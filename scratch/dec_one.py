"""One decode attention (batch B, ctx 256, 8B shapes) + silu_mul with planes, for ncu."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
B = int(os.environ.get("B", "16")); h, hq, hkv, d, ctx, f = 4096, 32, 8, 128, 256, 14336
bf = dict(dtype=torch.bfloat16, device="cuda")
qkv = torch.randn(B, (hq + 2 * hkv) * d, **bf); kc = torch.randn(B, ctx + 1, hkv, d, **bf); vc = torch.randn_like(kc)
att = torch.empty(B, hq * d, **bf); gu = torch.randn(B, 2 * f, **bf); act = torch.empty(B, f, **bf)
pa = rq.Planes(B, f)
for _ in range(3):
    rq.decode_attention(qkv, kc, vc, att, hq, hkv, ctx)
    rq.silu_mul(gu, act, planes=pa)
torch.cuda.synchronize()
