import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
B = int(os.environ.get("B", "16")); h, hq, hkv, d, ctx, f = 4096, 32, 8, 128, 256, 14336
bf = dict(dtype=torch.bfloat16, device="cuda")
x = torch.randn(B, h, **bf); w = torch.ones(h, **bf); y = torch.empty_like(x); delta = torch.randn(B, h, **bf)
qkv = torch.randn(B, (hq + 2 * hkv) * d, **bf); kc = torch.randn(B, ctx + 1, hkv, d, **bf); vc = torch.randn_like(kc)
att = torch.empty(B, hq * d, **bf); gu = torch.randn(B, 2 * f, **bf); act = torch.empty(B, f, **bf)
py = rq.Planes(B, h); pa = rq.Planes(B, f)
s = torch.cuda.Stream()
ops = {
    "add_rmsnorm": lambda: rq.add_rmsnorm(x, w, y, delta=delta, stream=s),
    "add_rmsnorm+planes": lambda: rq.add_rmsnorm(x, w, y, delta=delta, stream=s, planes=py),
    "act_planes(4096)": lambda: rq.act_planes(y, py, stream=s),
    "attention(ctx 256)": lambda: rq.decode_attention(qkv, kc, vc, att, hq, hkv, ctx, stream=s),
    "silu_mul": lambda: rq.silu_mul(gu, act, stream=s),
    "silu_mul+planes": lambda: rq.silu_mul(gu, act, stream=s, planes=pa),
    "act_planes(14336)": lambda: rq.act_planes(act, pa, stream=s),
}
for name, fn in ops.items():
    with torch.cuda.stream(s): fn()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20): fn()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s); g.replay(); e1.record(s)
        e1.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / 20)
    print(f"{name:22s} {statistics.median(ts):6.2f} us")
