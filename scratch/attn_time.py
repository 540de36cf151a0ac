import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
hq, hkv, d = 32, 8, 128
s = torch.cuda.Stream()
res = []
for B in (1, 16, 32):
    for ctx in (256, 1024, 4096):
        bf = dict(dtype=torch.bfloat16, device="cuda")
        qkv = torch.randn(B, (hq + 2 * hkv) * d, **bf); kc = torch.randn(B, ctx + 1, hkv, d, **bf); vc = torch.randn_like(kc)
        att = torch.empty(B, hq * d, **bf)
        fn = lambda: rq.decode_attention(qkv, kc, vc, att, hq, hkv, ctx, stream=s)
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
        res.append(f"B{B}c{ctx} {statistics.median(ts):.1f}")
print(os.environ.get("TAG", ""), " | ".join(res), flush=True)
