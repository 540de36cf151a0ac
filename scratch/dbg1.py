import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
torch.manual_seed(0)
def err(n, k, bits=4, g=128, m=1, ctas=None):
    if ctas: os.environ["RTNQ_WGEMM_CTAS"] = str(ctas)
    else: os.environ.pop("RTNQ_WGEMM_CTAS", None)
    w = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    q = rq.quantize_pack(w, bits, g)
    wd = rq.dequantize(q.codes, rq.layout(rq.NATIVE), bits, n, k, g, q.scales, rq.F16, rq.SCALES_NATIVE, torch.float32)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    ws = rq.Workspace(device="cuda")
    out = rq.linear(a, q, out_dtype=torch.float32, workspace=ws)
    ref = a.double() @ wd.double().t()
    e = ((out.double() - ref).norm() / ref.norm()).item()
    bad = ((out.double()-ref).abs() > 1e-3*ref.abs().max()).nonzero()
    rows = sorted(set(bad[:,1].tolist()))
    print(f"n={n} k={k} bits={bits} m={m} ctas={ctas}: err={e:.3e} badcols={len(rows)} first={rows[:8]} last={rows[-4:] if rows else []}", flush=True)
for n in (4096, 8192, 12288, 16384, 20480, 28672):
    err(n, 4096)
for k in (256, 1024, 2048):
    err(28672, k)
for c in (1, 16, 100, 148, 296):
    err(28672, 4096, ctas=c)
os.environ["RTNQ_NO_PDL"] = "1"
err(28672, 4096)
