import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
os.environ["RTNQ_WGEMM_DEBUG"] = os.environ.get("DBG", "4")
B = int(os.environ.get("B", "16"))
# warm the clocks
a = torch.randn(8192, 8192, device="cuda")
for _ in range(50): a @ a
for name, n, k in [("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]:
    w = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    q = rq.quantize_pack(w, 4, 128)
    x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    ws = rq.Workspace(device="cuda")
    for _ in range(3): rq.linear(x, q, workspace=ws)
    torch.cuda.synchronize()
    ts = ws.buf[32768:32768 + 296 * 64].view(torch.int64).view(-1, 8).cpu().numpy().astype(np.float64)
    ts = ts[ts[:, 0] > 0]
    t0 = ts[:, 0].min()
    r = ts.copy(); r[:, [0,1,2,3,4,6]] = (ts[:, [0,1,2,3,4,6]] - t0) / 1000.0
    last = r[:, 5] > 0
    print(f"{name} B={B}: CTAs={len(r)} first-data med={np.median(r[:,1]):.2f} last-stage[med,max]=({np.median(r[:,2]):.2f},{r[:,2].max():.2f}) "
          f"published[med,max]=({np.median(r[:,4]):.2f},{r[:,4].max():.2f}) end[med,max]=({np.median(r[:,3]):.2f},{r[:,3].max():.2f}) "
          f"combiners={last.sum()} combine-dur[med,max]=({np.median(r[last,6]-r[last,4]):.2f},{(r[last,6]-r[last,4]).max():.2f}) us")
    o = np.argsort(-r[:, 3])[:5]
    for i in o: print("   slow CTA", i, np.round(r[i], 2))
