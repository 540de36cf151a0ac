"""W4 int8-MMA kernel per-role cycles (RTNQ_WGEMM_DEBUG=32), median over CTAs (kcycles).
Needs a profiling build: RTNQ_KERNEL_DEBUG=1 python -c "import paper_2505_15909_b200.build as b; b.build()"."""
import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.getcwd())
os.environ["RTNQ_WGEMM_DEBUG"] = str(32 | int(os.environ.get("DBG", "0")))
import paper_2505_15909_b200 as rq
L = rq.lib()
B = int(os.environ.get("B", "16"))
a = torch.randn(8192, 8192, device="cuda")
for _ in range(30): a @ a
names = {0: "prod wait empty", 1: "mma issue", 7: "mma lat(1024)", 2: "exp wait full", 3: "exp wait aempty", 4: "exp wait tfree",
         6: "exp work", 8: "mma wait full", 9: "mma wait afull", 10: "mma wait tfree", 11: "epi wait", 12: "epi work",
         13: "epi total", 14: "stages", 15: "epi ld (incl. sring)"}
for name, n, k in [("qkv", 6144, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]:
    w = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    q = rq.quantize_pack(w, 4, 128)
    x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    ws = rq.Workspace(device="cuda")
    for _ in range(3): rq.linear(x, q, workspace=ws)
    torch.cuda.synchronize()
    buf = np.zeros(1024 * 16, np.uint64)
    L.rtnq_i4_debug_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    d = buf.reshape(1024, 16).astype(np.float64)[:1023]
    d = d[d[:, 13] > 0]
    print(f"{name} B={B} CTAs {len(d)}: " + "  ".join(f"{v}={np.median(d[:, i]) / (1 if i == 14 else 1e3):.1f}" for i, v in names.items()))
