import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.getcwd())
os.environ["RTNQ_WGEMM_DEBUG"] = str(32 | int(os.environ.get("DBG", "0")))
import paper_2505_15909_b200 as rq
L = rq.lib()
B = int(os.environ.get("B", "16"))
a = torch.randn(8192, 8192, device="cuda")
for _ in range(30): a @ a
for name, n, k in [("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]:
    w = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    q = rq.quantize_pack(w, 8, 1 << (k - 1).bit_length(), ragged=True)
    x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    ws = rq.Workspace(device="cuda")
    for _ in range(3): rq.linear(x, q, workspace=ws)
    torch.cuda.synchronize()
    buf = np.zeros(1024 * 8, np.uint64)
    L.rtnq_i8_debug_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    d = buf.reshape(1024, 8).astype(np.float64); d = d[d[:, 0] > 0]
    print(f"{name}: CTAs {len(d)}  prod total {np.median(d[:,0])/1e3:.1f}k wait-empty {np.median(d[:,1])/1e3:.1f}k | "
          f"mma total {np.median(d[:,2])/1e3:.1f}k wait-full {np.median(d[:,3])/1e3:.1f}k issue {np.median(d[:,4])/1e3:.1f}k")
