"""RTNQ_WGEMM_DEBUG=32 instrumentation: per-CTA stamps and blocked cycles per role/barrier."""
import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.getcwd())
os.environ["RTNQ_WGEMM_DEBUG"] = str(32 | int(os.environ.get("DBG", "0")))
import paper_2505_15909_b200 as rq
L = rq.lib()
B = int(os.environ.get("B", "16")); bits = int(os.environ.get("BITS", "4"))
a = torch.randn(8192, 8192, device="cuda")
for _ in range(30): a @ a
names = ["start", "tmem", "prod_end", "mma_end", "deq_end", "epi_seg_end", "combine_end"]
waits = {8: "prod wait empty", 12: "prod total", 20: "mma wait full", 21: "mma wait a_full",
         22: "mma wait d_empty", 23: "mma issue+commit", 24: "mma total", 32: "deq0 wait full", 33: "deq0 wait a_empty", 34: "deq0 lds+alu", 35: "deq0 sttm+wait",
         36: "deq0 total", 60: "isolated MMA cycles/unit", 44: "epi0 wait d_full", 45: "epi0 wait full", 48: "epi0 total(last seg)"}
buf = np.zeros(1024 * 64, np.uint64)
for name, n, k in [x for x in [("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)] if x[0] in os.environ.get("ONLY", "o,gate_up,down")]:
    w = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    g = 128 if bits == 4 else 1 << (k - 1).bit_length()
    q = rq.quantize_pack(w, bits, g, ragged=k % g != 0)
    x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    ws = rq.Workspace(nbytes=1 << 22, device="cuda")
    for _ in range(3): rq.linear(x, q, workspace=ws)
    torch.cuda.synchronize()
    L.rtnq_wgemm_debug_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes), 1)
    rq.linear(x, q, workspace=ws)
    torch.cuda.synchronize()
    L.rtnq_wgemm_debug_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes), 1)
    d = buf.reshape(1024, 64).astype(np.float64)
    d = d[d[:, 0] > 0]
    t0 = d[:, 0].min()
    r = (d[:, :7] - t0) / 1000.0
    print(f"{name} W{bits} B={B} CTAs={len(r)} (us from first CTA start; median / max)")
    for i, nm in enumerate(names):
        print(f"   {nm:12s} {np.median(r[:, i]):8.2f} {r[:, i].max():8.2f}")
    for sl, nm in waits.items():
        print(f"   {nm:24s} kcyc median {np.median(d[:, sl])/1e3:8.2f} max {d[:, sl].max()/1e3:8.2f}")
