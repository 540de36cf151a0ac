"""int8 W8 path timeline (RTNQ_WGEMM_DEBUG=64): planes kernel and per-CTA GEMM stamps (us).
Needs a profiling build: RTNQ_KERNEL_DEBUG=1 python -c "import paper_2505_15909_b200.build as b; b.build()"."""
import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.getcwd())
os.environ["RTNQ_WGEMM_DEBUG"] = str(64 | int(os.environ.get("DBG", "0")))
import paper_2505_15909_b200 as rq
L = rq.lib()
B = int(os.environ.get("B", "16")); BITS = int(os.environ.get("BITS", "8"))
a = torch.randn(8192, 8192, device="cuda")
for _ in range(30): a @ a
buf = np.zeros(1024 * 16, np.uint64)
for name, n, k in [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]:
    qs = [rq.quantize_pack((torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16), BITS,
                           (1 << (k - 1).bit_length()) if BITS == 8 else 128, ragged=BITS == 8) for _ in range(3)]
    x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    ws = rq.Workspace(device="cuda")
    out = torch.empty(B, n, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.Stream()
    for i in range(3): rq.linear(x, qs[i % 3], out=out, workspace=ws, pdl=True)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for i in range(6): rq.linear(x, qs[i % 3], out=out, workspace=ws, pdl=True, stream=st)
    g.replay(); torch.cuda.synchronize()
    buf[:] = 0
    (L.rtnq_i8_debug_read if BITS == 8 else L.rtnq_i4_debug_read)(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    d = buf.reshape(1024, 16).astype(np.float64)
    pl = d[1023, :3]
    g = d[:1023][d[:1023, 5] > 0]
    t0 = pl[1]
    f = lambda v: (v - t0) / 1e3
    print(f"{name} B={B} CTAs {len(g)}: planes issue {f(pl[0]):.2f} go 0 end {f(pl[2]):.2f} | "
          f"gemm start min/med/max {f(g[:,5].min()):.2f}/{f(np.median(g[:,5])):.2f}/{f(g[:,5].max()):.2f} "
          f"first-full med/max {f(np.median(g[:,6])):.2f}/{f(g[:,6].max()):.2f} "
          f"end min/med/max {f(g[:,7].min()):.2f}/{f(np.median(g[:,7])):.2f}/{f(g[:,7].max()):.2f}  "
          f"ideal {qs[0].weight_bytes/6.5e3/1e3:.2f}")
    print("     cycles: ldtm %.0f  math %.0f  arrive %.0f (median)" % tuple(np.median(g[:, 12 + i]) for i in range(3)))
    for i, nm in [x for x in enumerate(["prod_end", "mma_end", "epi_psum(last seg)", "epi_dfull(last seg)", "epi_done"] + [""] * 3 + ["seg start", "seg cor loaded", "seg acc done", "seg stored"]) if x[1]]:
        print(f"     {nm:26s} min/med/max {f(g[:,i].min()):.2f}/{f(np.median(g[:,i])):.2f}/{f(g[:,i].max()):.2f}")
