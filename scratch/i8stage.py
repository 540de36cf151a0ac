"""W8 per-stage timeline (RTNQ_WGEMM_DEBUG=128) of the last of 6 graph-launched linears, us
relative to the planes kernel's release (griddepcontrol.wait returning).
Needs a profiling build: RTNQ_KERNEL_DEBUG=1 python -c "import paper_2505_15909_b200.build as b; b.build()"."""
import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.getcwd())
os.environ["RTNQ_WGEMM_DEBUG"] = str(128 | int(os.environ.get("DBG", "0")))
import paper_2505_15909_b200 as rq
L = rq.lib()
B = int(os.environ.get("B", "16"))
buf = np.zeros(1024 * 16, np.uint64)
for name, n, k in [("qkv", 6144, 4096), ("o", 4096, 4096), ("down", 4096, 14336), ("gate_up", 28672, 4096)]:
    qs = [rq.quantize_pack((torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16), 8,
                           1 << (k - 1).bit_length(), ragged=True) for _ in range(3)]
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
    L.rtnq_i8_debug_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    d = buf.reshape(1024, 16).astype(np.float64)
    pl = d[1023, :3]
    t0 = pl[1]
    gd = d[:1023][d[:1023, 9] > 0]
    f = lambda v: (v - t0) / 1e3
    def row(nm, col, mask=None):
        v = gd[:, col] if mask is None else gd[mask, col]
        v = v[v > 0]
        if len(v): print(f"  {nm:28s} min/med/max {f(v.min()):7.2f} {f(np.median(v)):7.2f} {f(v.max()):7.2f}")
    print(f"{name} B={B} CTAs {len(gd)}: planes issue {f(pl[0]):.2f}, release 0, end {f(pl[2]):.2f}; "
          f"ideal HBM {qs[0].weight_bytes / 6.5e3 / 1e3:.2f} us")
    row("gemm start", 9); row("codes all issued", 12); row("planes wait released", 8)
    for i in range(8): row(f"stage iter {i} full", i)
    row("MMAs complete (dfull)", 13); row("leader rfull", 10); row("stored", 11)
