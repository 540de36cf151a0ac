"""W4 kernel per-CTA globaltimer stamps (RTNQ_WGEMM_DEBUG=64): start, first MMA, epilogue end, exit.
RTNQ_LIB=paper_2505_15909_b200/librtnq_b200_dbg.so B=16 python scratch/i4ends.py"""
import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.getcwd())
os.environ["RTNQ_WGEMM_DEBUG"] = "64"
import paper_2505_15909_b200 as rq
L = rq.lib()
B = int(os.environ.get("B", "16"))
for name, n, k in [(nm, int(nn), int(kk)) for nm, nn, kk in (x.split(":") for x in os.environ.get("SHAPES", "gate_up:28672:4096,o:4096:4096").split(","))]:
    w = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    q = rq.quantize_pack(w, 4, 128)
    x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    ws = rq.Workspace(device="cuda")
    for _ in range(3):
        rq.linear(x, q, workspace=ws, check=False)
    torch.cuda.synchronize()
    L.rtnq_i4_debug_read  # (stamps of the LAST launch: clear first, then one launch)
    import ctypes as C
    zero = np.zeros(1024 * 16, np.uint64)
    sym = C.c_void_p()
    torch.cuda.synchronize()
    rq.linear(x, q, workspace=ws, check=False)
    torch.cuda.synchronize()
    buf = np.zeros(1024 * 16, np.uint64)
    L.rtnq_i4_debug_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    d = buf.reshape(1024, 16).astype(np.int64)
    planes = d[1023, :3]  # planes kernel stamps: start, after wait, done
    d = d[:1023]
    live = d[:, 5] > 0
    d = d[live]
    t0 = min(d[:, 5].min(), planes[0] if planes[0] else d[:, 5].min())
    st, mma, epi, end = d[:, 5] - t0, d[:, 6] - t0, d[:, 4] - t0, d[:, 7] - t0
    pc = lambda a: f"min {a.min()/1e3:.2f} med {np.median(a)/1e3:.2f} max {a.max()/1e3:.2f}"
    print(f"{name} B={B} CTAs {live.sum()} (us): planes kernel {planes[0]-t0 if planes[0] else -1}/{(planes[2]-t0)/1e3 if planes[2] else -1:.2f}"
          f" | start {pc(st)} | first MMA {pc(mma)} | epi end {pc(epi)} | exit {pc(end)}")
