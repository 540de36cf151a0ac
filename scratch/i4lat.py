"""W4 steady-state stage latency (RTNQ_WGEMM_DEBUG=256): issue -> full (seen by the expansion),
-> expansion done, and MMA full pass, for stage iterations 8..11 of gate_up (us, median over CTAs).
Needs a profiling build: RTNQ_KERNEL_DEBUG=1 python -c "import paper_2505_15909_b200.build as b; b.build()"."""
import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.getcwd())
os.environ["RTNQ_WGEMM_DEBUG"] = str(256 | int(os.environ.get("DBG", "0")))
import paper_2505_15909_b200 as rq
L = rq.lib()
for B in (1, 16):
    for name, n, k in [("gate_up", 28672, 4096), ("down", 4096, 14336)]:
        qs = [rq.quantize_pack((torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16), 4, 128) for _ in range(3)]
        x = torch.empty(B, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
        ws = rq.Workspace(device="cuda"); out = torch.empty(B, n, device="cuda", dtype=torch.bfloat16)
        st = torch.cuda.Stream()
        for i in range(3): rq.linear(x, qs[i % 3], out=out, workspace=ws, pdl=True)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(6): rq.linear(x, qs[i % 3], out=out, workspace=ws, pdl=True, stream=st)
        g.replay(); torch.cuda.synchronize()
        buf = np.zeros(1024 * 16, np.uint64)
        L.rtnq_i4_debug_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
        d = buf.reshape(1024, 16).astype(np.float64)[:1023]
        d = d[(d[:, 0] > 0) & (d[:, 7] > 0)]
        lat = (d[:, 4:8] - d[:, 0:4]) / 1e3
        hold = (d[:, 8:12] - d[:, 4:8]) / 1e3
        mma = (d[:, 12:16] - d[:, 4:8]) / 1e3
        per = (d[:, 3] - d[:, 0]) / 3e3
        print(f"{name} B={B} CTAs {len(d)}: issue->full {np.median(lat):.2f} us, full->exp done {np.median(hold):.2f}, "
              f"full->MMA pass {np.median(mma):.2f}, issue period {np.median(per):.2f} us/stage", flush=True)
