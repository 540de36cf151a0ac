"""Near-tie rate of the W4 quantize fast path (build with RTNQ_EXTRA_CUFLAGS=-DRTNQ_QI4_COUNT via scratch/ab_build.sh cnt)."""
import os, sys, ctypes, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
L = rq.lib()
n, k = 28672, 4096
for name, w in (("uniform*0.02", ((torch.rand(n, k, device="cuda") * 2 - 1) * 0.02).to(torch.bfloat16)),
                ("normal", (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16))):
    buf = np.zeros(4, np.uint64)
    L.rtnq_qi4_count_read(buf.ctypes.data_as(ctypes.c_void_p))
    before = buf.copy()
    rq.quantize_pack(w, 4, 128, check=False); torch.cuda.synchronize()
    L.rtnq_qi4_count_read(buf.ctypes.data_as(ctypes.c_void_p))
    d = buf - before
    print(name, "warp-passes", d[0], "with near-tie", d[1], f"({100*d[1]/d[0]:.1f} %)", "near-tie lanes", d[2], f"per weight {d[2]/(n*k/16):.2e}")
