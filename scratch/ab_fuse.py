import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2505_15909_b200 as rq
from paper_2505_15909_b200 import tp
B = int(os.environ.get("B", "16")); NL = 8
for bits in (4, 8):
    table = np.full((NL, 4), bits, np.uint8)
    for fuse in (False, True, False, True):
        st = tp.TPDecodeStack(tp.LLAMA_8B, table, 1, 0, B, layers=NL, seed=1, w8_per_channel=bits == 8, fuse_planes=fuse)
        s = torch.cuda.Stream(); x0 = torch.randn(B, 4096, device="cuda").to(torch.bfloat16)
        with torch.cuda.stream(s): st.step(x0, stream=s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s): st.step(x0, stream=s)
        ts = []
        for _ in range(7):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s); g.replay(); e1.record(s)
            e1.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / NL)
        print(f"W{bits} fuse={fuse}: {statistics.median(ts[2:]):.2f} us/layer", flush=True)
        del st, g
        torch.cuda.empty_cache()
