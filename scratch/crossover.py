"""Fused (kind::i8 weight-only) vs dequant-first (hi+lo split + the tcgen05 dense GEMM) on the 8B gate_up and
qkv shapes, over the batch: the B200 crossover for gemm_auto (bench.cpp:69-192)."""
import json, os, statistics, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
res = {}
for bits in (4, 8):
    for name, n, k in (("qkv", 6144, 4096), ("gate_up", 28672, 4096)):
        g = 128 if bits == 4 else 4096
        q = rq.quantize_pack((torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16), bits, g)
        ws = rq.Workspace(device="cuda")
        for m in (64, 256, 512, 1024, 2048, 4096):
            a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
            out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
            row = {}
            for path, pname in ((rq.PATH_FUSED, "fused"), (rq.PATH_DEQUANT_FIRST, "dequant_first")):
                for _ in range(2): rq.linear(a, q, out=out, path=path, workspace=ws)
                torch.cuda.synchronize()
                ts = []
                for _ in range(3):
                    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(); rq.linear(a, q, out=out, path=path, workspace=ws); e1.record(); e1.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3)
                row[pname] = round(statistics.median(ts), 1)
            res[f"w{bits}_{name}_m{m}"] = row
            print(bits, name, m, row, flush=True)
            json.dump(res, open(os.environ.get("OUT", "gpurun_out/crossover.json"), "w"), indent=1)
json.dump(res, open(os.environ.get("OUT", "gpurun_out/crossover.json"), "w"), indent=1)
