"""Same-box comparator: vLLM's Marlin weight-only GEMM vs this library's fused
kind::i8 linear on the Llama-3.1-8B linears, W4 g128 and W8 per-channel, batch 1/4/16.
Each timing is a CUDA graph of 20 launches cycling over 4 weight copies (more than L2),
median of 5 replays; GB/s = algorithmic weight bytes (codes + f16 scales) / launch time."""
import json, os, statistics, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_15909_b200 as rq
from vllm import _custom_ops as ops
from vllm.scalar_type import scalar_types
from vllm.model_executor.layers.quantization.utils.marlin_utils import marlin_make_workspace_new
from vllm.model_executor.layers.quantization.utils.marlin_utils_test import marlin_quantize

COPIES, LAUNCHES = 4, 20
s = torch.cuda.Stream()


def time_graph(fns):
    with torch.cuda.stream(s):
        for f in fns: f()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(LAUNCHES): fns[i % len(fns)]()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s); g.replay(); e1.record(s)
        e1.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / LAUNCHES)
    return statistics.median(ts)


res = []
for bits in (4, 8):
    qt = scalar_types.uint4b8 if bits == 4 else scalar_types.uint8b128
    for name, n, k in (("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)):
        g = 128 if bits == 4 else 1 << (k - 1).bit_length()  # W8: one ragged group per row
        wbytes = n * k * bits // 8 + n * (-(-k // g)) * 2
        mar, ours = [], []
        for c in range(COPIES):
            w = torch.randn(k, n, device="cuda", dtype=torch.float16) * 0.02
            _, mq, ms, gi, si, _ = marlin_quantize(w, qt, g if bits == 4 else -1, False)
            mar.append((mq, ms, gi, si))
            ours.append(rq.quantize_pack(w.t().contiguous().to(torch.bfloat16), bits, g, ragged=bits == 8))
            del w
        mws = marlin_make_workspace_new(torch.device("cuda"))
        rws = rq.Workspace(device="cuda")
        for m in (1, 4, 16):
            a16 = torch.randn(m, k, device="cuda", dtype=torch.float16)
            ab = a16.to(torch.bfloat16)
            ob = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
            row = {"bits": bits, "linear": name, "n": n, "k": k, "batch": m}
            try:
                fm = [lambda t=t: ops.marlin_gemm(a16, None, t[0], None, t[1], None, None, None, t[2], t[3], mws,
                                                  qt, m, n, k, is_k_full=True) for t in mar]
                us = time_graph(fm)
                row["marlin_us"], row["marlin_gbs"] = round(us, 2), round(wbytes / us / 1e3, 1)
            except Exception as e:  # noqa: BLE001
                row["marlin_error"] = str(e)[:200]
            fo = [lambda q=q: rq.linear(ab, q, out=ob, workspace=rws, stream=s) for q in ours]
            us = time_graph(fo)
            row["ours_us"], row["ours_gbs"] = round(us, 2), round(wbytes / us / 1e3, 1)
            print(json.dumps(row), flush=True)
            res.append(row)
        del mar, ours
        torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/marlin_cmp.json", "w"), indent=1)
