#!/usr/bin/env python
"""bench.py -- W4/W8 weight-only GEMM weight-streaming throughput on B200.

Workload (BASELINE.json configs[1]; --bits 8 for configs[2]): one decode step of
Llama-3.1-8B -- every quantized linear of its 32 layers (qkv 6144x4096, o 4096x4096,
gate_up 28672x4096, down 4096x14336), W4A16 g128 (W8A16 per-channel with --bits 8), bf16
activations, one decode batch.  Under torchrun the same model runs tensor parallel
(TP=N, Megatron column/row split, the row-parallel outputs sum-allreduced over NCCL), so
every N streams the same 3.6 GB (W4) of weights per step: "scaling" is strong.
The weights never fit in L2 (126 MB), so no flush is needed between steps.
value = algorithmic weight bytes of the whole job (codes + f16 scales) / step time
(CUDA events, max over ranks).  The full decode step (RMSNorm, attention over a 256-token
KV cache, SiLU, allreduces) is timed as well and reported as decode_layer_us /
decode_us_per_token.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--bits 4|8]
                  [--model 8b|70b|405b] [--plan "explicit:0 modules:4"]
  python bench.py --impl reference     # the reference CPU gemm_fused, same metric

Prints ONE JSON line (rank 0).  DESIGN.md §5 describes every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LLAMA8B = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
LAYERS = 32
METRIC = "W4/W8 GEMM weight HBM GB/s (% of peak) at batch 1-16; decode layer us/token"


def group_for(bits):
    """W4: g128 (configs[1]); W8: per-channel = one group per row (configs[2]),
    expressed like the reference as the next power of two >= k, ragged."""
    if bits == 4:
        return lambda k: 128
    return lambda k: 1 << (k - 1).bit_length()


def weight_bytes(n, k, bits, g):
    gpr = -(-k // g)
    return n * k * bits // 8 + n * gpr * 2


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Polls SM clocks and throttle reasons through NVML during the timed region."""

    def __init__(self, index=0, period=0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self.index = period, index
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            names = {
                getattr(N, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
                getattr(N, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
                getattr(N, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
                getattr(N, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
                getattr(N, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake",
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                        r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for bit, name in names.items():
                            if r & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as e:  # NVML missing: report nothing rather than guess
            self.reasons.add(f"nvml_unavailable:{type(e).__name__}")
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def ncu_traffic(bits, batch):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"w{bits}_m{batch}")


# ---------------------------------------------------------------------------------------
def _trace(msg):
    if os.environ.get("BENCH_TRACE"):
        print(f"[bench] {msg}", file=sys.stderr, flush=True)


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2505_15909_b200 as rq
    from paper_2505_15909_b200 import tp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    bits, B = args.bits, args.batch
    shape = tp.SHAPES[args.model]
    nl = args.layers or shape.layers
    if args.plan:
        table, plan = rq.plan.resolve(args.plan, nl)
    else:  # uniform precision (configs[1] / configs[2])
        import numpy as np
        table, plan = np.full((nl, 4), bits, np.uint8), f"uniform W{bits}"
    w8pc = bits == 8 and not args.plan  # configs[2]: W8 per-channel

    # ---- this rank's tensor-parallel shard of every layer, quantized on the GPU ----
    stack = tp.TPDecodeStack(shape, table, world, rank, B, max_len=args.ctx + 1, pos=args.ctx,
                             layers=nl, seed=1234, device=dev, w8_per_channel=w8pc)
    torch.cuda.synchronize()
    dims = stack.layers[0].dims
    step_bytes_rank = stack.weight_bytes
    ws = rq.Workspace(device=dev)
    stream = torch.cuda.Stream(device=dev)

    def bufs(b):
        bf = dict(dtype=torch.bfloat16, device=dev)
        return {"x": torch.empty(b, shape.hidden, **bf).uniform_(-1, 1),
                "attn": torch.empty(b, dims.attn_cols, **bf).uniform_(-1, 1),
                "act": torch.empty(b, dims.ffn, **bf).uniform_(-1, 1),
                "qkv": torch.empty(b, dims.qkv_rows, **bf), "o": torch.empty(b, shape.hidden, **bf),
                "gu": torch.empty(b, 2 * dims.ffn, **bf), "d": torch.empty(b, shape.hidden, **bf)}

    # The weight-streaming step (the metric): every quantized linear of every layer, with
    # the row-parallel outputs (attn_out_proj, ffn_down) sum-allreduced across ranks.
    def gemm_step(bb):
        for layer in stack.layers:
            q = layer.q
            rq.linear(bb["x"], q["qkv_proj"], out=bb["qkv"], workspace=ws, stream=stream, pdl=args.pdl,
                      check=False)
            rq.linear(bb["attn"], q["attn_out_proj"], out=bb["o"], workspace=ws, stream=stream,
                      pdl=args.pdl, check=False)
            if world > 1:
                dist.all_reduce(bb["o"])
            rq.linear(bb["x"], q["ffn_up"], out=bb["gu"], workspace=ws, stream=stream, pdl=args.pdl,
                      check=False)
            rq.linear(bb["act"], q["ffn_down"], out=bb["d"], workspace=ws, stream=stream,
                      pdl=args.pdl, check=False)
            if world > 1:
                dist.all_reduce(bb["d"])

    def capture(fn):
        """CUDA graph of one step (NCCL collectives included); None if capture fails."""
        with torch.cuda.stream(stream):
            fn()
        stream.synchronize()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                fn()
            return g
        except Exception:  # noqa: BLE001 -- fall back to eager launches, reported in config
            torch.cuda.synchronize()
            return None

    def runner(g, fn):
        def run():
            with torch.cuda.stream(stream):
                if g is not None:
                    g.replay()
                else:
                    fn()
        return run

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        stream.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:  # max over ranks
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms / steps

    # total weight bytes streamed per step by the whole job (all ranks' shards)
    step_bytes = step_bytes_rank
    if world > 1:
        t = torch.tensor([float(step_bytes_rank)], device=dev, dtype=torch.float64)
        dist.all_reduce(t)
        step_bytes = int(t.item())

    main = bufs(B)
    _trace("stack built")
    graph = capture(lambda: gemm_step(main))
    _trace(f"captured (graph={graph is not None})")
    with ClockSampler(local) as clk:
        ms = timed(runner(graph, lambda: gemm_step(main)), args.steps, args.warmup)
    value = step_bytes / (ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    _trace(f"timed step {ms:.3f} ms")

    sweep = {}
    for b in args.sweep:
        if b == B:
            sweep[str(b)] = round(value, 1)
            continue
        bb = bufs(b)
        gb = capture(lambda: gemm_step(bb))
        msb = timed(runner(gb, lambda: gemm_step(bb)), max(3, args.steps // 2), args.warmup)
        sweep[str(b)] = round(step_bytes / (msb * 1e-3) / 1e9, 1)
        del gb
        _trace(f"sweep {b} done")

    # ---- e2e: pinned host activations in, host outputs back, through the public API ----
    hin = {k: torch.empty_like(main[k], device="cpu").uniform_(-1, 1).pin_memory()
           for k in ("x", "attn", "act")}
    hout = {k: torch.empty_like(main[k], device="cpu").pin_memory() for k in ("qkv", "o", "gu", "d")}
    h2d = sum(t.numel() for t in hin.values()) * 2
    d2h = sum(t.numel() for t in hout.values()) * 2

    def e2e_step():
        with torch.cuda.stream(stream):
            for k, t in hin.items():
                main[k].copy_(t, non_blocking=True)
            if graph is not None:
                graph.replay()
            else:
                gemm_step(main)
            for k, t in hout.items():
                t.copy_(main[k], non_blocking=True)

    ms_e2e = timed(e2e_step, args.steps, args.warmup)
    _trace("e2e done")
    e2e = step_bytes / (ms_e2e * 1e-3) / 1e9

    # ---- the full decode step (norms, attention over the KV cache, SiLU, allreduces) ----
    x0 = torch.empty(B, shape.hidden, dtype=torch.bfloat16, device=dev).uniform_(-1, 1)
    dgraph = capture(lambda: stack.step(x0, stream=stream, pdl=args.pdl))
    ms_dec = timed(runner(dgraph, lambda: stack.step(x0, stream=stream, pdl=args.pdl)),
                   max(3, args.steps // 2), args.warmup)

    _trace("decode step done")
    linears = nl * 4
    # ---- roofline of the dominant kernel: the largest linear (ffn_up), 20 back-to-back
    # launches over 4 weight copies (> L2) in a CUDA graph, CUDA events on its stream ----
    q_up = [l.q["ffn_up"] for l in stack.layers[:4]]
    bb_up = main

    def up_step():
        for i in range(20):
            rq.linear(bb_up["x"], q_up[i % len(q_up)], out=bb_up["gu"], workspace=ws, stream=stream,
                      pdl=args.pdl, check=False)

    g_up = capture(up_step)
    ms_up = timed(runner(g_up, up_step), max(3, args.steps // 5), args.warmup) / 20
    up_bytes = q_up[0].weight_bytes
    achieved = up_bytes / (ms_up * 1e-3) / 1e9
    step_achieved = step_bytes_rank / (ms * 1e-3) / 1e9  # one GPU's share of the whole step
    kern = {rq.NATIVE_I4: "rtnq_b200::i4::wgemm_i4_kernel", rq.NATIVE_I8: "rtnq_b200::i8::wgemm_i8_kernel",
            rq.NATIVE: "rtnq_b200::tc::wgemm_tc_kernel"}[q_up[0].layout]
    per_linear = 1 + (-(-B // 64))  # the activation-planes kernel + one GEMM per 64 tokens
    if q_up[0].layout == rq.NATIVE:
        per_linear = -(-B // 64)
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": f"u{bits} weights x bf16 activations, f32 accumulate", "data": "synthetic",
        "config": {"workload": f"{shape.name} decode step, {nl} layers x 4 quantized linears, "
                               f"W{bits}A16 {'per-channel' if w8pc else 'g128'}, decode batch {B}, "
                               f"tensor parallel TP={world}",
                   "model": shape.name, "batch": B, "layers": nl, "bits": bits,
                   "plan": plan, "group": "per-channel" if w8pc else 128,
                   "weight_bytes_per_step": step_bytes,
                   "l2": "inputs larger than L2 (weights per step >> 126 MB), no flush",
                   "parallelism": f"tp{world}" if world > 1 else "single GPU",
                   "cuda_graph": graph is not None,
                   "pct_of_hbm_peak_per_gpu": round(100 * step_achieved / peak, 1),
                   "sweep_gbs_by_batch": sweep,
                   "decode_step_ms": round(ms_dec, 4),
                   "decode_layer_us": round(ms_dec * 1e3 / nl, 2),
                   "decode_us_per_token": round(ms_dec * 1e3 / B, 2),
                   "decode_ctx_len": args.ctx,
                   "decode_cuda_graph": dgraph is not None},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4),
                     "traffic": ncu_traffic(bits, B) if world == 1 and args.model == "8b" else None,
                     "peak_source": peak_src,
                     "kernel": kern,
                     "measured_on": f"ffn_up {2 * dims.ffn}x{shape.hidden}, 20 launches in a CUDA "
                                    f"graph, CUDA events; us per launch {ms_up * 1e3:.2f} (planes kernel "
                                    f"included)",
                     "algorithmic_bytes_per_launch": up_bytes,
                     "step_average_gbs": round(step_achieved, 1)},
        "e2e": {"value": round(e2e, 1), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(ms_e2e, 4)},
        "gpu_launches": linears * per_linear * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.model == "8b":
        g_of = group_for(bits)
        line["cpu_baseline"] = cpu_baseline(args, bits=bits, B=B, g_of=g_of)
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def cpu_baseline(args, bits, B, g_of, budget_s=None):
    """Reference gemm_fused (oracle/_ref) on the host cores, one layer's 4 linears per rep."""
    import numpy as np
    import torch
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import KERNEL, Ref

    if not Ref.available():
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref/librtnq_ref.so not built"}
    import paper_2505_15909_b200 as rq
    ref = Ref()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    budget = budget_s if budget_s is not None else args.cpu_seconds
    # weights in the reference's own kernel_interleaved(16,4) layout + f32 scales,
    # produced bit-exactly by our quantize kernel (the reference's reshuffle of a
    # whole 8B layer takes ~3.5 s on 8 cores; its output is identical)
    prep = []
    for (name, n, k) in LLAMA8B:
        w = ((torch.rand(n, k, device="cuda") * 2 - 1) * (3.0 / k) ** 0.5).to(torch.bfloat16)
        q = rq.quantize_pack(w, bits, g_of(k), ragged=k % g_of(k) != 0, native=False, kernel=True,
                             scales_f32=True)
        prep.append((n, k, q.codes_kernel.cpu().numpy(), q.scales_f32.cpu().numpy()))
    rng = np.random.default_rng(0)
    acts = {k: rng.uniform(-1, 1, (B, k)).astype(np.float32) for k in (4096, 14336)}
    nbytes, t0, reps = 0, time.perf_counter(), 0
    while True:
        for n, k, kern, sc in prep:
            ref.gemm("fused", acts[k], kern, n, bits, g_of(k), sc, KERNEL, ragged=k % g_of(k) != 0)
            nbytes += weight_bytes(n, k, bits, g_of(k))
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= budget or reps >= 50:
            break
    return {"value": round(nbytes / dt / 1e9, 4), "unit": "GB/s", "cores": cores,
            "kind": "reference",
            "sample": f"{reps} x (4 Llama-3.1-8B layer linears, batch {B}) through the reference "
                      f"gemm_fused, set_threads({cores}), {dt:.1f} s"}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation, same metric/config."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import KERNEL, Ref
    bits, B = args.bits, args.batch
    g_of = group_for(bits)
    if not Ref.available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/librtnq_ref.so was not built (needs /root/reference)"}))
        return
    ref = Ref()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    rng = np.random.default_rng(0)
    prep = []
    for (name, n, k) in LLAMA8B:  # reference quantize + reshuffle, untimed (model load)
        w = (rng.uniform(-1, 1, (n, k)) * (3.0 / k) ** 0.5).astype(np.float32)
        rg = k % g_of(k) != 0
        data, sc = ref.quantize(w, bits, g_of(k), rg)
        kern = ref.reshuffle(data, n, k, bits, g_of(k), sc, 0, KERNEL, ragged=rg)
        prep.append((n, k, kern, sc))
    acts = {k: rng.uniform(-1, 1, (B, k)).astype(np.float32) for k in (4096, 14336)}
    step_bytes = sum(weight_bytes(n, k, bits, g_of(k)) for _, n, k in LLAMA8B)

    def step():
        for n, k, kern, sc in prep:
            ref.gemm("fused", acts[k], kern, n, bits, g_of(k), sc, KERNEL, ragged=k % g_of(k) != 0)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    v = step_bytes / dt / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 2), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 activations, u4/u8 codes (reference CPU)",
        "data": "synthetic",
        # the same workload as our arm's line; each reference step is a bounded sample of it
        # (one layer's 4 linears: the metric is bytes per second, so the sample is comparable)
        "config": {"workload": f"Llama-3.1-8B decode step, 32 layers x 4 quantized linears, "
                               f"W{bits}A16 {'per-channel' if bits == 8 and not args.plan else 'g128'}, "
                               f"decode batch {B}, tensor parallel TP={world}",
                   "model": "Llama-3.1-8B", "batch": B, "bits": bits,
                   "reference_sample": "each step = one layer's 4 linears through gemm_fused"},
        "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} steps x one layer's 4 linears via gemm_fused"},
        "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--bits", type=int, default=4, choices=(4, 8))
    ap.add_argument("--model", default="8b", choices=("8b", "70b", "405b"))
    ap.add_argument("--layers", type=int, default=0, help="0: all layers of the model")
    ap.add_argument("--plan", default="", help="selective-precision plan (plan.hpp grammar)")
    ap.add_argument("--ctx", type=int, default=256, help="KV-cache length of the decode step")
    ap.add_argument("--sweep", type=lambda s: [int(x) for x in s.split(",")], default=[1, 4, 16])
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pdl", dest="pdl", action="store_false",
                    help="launch the GEMMs without programmatic dependent launch")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        args.steps = min(args.steps, 5)
        args.warmup = min(args.warmup, 1)
        return run_reference(args)
    run_gpu(args)


if __name__ == "__main__":
    main()
