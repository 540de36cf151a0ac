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

The same JSON line carries sub-records measured in the same run: "w8" (configs[2], W8A16
per-channel step, batch sweep 1-64 and its ffn_up roofline), "quantize" (the model-load
quantize-and-pack kernel on the 8B gate_up, W4 and W8), "llama70b" (configs[3]: the 80-layer
70B stack with plan "explicit:0 modules:4" at TP = N) and "llama405b_tp8_rank_shard"
(configs[4]: one TP=8 rank's 405B shards, batch 1-32, on one GPU).

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


def base_config(args, world, shape, nl, bits, plan, w8pc, B, step_bytes):
    """The workload description, identical for both arms (--impl ours / reference)."""
    return {"workload": f"{shape.name} decode step, {nl} layers x 4 quantized linears, "
                        f"W{bits}A16 {'per-channel' if w8pc else 'g128'}, decode batch {B}, "
                        f"tensor parallel TP={world}",
            "model": shape.name, "batch": B, "layers": nl, "bits": bits, "plan": plan,
            "group": "per-channel" if w8pc else 128, "weight_bytes_per_step": step_bytes,
            "l2": "inputs larger than L2 (weights per step >> 126 MB), no flush",
            "parallelism": f"tp{world}" if world > 1 else "single GPU"}


class Ctx:
    """Per-process GPU bench state: stream, workspace, timing helpers."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.args = torch, dist, args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        self.dev = torch.device("cuda", self.local)
        self.stream = torch.cuda.Stream(device=self.dev)
        self.capture_errors = []

    def capture(self, fn):
        """CUDA graph of one step (NCCL collectives included); None if capture fails -- the
        failure is reported in the JSON line ("capture_errors") and on stderr."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            fn()
        self.stream.synchronize()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                fn()
            return g
        except Exception as e:  # noqa: BLE001 -- eager launches instead, reported
            torch.cuda.synchronize()
            msg = f"{type(e).__name__}: {str(e).splitlines()[0][:200] if str(e) else ''}"
            self.capture_errors.append(msg)
            print(f"[bench] WARNING: CUDA-graph capture failed, timing eager launches: {msg}",
                  file=sys.stderr, flush=True)
            return None

    def runner(self, g, fn):
        def run():
            with self.torch.cuda.stream(self.stream):
                if g is not None:
                    g.replay()
                else:
                    fn()
        return run

    def timed(self, fn, steps, warmup):
        torch, dist = self.torch, self.dist
        for _ in range(warmup):
            fn()
        self.stream.synchronize()
        if self.world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        for _ in range(steps):
            fn()
        e1.record(self.stream)
        e1.synchronize()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if self.world > 1:  # max over ranks
            t = torch.tensor([ms], device=self.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms / steps

    def allsum(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([float(x)], device=self.dev, dtype=self.torch.float64)
        self.dist.all_reduce(t)
        return t.item()


def measure(cx, shape, table, B, nl, w8pc, sweep, steps, warmup, *, sim_world=None, e2e=False,
            decode=True, roofline=True, ctx_len=256):
    """Build this rank's shard stack and time its weight-streaming step (every quantized linear
    of every layer, row-parallel outputs allreduced), the batch sweep, optionally the e2e step
    (host buffers), the full decode step and the dominant kernel (ffn_up)."""
    import paper_2505_15909_b200 as rq
    from paper_2505_15909_b200 import tp
    torch, dist, args = cx.torch, cx.dist, cx.args
    world = sim_world or cx.world
    rank = 0 if sim_world else cx.rank
    stack = tp.TPDecodeStack(shape, table, world, rank, B, max_len=ctx_len + 1, pos=ctx_len,
                             layers=nl, seed=1234, device=cx.dev, w8_per_channel=w8pc,
                             collectives=sim_world is None)
    torch.cuda.synchronize()
    dims = stack.layers[0].dims
    ws = rq.Workspace(device=cx.dev)
    stream = cx.stream
    coll = sim_world is None and cx.world > 1

    def bufs(b):
        bf = dict(dtype=torch.bfloat16, device=cx.dev)
        return {"x": torch.empty(b, shape.hidden, **bf).uniform_(-1, 1),
                "attn": torch.empty(b, dims.attn_cols, **bf).uniform_(-1, 1),
                "act": torch.empty(b, dims.ffn, **bf).uniform_(-1, 1),
                "qkv": torch.empty(b, dims.qkv_rows, **bf), "o": torch.empty(b, shape.hidden, **bf),
                "gu": torch.empty(b, 2 * dims.ffn, **bf), "d": torch.empty(b, shape.hidden, **bf)}

    def gemm_step(bb):
        for layer in stack.layers:
            q = layer.q
            kw = dict(workspace=ws, stream=stream, pdl=args.pdl, check=False)
            rq.linear(bb["x"], q["qkv_proj"], out=bb["qkv"], **kw)
            rq.linear(bb["attn"], q["attn_out_proj"], out=bb["o"], **kw)
            if coll:
                dist.all_reduce(bb["o"])
            rq.linear(bb["x"], q["ffn_up"], out=bb["gu"], **kw)
            rq.linear(bb["act"], q["ffn_down"], out=bb["d"], **kw)
            if coll:
                dist.all_reduce(bb["d"])

    step_bytes_rank = stack.weight_bytes
    step_bytes = int(cx.allsum(step_bytes_rank)) if not sim_world else step_bytes_rank
    main = bufs(B)
    graph = cx.capture(lambda: gemm_step(main))
    with ClockSampler(cx.local) as clk:
        ms = cx.timed(cx.runner(graph, lambda: gemm_step(main)), steps, warmup)
    out = {"ms_per_step": round(ms, 4), "gbs": round(step_bytes / (ms * 1e-3) / 1e9, 1),
           "step_bytes": step_bytes, "step_bytes_rank": step_bytes_rank,
           "gbs_per_gpu": round(step_bytes_rank / (ms * 1e-3) / 1e9, 1), "cuda_graph": graph is not None,
           "clocks": clk.summary(), "launches_per_step": nl * 4 * (1 + -(-B // 64))}
    sw = {}
    for b in sweep:
        if b == B:
            sw[str(b)] = out["gbs"]
            continue
        bb = bufs(b)
        gb = cx.capture(lambda: gemm_step(bb))
        msb = cx.timed(cx.runner(gb, lambda: gemm_step(bb)), max(3, steps // 2), warmup)
        sw[str(b)] = round(step_bytes / (msb * 1e-3) / 1e9, 1)
        del gb
    out["sweep_gbs_by_batch"] = sw
    if e2e:  # pinned host activations in, host outputs back, through the public API
        hin = {k: torch.empty_like(main[k], device="cpu").uniform_(-1, 1).pin_memory()
               for k in ("x", "attn", "act")}
        hout = {k: torch.empty_like(main[k], device="cpu").pin_memory() for k in ("qkv", "o", "gu", "d")}

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

        ms_e2e = cx.timed(e2e_step, steps, warmup)
        out["e2e"] = {"value": round(step_bytes / (ms_e2e * 1e-3) / 1e9, 1), "unit": "GB/s",
                      "h2d_bytes_per_step": sum(t.numel() for t in hin.values()) * 2,
                      "d2h_bytes_per_step": sum(t.numel() for t in hout.values()) * 2,
                      "ms_per_step": round(ms_e2e, 4)}
    if decode:  # the full decode step (norms, attention over the KV cache, SiLU, allreduces)
        x0 = torch.empty(B, shape.hidden, dtype=torch.bfloat16, device=cx.dev).uniform_(-1, 1)
        dgraph = cx.capture(lambda: stack.step(x0, stream=stream, pdl=args.pdl))
        ms_dec = cx.timed(cx.runner(dgraph, lambda: stack.step(x0, stream=stream, pdl=args.pdl)),
                          max(3, steps // 2), warmup)
        stack.check(stream)  # no non-finite activation flagged during the timed steps
        out.update({"decode_step_ms": round(ms_dec, 4), "decode_layer_us": round(ms_dec * 1e3 / nl, 2),
                    "decode_us_per_token": round(ms_dec * 1e3 / B, 2), "decode_ctx_len": ctx_len,
                    "decode_cuda_graph": dgraph is not None})
    if roofline:  # the dominant kernel: ffn_up, 20 launches over 4 weight copies (> L2), graph
        q_up = [l.q["ffn_up"] for l in stack.layers[:4]]

        def up_step():
            for i in range(20):
                rq.linear(main["x"], q_up[i % len(q_up)], out=main["gu"], workspace=ws, stream=stream,
                          pdl=args.pdl, check=False)

        g_up = cx.capture(up_step)
        ms_up = cx.timed(cx.runner(g_up, up_step), max(3, steps // 5), warmup) / 20
        up_bytes = q_up[0].weight_bytes
        peak, peak_src = peaks()
        achieved = up_bytes / (ms_up * 1e-3) / 1e9
        kern = {rq.NATIVE_I4: "rtnq_b200::i4::wgemm_i4_kernel", rq.NATIVE_I8: "rtnq_b200::i8::wgemm_i8_kernel",
                rq.NATIVE: "rtnq_b200::tc::wgemm_tc_kernel"}[q_up[0].layout]
        out["roofline"] = {
            "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "peak_source": peak_src, "kernel": kern,
            "measured_on": f"ffn_up {2 * dims.ffn}x{shape.hidden}, 20 launches in a CUDA graph, CUDA "
                           f"events on the launch stream; us per launch {ms_up * 1e3:.2f} (planes "
                           f"kernel included)",
            "algorithmic_bytes_per_launch": up_bytes,
            "step_average_gbs": round(step_bytes_rank / (ms * 1e-3) / 1e9, 1)}
    del stack
    torch.cuda.empty_cache()
    return out


def quantize_record(cx, bits, n=28672, k=4096, reps=10):
    """The model-load pass (rtnq_dev_quantize_pack_ex) on the 8B gate_up weight: bf16 in, the
    kernel's operand layout + native f16 scales out, CUDA events.  Algorithmic bytes = 2 B read
    + bits/8 B written per weight + the scales."""
    import paper_2505_15909_b200 as rq
    torch = cx.torch
    g = 128 if bits == 4 else 1 << (k - 1).bit_length()
    ws = [((torch.rand(n, k, device=cx.dev) * 2 - 1) * 0.02).to(torch.bfloat16) for _ in range(2)]
    with torch.cuda.stream(cx.stream):
        q = rq.quantize_pack(ws[0], bits, g, k % g != 0, stream=cx.stream)
    nbytes = n * k * 2 + n * k * bits // 8 + n * (-(-k // g)) * 2

    def run():
        for i in range(reps):
            rq.quantize_pack(ws[i % 2], bits, g, k % g != 0, check=False, stream=cx.stream)

    ms = cx.timed(lambda: cx.runner(None, run)(), 3, 1) / reps
    peak, _ = peaks()
    del ws, q
    return {"shape": f"{n}x{k}", "layout": "NATIVE_I4" if bits == 4 else "NATIVE_I8",
            "us": round(ms * 1e3, 2), "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1),
            "frac": round(nbytes / (ms * 1e-3) / 1e9 / peak, 4), "algorithmic_bytes": nbytes,
            "note": "one quantize_pack call (allocations + the fused kernel), 2 weight copies alternating"}


def exact_record(cx, reps=5):
    """The drop-in path a reference consumer gets (rtnq::gemm_fused: f32 activations, the
    reference's kernel_interleaved(16, 4) codes and f32 scales, bit-identical to the reference):
    the four Llama-3.1-8B layer linears at W4 g128, batch 1 and 16, CUDA events."""
    import paper_2505_15909_b200 as rq
    torch = cx.torch
    qs, nbytes = [], 0
    with torch.cuda.stream(cx.stream):  # inputs made on the stream that uses them
        for n, k in ((6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)):
            w = ((torch.rand(n, k, device=cx.dev) * 2 - 1) * 0.02).to(torch.bfloat16)
            qs.append((n, k, rq.quantize_pack(w, 4, 128, native=True, kernel=True, scales_f32=True,
                                              stream=cx.stream)))
            nbytes += n * k // 2 + n * (-(-k // 128)) * 2
    out = {}
    for m in (1, 16):
        args = []
        for n, k, q in qs:
            with torch.cuda.stream(cx.stream):
                a = torch.empty(m, k, device=cx.dev).uniform_(-1, 1)
                o = torch.empty(m, n, device=cx.dev)
            args.append((a, rq.F32, m, k, q.codes_kernel, rq.layout(rq.KERNEL_INTERLEAVED), 4, n, 128, 0,
                         q.scales_f32, rq.F32, rq.SCALES_REF, o, rq.F32))

        def run():
            for x in args:
                rq.linear_raw(*x, path=rq.PATH_FUSED, stream=cx.stream)

        ms = cx.timed(lambda: cx.runner(None, run)(), reps, 1)
        out[f"m{m}"] = {"us_per_layer": round(ms * 1e3, 1), "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1)}
    return {"workload": "one Llama-3.1-8B layer (qkv, o, gate_up, down) W4 g128 through the drop-in gemm_fused "
                        "(f32 activations, kernel_interleaved(16,4) codes, bit-identical to the reference)",
            "weight_bytes_per_layer": nbytes, **out}


def attention_record(cx, launches=10, reps=5):
    """GQA decode attention (32 query / 8 KV heads, head dim 128, RoPE, KV append) over a bf16
    cache: KV bytes per second per (batch, context), `launches` back to back in a CUDA graph."""
    import paper_2505_15909_b200 as rq
    torch = cx.torch
    hq, hkv, d = 32, 8, 128
    out = {}
    for b, ctx in ((16, 256), (16, 4096), (32, 4096)):
        with torch.cuda.stream(cx.stream):
            qkv = torch.randn(b, (hq + 2 * hkv) * d, device=cx.dev).to(torch.bfloat16)
            kc = torch.randn(b, ctx + 1, hkv, d, device=cx.dev).to(torch.bfloat16)
            vc = torch.randn_like(kc)
            att = torch.empty(b, hq * d, device=cx.dev, dtype=torch.bfloat16)
            ws = rq.Workspace(0, cx.dev)  # sized by the first call

        def run():
            for _ in range(launches):
                rq.decode_attention(qkv, kc, vc, att, hq, hkv, ctx, stream=cx.stream, workspace=ws)

        run()
        cx.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cx.stream):
            run()
        us = cx.timed(cx.runner(g, None), reps, 1) * 1e3 / launches
        kv = 2 * b * (ctx + 1) * hkv * d * 2
        out[f"b{b}_ctx{ctx}"] = {"us": round(us, 2), "kv_gbs": round(kv / (us * 1e-6) / 1e9, 1)}
        del kc, vc
    return {"workload": "Llama-3.1-8B GQA decode attention (32/8 heads, d 128, RoPE + KV append), bf16 KV cache, "
                        "CUDA graph of back-to-back launches", **out}


def run_gpu(args):
    import numpy as np

    import paper_2505_15909_b200 as rq
    from paper_2505_15909_b200 import tp
    cx = Ctx(args)
    world, rank = cx.world, cx.rank
    bits, B = args.bits, args.batch
    shape = tp.SHAPES[args.model]
    nl = args.layers or shape.layers
    if args.plan:
        table, plan = rq.plan.resolve(args.plan, nl)
    else:  # uniform precision (configs[1] / configs[2])
        table, plan = np.full((nl, 4), bits, np.uint8), f"uniform W{bits}"
    w8pc = bits == 8 and not args.plan  # configs[2]: W8 per-channel
    steps, warmup = args.steps, args.warmup
    sub_steps = max(5, steps // 5)

    main = measure(cx, shape, table, B, nl, w8pc, args.sweep, steps, warmup, e2e=True)
    _trace(f"headline step {main['ms_per_step']} ms")
    peak, peak_src = peaks()
    value = main["gbs"]
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": main["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": f"u{bits} weights x bf16 activations, f32 accumulate", "data": "synthetic",
        "config": base_config(args, world, shape, nl, bits, plan, w8pc, B, main["step_bytes"]),
        "roofline": dict(main["roofline"], traffic=ncu_traffic(bits, B) if world == 1 and args.model == "8b" else None),
        "e2e": main["e2e"],
        "gpu_launches": main["launches_per_step"] * steps,
        "clocks": main["clocks"],
        "details": {k: main[k] for k in ("cuda_graph", "sweep_gbs_by_batch", "decode_step_ms", "decode_layer_us",
                                         "decode_us_per_token", "decode_ctx_len", "decode_cuda_graph",
                                         "gbs_per_gpu")},
    }
    line["details"]["pct_of_hbm_peak_per_gpu"] = round(100 * main["gbs_per_gpu"] / peak, 1)
    if not args.headline_only and args.model == "8b" and not args.plan:
        # the other half of the metric: W8A16 per-channel (configs[2]) or W4 (configs[1])
        other = 8 if bits == 4 else 4
        t2 = np.full((nl, 4), other, np.uint8)
        m2 = measure(cx, shape, t2, B, nl, other == 8, [1, 4, 16, 32, 64] if other == 8 else [1, 4, 16],
                     sub_steps, warmup, decode=False)
        line[f"w{other}"] = {"value": m2["gbs"], "unit": "GB/s", "ms_per_step": m2["ms_per_step"],
                             "workload": base_config(args, world, shape, nl, other, f"uniform W{other}",
                                                     other == 8, B, m2["step_bytes"])["workload"],
                             "sweep_gbs_by_batch": m2["sweep_gbs_by_batch"], "roofline": m2["roofline"],
                             "cuda_graph": m2["cuda_graph"]}
        _trace("second bit width done")
        if world == 1:
            line["quantize"] = {f"w{b}": quantize_record(cx, b) for b in (4, 8)}
            line["dropin_exact"] = exact_record(cx)
            line["decode_attention"] = attention_record(cx)
        # configs[3]: Llama-3.1-70B, 80 layers, W4 + layer-0 down_proj W8, at TP = world
        t70, p70 = rq.plan.resolve("explicit:0 modules:4", tp.LLAMA_70B.layers)
        m70 = measure(cx, tp.LLAMA_70B, t70, 1, tp.LLAMA_70B.layers, False, [1, 4, 16], sub_steps, warmup,
                      roofline=False)
        line["llama70b"] = {
            "workload": f"Llama-3.1-70B decode step, 80 layers, plan '{p70}' (W4 g128 + layer-0 ffn_down W8 g128), "
                        f"TP={world}, batch 1",
            "ms_per_token_batch1": m70["ms_per_step"], "gbs": m70["gbs"], "sweep_gbs_by_batch": m70["sweep_gbs_by_batch"],
            "weight_bytes_per_step": m70["step_bytes"], "floor_ms_at_peak": round(m70["step_bytes_rank"] / peak / 1e6, 4),
            "decode_step_ms_batch1": m70["decode_step_ms"], "decode_layer_us": m70["decode_layer_us"],
            "cuda_graph": m70["cuda_graph"]}
        _trace("70b done")
        if world == 1:
            # configs[4]: one rank's shard stack of Llama-3.1-405B at TP=8, batch 1-32 (the per-GPU
            # work of that configuration; its two allreduces per layer are not on this GPU)
            t405 = np.full((tp.LLAMA_405B.layers, 4), 4, np.uint8)
            m405 = measure(cx, tp.LLAMA_405B, t405, 1, tp.LLAMA_405B.layers, False, [1, 4, 16, 32], sub_steps,
                           warmup, sim_world=8, roofline=False, decode=True)
            line["llama405b_tp8_rank_shard"] = {
                "workload": "Llama-3.1-405B, 126 layers, W4 g128, the TP=8 rank-0 shards (qkv 2304x16384, o "
                            "16384x2048, gate_up 13312x16384, down 16384x6656) on one GPU, allreduces excluded",
                "ms_per_step_batch1": m405["ms_per_step"], "gbs": m405["gbs"],
                "sweep_gbs_by_batch": m405["sweep_gbs_by_batch"], "weight_bytes_per_step": m405["step_bytes"],
                "decode_step_ms_batch1": m405["decode_step_ms"], "cuda_graph": m405["cuda_graph"]}
            _trace("405b done")
    if cx.capture_errors:
        line["capture_errors"] = cx.capture_errors
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.model == "8b":
        line["cpu_baseline"] = cpu_baseline(args, bits=bits, B=B, g_of=group_for(bits))
    if world > 1:
        cx.dist.destroy_process_group()
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
    """--impl reference: the reference's own CPU gemm_fused (oracle/_ref, built from the
    unmodified sources), all host threads, same metric / unit / config as our arm.  Each step
    is a bounded sample of the workload: one layer's 4 linears (bytes per second is
    size-independent, so the sample is comparable)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import KERNEL, Ref

    from paper_2505_15909_b200 import tp
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
    layer_bytes = sum(weight_bytes(n, k, bits, g_of(k)) for _, n, k in LLAMA8B)
    shape = tp.SHAPES[args.model]
    nl = args.layers or shape.layers
    w8pc = bits == 8 and not args.plan
    plan = args.plan or f"uniform W{bits}"

    def step():
        for n, k, kern, sc in prep:
            ref.gemm("fused", acts[k], kern, n, bits, g_of(k), sc, KERNEL, ragged=k % g_of(k) != 0)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    v = layer_bytes / dt / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3 * nl, 2), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 activations, u4/u8 codes (reference CPU)",
        "data": "synthetic",
        "config": base_config(args, world, shape, nl, bits, plan, w8pc, B, layer_bytes * nl),
        "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                         "sample": f"each of the {args.steps} steps = one Llama-3.1-8B layer's 4 linears "
                                   f"(batch {B}) through the reference gemm_fused, set_threads({cores}); "
                                   f"ms_per_step scaled to {nl} layers"},
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
    ap.add_argument("--headline-only", action="store_true",
                    help="skip the W8/W4 sub-record, the quantize pass and the 70B / 405B configs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    run_gpu(args)


if __name__ == "__main__":
    main()
