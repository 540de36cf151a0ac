"""Selective-precision accuracy methodology on the GPU linears.

The reference's toy decoder (toy.cpp:91-209) and eval harness (eval.cpp:147-243) with every
linear on this library's device kernels:

- weights and inputs come from the reference's pinned PRNG (xoshiro256** seeded by
  splitmix64, rng.hpp:29-66; make_toy_weight / make_toy_input, toy.cpp:155-185);
- a quantized candidate is ``quantize_model`` (store.cpp:424-446): per (layer, module) bits
  from the plan (plan.resolve), RTN quantize-and-pack on the GPU into the reference's
  interleaved kernel layout with f32 scales;
- the forward (toy.cpp:91-117) runs its linears through ``rtnq_dev_linear`` with
  ``PATH_AUTO`` (gemm_auto: the reference-exact fused kernel below the threshold, dequant-first
  above it) for a quantized model, and ``rtnq_dev_gemm_float`` (gemm_float) for the float
  reference; RMSNorm, attention and SiLU follow toy.cpp's precision (double accumulation,
  one f32 rounding) as torch ops on the same device;
- ``compare``, ``horizontal_sweep``, ``vertical_sweep`` and ``sweep_to_csv`` follow
  eval.cpp:52-243 (KL and logit deviation in double).

Parity: tests/test_eval.py against the reference's own sweep CSV and compare reports
(tests/golden/toy_sweeps.csv, toy_compare.txt; tests/golden/make_sweep_golden.py).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import plan as _plan

MODULES = (1, 2, 3, 4)  # ModuleId qkv_proj, attn_out_proj, ffn_up, ffn_down
_M64 = (1 << 64) - 1


@dataclass(frozen=True)
class ToyConfig:
    """ToyTransformerConfig (toy.hpp:16-30) and the toy group size (kToyGroupSize = 64)."""
    layers: int = 8
    dim: int = 64
    heads: int = 4
    ffn: int = 256
    seq: int = 32
    seed: int = 0
    group: int = 64

    def shape(self, module: int):  # toy_shape, toy.cpp:75-83
        return {1: (3 * self.dim, self.dim), 2: (self.dim, self.dim), 3: (2 * self.ffn, self.dim),
                4: (self.dim, self.ffn)}[module]


# ---- pinned PRNG (rng.hpp:29-66) ------------------------------------------------------------

def _units(seed: int, stream: int, n: int) -> np.ndarray:
    """n Xoshiro256ss(seed, stream).next_unit() values: top 24 bits -> [-1, 1) in f32."""
    z = (seed ^ ((stream * 0x9E3779B97F4A7C15) & _M64)) & _M64
    s = []
    for _ in range(4):  # SplitMix64
        z = (z + 0x9E3779B97F4A7C15) & _M64
        x = z
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
        s.append(x ^ (x >> 31))
    s0, s1, s2, s3 = s
    u24 = np.empty(n, np.uint32)
    for i in range(n):
        r = (s1 * 5) & _M64
        r = ((((r << 7) | (r >> 57)) & _M64) * 9) & _M64
        t = (s1 << 17) & _M64
        s2 ^= s0
        s3 ^= s1
        s1 ^= s2
        s0 ^= s3
        s2 ^= t
        s3 = ((s3 << 45) | (s3 >> 19)) & _M64
        u24[i] = r >> 40
    # float(u24) * 2^-23 - 1 in f32: both steps exact
    return (u24.astype(np.float32) * np.float32(1.0 / 8388608.0) - np.float32(1.0)).astype(np.float32)


def toy_weight(cfg: ToyConfig, layer: int, module: int) -> np.ndarray:
    """make_toy_weight (toy.cpp:155-166): amp * next_unit(), amp = f32(sqrt(3 / cols))."""
    rows, cols = cfg.shape(module)
    amp = np.float32(math.sqrt(3.0 / cols))
    return (amp * _units(cfg.seed, layer * 4 + (module - 1), rows * cols)).reshape(rows, cols)


def toy_input(cfg: ToyConfig, index: int) -> np.ndarray:
    """make_toy_input (toy.cpp:177-185): seq x dim next_unit() values, stream (1 << 32) | index."""
    return _units(cfg.seed, (1 << 32) | index, cfg.seq * cfg.dim).reshape(cfg.seq, cfg.dim)


# ---- models ---------------------------------------------------------------------------------

class FloatModel:
    """The float reference: f32 weights on the device, layer-major, module order 1..4."""

    def __init__(self, cfg: ToyConfig, device="cuda"):
        import torch
        self.cfg = cfg
        self.w = {(l, m): torch.from_numpy(toy_weight(cfg, l, m)).to(device)
                  for l in range(cfg.layers) for m in MODULES}


class QuantModel:
    """quantize_model (store.cpp:424-446): every tensor RTN-quantized on the GPU at the plan's
    bits for its (layer, module), reference interleaved layout, f32 scales."""

    def __init__(self, model: FloatModel, plan_text: str):
        import paper_2505_15909_b200 as rq
        cfg = model.cfg
        self.cfg = cfg
        self.table, self.plan_text = _plan.resolve(plan_text, cfg.layers)
        self.q = {}
        for (l, m), w in model.w.items():
            bits = int(self.table[l][m - 1])
            self.q[(l, m)] = rq.quantize_pack(w, bits, cfg.group, native=False, kernel=True,
                                              scales_f32=True)

    def dequantized(self, layer: int, module: int):
        """dequantize_tensor (quant.cpp:143-171) on the device: code * scale in f32."""
        import paper_2505_15909_b200 as rq
        qw = self.q[(layer, module)]
        return rq.dequantize(qw.codes_kernel, rq.layout(rq.KERNEL_INTERLEAVED), qw.bits, qw.rows,
                             qw.cols, qw.group, qw.scales_f32, rq.F32, rq.SCALES_REF)

    def effective_bits(self) -> float:
        return effective_bits(self.table, self.cfg)


def effective_bits(table, cfg: ToyConfig) -> float:
    """Stored weight bits per parameter, scales excluded (plan.cpp:226-251)."""
    rows = [cfg.shape(m)[0] for m in MODULES]
    cols = [cfg.shape(m)[1] for m in MODULES]
    return _plan.effective_bits(table, rows, cols, cfg.group)


# ---- forward (toy.cpp:17-117) ---------------------------------------------------------------

def _linear_quant(qw, x, threshold):
    import torch

    import paper_2505_15909_b200 as rq
    m, k = x.shape
    out = torch.empty(m, qw.rows, dtype=torch.float32, device=x.device)
    lay = rq.layout(rq.KERNEL_INTERLEAVED)
    wsb = rq.lib().rtnq_dev_linear_workspace_bytes(m, qw.rows, k, qw.bits, qw.group, rq.PATH_AUTO, lay)
    ws = torch.empty(max(int(wsb), 1), dtype=torch.uint8, device=x.device)
    rq.linear_raw(x, rq.F32, m, k, qw.codes_kernel, lay, qw.bits, qw.rows, qw.group, qw.ragged,
                  qw.scales_f32, rq.F32, rq.SCALES_REF, out, rq.F32, path=rq.PATH_AUTO,
                  threshold=threshold, ws=ws, ws_bytes=int(wsb))
    return out


def _linear_float(w, x, block):
    import torch

    import paper_2505_15909_b200 as rq
    m, k = x.shape
    out = torch.empty(m, w.shape[0], dtype=torch.float32, device=x.device)
    rq._check(rq.lib().rtnq_dev_gemm_float(rq._ptr(x), m, k, rq._ptr(w), w.shape[0], block,
                                           rq._ptr(out), rq._stream(None)))
    return out


def _rmsnorm(x):
    import torch
    ss = (x.double() * x.double()).sum(1, keepdim=True)
    inv = (1.0 / torch.sqrt(ss / x.shape[1] + 1e-5)).float()
    return (x * inv).contiguous()


def _attention(qkv, heads, causal=True):
    import torch
    s, d = qkv.shape[0], qkv.shape[1] // 3
    dh = d // heads
    q, k, v = (qkv[:, i * d:(i + 1) * d].double().reshape(s, heads, dh).transpose(0, 1) for i in range(3))
    score = torch.matmul(q, k.transpose(1, 2)) * (1.0 / math.sqrt(dh))
    if causal:
        mask = torch.ones(s, s, dtype=torch.bool, device=qkv.device).triu(1)
        score = score.masked_fill(mask, -math.inf)
    p = torch.exp(score - score.amax(-1, keepdim=True))
    out = torch.matmul(p, v) / p.sum(-1, keepdim=True)
    return out.float().transpose(0, 1).reshape(s, d).contiguous()


def toy_forward(model, x, threshold: int = 1024, causal: bool = True):
    """forward_impl (toy.cpp:91-117) for a FloatModel (gemm_float) or QuantModel (gemm_auto)."""
    import torch
    cfg = model.cfg
    x = torch.as_tensor(x).to("cuda", torch.float32).contiguous().clone()
    if x.dim() != 2 or x.shape[1] != cfg.dim or x.shape[0] < 1:
        from .errors import ShapeError
        raise ShapeError("forward input must be rows x model width")
    if isinstance(model, QuantModel):
        lin = lambda l, m, a: _linear_quant(model.q[(l, m)], a, threshold)  # noqa: E731
    else:
        lin = lambda l, m, a: _linear_float(model.w[(l, m)], a, cfg.group)  # noqa: E731
    f = cfg.ffn
    for layer in range(cfg.layers):
        qkv = lin(layer, 1, _rmsnorm(x))
        x = x + lin(layer, 2, _attention(qkv, cfg.heads, causal))
        ug = lin(layer, 3, _rmsnorm(x))
        z = ug[:, :f].double()
        gated = ((z / (1.0 + torch.exp(-z))).float() * ug[:, f:]).contiguous()
        x = x + lin(layer, 4, gated)
    return x


# ---- eval (eval.cpp:52-243) -----------------------------------------------------------------

def _logit_metrics(yr, yc):
    """accumulate_logit_metrics (eval.cpp:52-80): -> (max |dev|, sum of per-row KL, rows)."""
    import torch
    a, b = yr.double(), yc.double()
    dev = (a - b).abs().max().item()
    lse_a = a.amax(1, keepdim=True) + torch.log(torch.exp(a - a.amax(1, keepdim=True)).sum(1, keepdim=True))
    lse_b = b.amax(1, keepdim=True) + torch.log(torch.exp(b - b.amax(1, keepdim=True)).sum(1, keepdim=True))
    log_p = a - lse_a
    kl = (torch.exp(log_p) * (log_p - (b - lse_b))).sum(1).clamp_min(0.0)
    return dev, kl.sum().item(), a.shape[0]


@dataclass
class TensorError:
    layer: int
    module: int
    max_abs: float
    mse: float
    rel_frobenius: float


@dataclass
class ErrorReport:
    plan_text: str
    effective_bits: float
    tensors: list
    max_logit_dev: float
    mean_kl: float


def compare(ref: FloatModel, cand, inputs, threshold: int = 1024) -> ErrorReport:
    """compare (eval.cpp:147-182): weight-space error per tensor, output-space KL / deviation."""
    tensors = []
    for l in range(ref.cfg.layers):
        for m in MODULES:
            w = ref.w[(l, m)].double()
            c = (cand.dequantized(l, m) if isinstance(cand, QuantModel) else cand.w[(l, m)]).double()
            d = w - c
            ss, rs = (d * d).sum().item(), (w * w).sum().item()
            tensors.append(TensorError(l, m, d.abs().max().item(), ss / w.numel(),
                                       math.sqrt(ss / rs) if rs > 0 else 0.0))
    dev, kl, rows = 0.0, 0.0, 0
    for x in inputs:
        yr = toy_forward(ref, x)
        yc = toy_forward(cand, x, threshold)
        d, k, r = _logit_metrics(yr, yc)
        dev, kl, rows = max(dev, d), kl + k, rows + r
    quant = isinstance(cand, QuantModel)
    return ErrorReport(cand.plan_text if quant else "", cand.effective_bits() if quant else 32.0,
                       tensors, dev, kl / rows if rows else 0.0)


@dataclass
class SweepRow:
    strategy: str
    label: str
    effective_bits: float
    max_logit_dev: float
    mean_kl: float


def _sweep(model: FloatModel, inputs, points, threshold):
    """SweepContext (eval.cpp:112-143): the float forward once per input, then each plan."""
    refs = [toy_forward(model, x) for x in inputs]
    rows = []
    for strategy, label, text in points:
        qm = QuantModel(model, text)
        dev, kl, n = 0.0, 0.0, 0
        for x, yr in zip(inputs, refs):
            d, k, r = _logit_metrics(yr, toy_forward(qm, x, threshold))
            dev, kl, n = max(dev, d), kl + k, n + r
        rows.append(SweepRow(strategy, label, qm.effective_bits(), dev, kl / n if n else 0.0))
    return rows


def mask_label(mask: int) -> str:
    """mask_label (eval.cpp:184-193): '1+3', or 'none'."""
    return "+".join(str(m) for m in MODULES if mask & (1 << (m - 1))) or "none"


def horizontal_sweep(model: FloatModel, kind: str, inputs, threshold: int = 1024):
    """horizontal_sweep (eval.cpp:195-208): X = 0..layers layers of block `kind` at 8 bits."""
    if kind not in ("first", "middle", "last"):
        from .errors import InvalidInputError
        raise InvalidInputError("sweeps cover the first/middle/last strategies only")
    pts = [(kind, str(x), f"{kind}:{x}") for x in range(model.cfg.layers + 1)]
    return _sweep(model, inputs, pts, threshold)


def vertical_sweep(model: FloatModel, inputs, threshold: int = 1024):
    """vertical_sweep (eval.cpp:210-224): all 16 module masks across every layer."""
    pts = [("modules", mask_label(mask), f"first:{model.cfg.layers} modules:{mask_label(mask)}")
           for mask in range(16)]
    return _sweep(model, inputs, pts, threshold)


def sweep_to_csv(rows) -> str:
    """sweep_to_csv (eval.cpp:226-243): %.9g numbers."""
    out = "strategy,x_or_mask,effective_bits,max_logit_dev,mean_kl\n"
    for r in rows:
        out += f"{r.strategy},{r.label},{r.effective_bits:.9g},{r.max_logit_dev:.9g},{r.mean_kl:.9g}\n"
    return out
