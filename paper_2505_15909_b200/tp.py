"""Tensor-parallel decode stack over the rtnq kernels.

Megatron-style sharding of a Llama-3.1 decoder layer across ``world`` ranks (one
process per GPU, ``torch.distributed`` NCCL for the two sum-allreduces per layer):

* column split (no communication) -- ``qkv_proj`` by heads (each rank owns
  ``heads/world`` query heads and ``kv_heads/world`` KV heads) and ``ffn_up`` (the
  fused [gate | up] rows of toy.cpp:108-112: each rank keeps the matching slices of
  both halves);
* row split -- ``attn_out_proj`` and ``ffn_down`` along K, at quantization-group
  boundaries, each rank producing a partial [batch x hidden] that is summed by an
  allreduce.

Weights are quantized BEFORE sharding: each rank quantizes the full module
weight once (rq.quantize_pack, the same kernel as TP=1), then keeps its rows (column split)
or its K slice (row split) of the row-major codes and of the scales (``shard_quantized``) and
relays them out into the kernels' layout.  For group-128 weights this equals quantizing the
shard (rows quantize independently, quant.cpp:118-136, and the K split falls on group
boundaries); for W8 per-channel (one group per full row, configs[2]) it does NOT -- a row-split
shard keeps the full row's scale, which only the full row's absmax gives (tests/test_tp.py).

The per-(layer, module) bit width comes from the selective-precision table
(plan.resolve, plan.cpp:189-224): the same table on every rank picks the W4 or W8
kernel for each linear.

The sharding functions work on numpy or torch tensors and need no GPU; the layer and
stack need CUDA (and librtnq_b200.so) -- there is no CPU fallback.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

MODULES = ("qkv_proj", "attn_out_proj", "ffn_up", "ffn_down")  # ModuleId 1..4 (types.hpp:46-51)


@dataclass(frozen=True)
class LlamaShape:
    name: str
    hidden: int
    heads: int
    kv_heads: int
    head_dim: int
    ffn: int
    layers: int
    rope_theta: float = 500000.0
    eps: float = 1e-5


LLAMA_8B = LlamaShape("Llama-3.1-8B", 4096, 32, 8, 128, 14336, 32)
LLAMA_70B = LlamaShape("Llama-3.1-70B", 8192, 64, 8, 128, 28672, 80)
LLAMA_405B = LlamaShape("Llama-3.1-405B", 16384, 128, 8, 128, 53248, 126)
SHAPES = {"8b": LLAMA_8B, "70b": LLAMA_70B, "405b": LLAMA_405B}


@dataclass(frozen=True)
class LocalDims:
    """One rank's share of a layer."""
    hq: int       # query heads
    hkv: int      # kv heads
    ffn: int      # ffn columns (per half of gate_up)
    qkv_rows: int
    attn_cols: int

    def module_shape(self, shape: LlamaShape, module: str):
        """(N, K) of this rank's weight for `module` (rows = output channels)."""
        return {"qkv_proj": (self.qkv_rows, shape.hidden),
                "attn_out_proj": (shape.hidden, self.attn_cols),
                "ffn_up": (2 * self.ffn, shape.hidden),
                "ffn_down": (shape.hidden, self.ffn)}[module]


def local_dims(shape: LlamaShape, world: int, group: int = 128) -> LocalDims:
    if shape.heads % world or shape.kv_heads % world or shape.ffn % world:
        raise ValueError(f"{shape.name}: heads/kv_heads/ffn must divide by TP={world}")
    hq, hkv, f = shape.heads // world, shape.kv_heads // world, shape.ffn // world
    for k in (hq * shape.head_dim, f):  # row-split K extents must be whole groups
        if k % group:
            raise ValueError(f"row-split width {k} is not a multiple of the group size {group}")
    return LocalDims(hq, hkv, f, (hq + 2 * hkv) * shape.head_dim, hq * shape.head_dim)


# ---- sharding of full (unsharded) weights ------------------------------------------------

def shard_qkv(w, shape: LlamaShape, rank: int, world: int):
    """Rows of this rank's heads from the full [ (H + 2 Hkv) D, hidden ] QKV weight."""
    d, hq, hkv = shape.head_dim, shape.heads // world, shape.kv_heads // world
    q0 = rank * hq * d
    k0 = shape.heads * d + rank * hkv * d
    v0 = (shape.heads + shape.kv_heads) * d + rank * hkv * d
    parts = [w[q0:q0 + hq * d], w[k0:k0 + hkv * d], w[v0:v0 + hkv * d]]
    return _cat(parts)


def shard_gate_up(w, shape: LlamaShape, rank: int, world: int):
    """Matching gate and up slices of the fused [gate | up] rows (toy.cpp:108-112)."""
    f = shape.ffn // world
    return _cat([w[rank * f:(rank + 1) * f], w[shape.ffn + rank * f:shape.ffn + (rank + 1) * f]])


def shard_cols(w, rank: int, world: int):
    """K-split (row-parallel linear): columns [rank*K/world, (rank+1)*K/world)."""
    k = w.shape[1] // world
    return w[:, rank * k:(rank + 1) * k]


def shard_module(w, module: str, shape: LlamaShape, rank: int, world: int):
    if module == "qkv_proj":
        return shard_qkv(w, shape, rank, world)
    if module == "ffn_up":
        return shard_gate_up(w, shape, rank, world)
    return shard_cols(w, rank, world)


def shard_quantized(codes_rm, scales, module: str, shape: LlamaShape, rank: int, world: int,
                    bits: int, group: int):
    """This rank's shard of a weight quantized in full (quantize-before-shard).

    ``codes_rm`` are the full weight's row-major packed codes viewed as [rows, cols*bits/8]
    bytes (QuantTensor::data, quant.cpp:139), ``scales`` its [rows, groups_per_row] scales
    (any dtype; reference order, quant.hpp:33); ``group`` the full weight's group size.
    Returns (codes [n, k*bits/8], scales [n, gpr'], k, group', ragged') of the shard:
    column splits keep whole rows; row splits keep a K slice of every row and the scales of
    the groups in it -- for one group per row (W8 per-channel) that is the FULL row's scale,
    and the shard is again one (ragged) group per row."""
    rows, nbytes = codes_rm.shape
    k_full = nbytes * 8 // bits
    if module in ("qkv_proj", "ffn_up"):
        return (shard_module(codes_rm, module, shape, rank, world),
                shard_module(scales, module, shape, rank, world), k_full, group,
                k_full % group != 0)
    k = k_full // world
    b0, b1 = rank * k * bits // 8, (rank + 1) * k * bits // 8
    c = codes_rm[:, b0:b1]
    c = np.ascontiguousarray(c) if isinstance(c, np.ndarray) else c.contiguous()
    if group >= k_full:  # one group per row: the shard keeps the full-row scale
        g = 1 << (k - 1).bit_length()
        s = scales[:, :1]
        s = np.ascontiguousarray(s) if isinstance(s, np.ndarray) else s.contiguous()
        return c, s, k, g, k % g != 0
    if k % group:
        raise ValueError(f"row-split width {k} is not a multiple of the group size {group}")
    s = scales[:, rank * (k // group):(rank + 1) * (k // group)]
    s = np.ascontiguousarray(s) if isinstance(s, np.ndarray) else s.contiguous()
    return c, s, k, group, False


def _cat(parts):
    if isinstance(parts[0], np.ndarray):
        return np.ascontiguousarray(np.concatenate(parts, axis=0))
    import torch
    return torch.cat(parts, dim=0).contiguous()


def module_bits(table, layer: int):
    """Per-module bit widths of one layer from a plan table (plan.resolve)."""
    return {m: int(table[layer][i]) for i, m in enumerate(MODULES)}


def group_for(bits: int, k: int, group: int = 128, w8_per_channel: bool = False) -> int:
    """W8 per-channel (configs[2]) is one group per row: next power of two >= k, ragged."""
    if bits == 8 and w8_per_channel:
        return 1 << (k - 1).bit_length()
    return group


# ---- the layer (CUDA) ------------------------------------------------------------------------

def quantize_module(w, module: str, shape: LlamaShape, rank: int, world: int, bits: int,
                    group: int, stream=None):
    """Quantize the FULL module weight ``w`` (bf16/f16/f32 CUDA, [rows, cols]) on the GPU and
    return this rank's shard as a QuantWeight in the layout its kernel reads."""
    import paper_2505_15909_b200 as rq
    n, k = w.shape
    ragged = k % group != 0
    if world == 1:
        return rq.quantize_pack(w.contiguous(), bits, group, ragged=ragged, check=False,
                                stream=stream)
    q = rq.quantize_pack(w.contiguous(), bits, group, ragged=ragged, native=False,
                         row_major=True, scales_f16=True, check=False, stream=stream)
    codes = q.codes_row_major.view(n, k * bits // 8)
    c, s, ks, gs, rg = shard_quantized(codes, q.scales_f16, module, shape, rank, world, bits,
                                       group)
    return rq.from_row_major(c.reshape(-1), s.contiguous(), c.shape[0], ks, bits, gs, rg,
                             stream=stream)


class TPDecodeLayer:
    """One rank's shard of a decoder layer, all weights quantized on the GPU.

    ``weights`` (optional) maps module -> full bf16 CUDA weight; without it the rank's
    shards are drawn from a seeded generator (synthetic weights of the same shapes).
    The forward pass is split at the two allreduce points so a caller can either run
    NCCL between the halves (``TPDecodeStack``) or simulate TP on one GPU by summing
    the partials of several rank objects (tests).
    """

    def __init__(self, shape: LlamaShape, layer: int, world: int, rank: int, bits: dict,
                 batch: int, max_len: int, pos: int, group: int = 128, weights=None, seed=0,
                 device="cuda", w8_per_channel=False, fuse_planes=True):
        import torch

        import paper_2505_15909_b200 as rq
        self.shape, self.layer, self.world, self.rank = shape, layer, world, rank
        self.dims = local_dims(shape, world, group)
        self.batch, self.max_len, self.pos = batch, max_len, pos
        self.bits = bits
        dev = torch.device(device)
        self.q = {}
        full = local_dims(shape, 1, group)
        for mi, m in enumerate(MODULES):
            n, k = full.module_shape(shape, m)
            if weights is not None:
                w = weights[m]
            else:  # synthetic full weight, the same on every rank (seeded by layer and module)
                gen = torch.Generator(device=dev).manual_seed(seed * 1000003 + layer * 101 + mi)
                w = ((torch.rand(n, k, device=dev, generator=gen) * 2 - 1) * (3.0 / k) ** 0.5
                     ).to(torch.bfloat16)
            self.q[m] = quantize_module(w, m, shape, rank, world, bits[m],
                                        group_for(bits[m], k, group, w8_per_channel))
            del w
        h, d = shape.hidden, shape.head_dim
        bf = dict(dtype=torch.bfloat16, device=dev)
        norm_gen = torch.Generator(device=dev).manual_seed(seed * 7919 + layer)
        self.attn_norm = (1 + 0.1 * torch.rand(h, device=dev, generator=norm_gen)).to(torch.bfloat16)
        self.ffn_norm = (1 + 0.1 * torch.rand(h, device=dev, generator=norm_gen)).to(torch.bfloat16)
        # synthetic KV cache: positions [0, pos) filled, the step appends at `pos`; drawn for all
        # KV heads (the same on every rank), each rank keeps its heads
        kv_gen = torch.Generator(device=dev).manual_seed(seed * 31 + layer * 7)
        h0, h1 = rank * self.dims.hkv, (rank + 1) * self.dims.hkv
        self.k_cache = (torch.rand(batch, max_len, shape.kv_heads, d, device=dev, generator=kv_gen)
                        - 0.5).to(torch.bfloat16)[:, :, h0:h1].contiguous()
        self.v_cache = (torch.rand(batch, max_len, shape.kv_heads, d, device=dev, generator=kv_gen)
                        - 0.5).to(torch.bfloat16)[:, :, h0:h1].contiguous()
        self.y = torch.empty(batch, h, **bf)
        self.qkv = torch.empty(batch, self.dims.qkv_rows, **bf)
        self.attn = torch.empty(batch, self.dims.attn_cols, **bf)
        self.o = torch.empty(batch, h, **bf)
        self.gu = torch.empty(batch, 2 * self.dims.ffn, **bf)
        self.act = torch.empty(batch, self.dims.ffn, **bf)
        self.d = torch.empty(batch, h, **bf)
        # int8-kernel linears read activation planes; the norms and SiLU*up emit them directly
        self.fuse = fuse_planes
        imma = (rq.NATIVE_I4, rq.NATIVE_I8)
        self.py = rq.Planes(batch, h, dev) if fuse_planes and (
            self.q["qkv_proj"].layout in imma or self.q["ffn_up"].layout in imma) else None
        # SiLU*up emits the down projection's planes too (a cluster of CTAs per token row)
        self.pa = rq.Planes(batch, self.dims.ffn, dev) if fuse_planes and self.q["ffn_down"].layout in imma \
            else None
        # the o-projection's planes: the stand-alone planes kernel (PDL-overlapped).  The attention
        # can emit them itself (decode_attention(planes=...), its last CTA per token); measured
        # 1.3 us per layer slower at batch 16 (one CTA per token computes a 4096-wide row in the
        # attention's tail), so it is opt-in: RTNQ_ATTN_PLANES=1
        self.pat = rq.Planes(batch, self.dims.attn_cols, dev) \
            if fuse_planes and self.q["attn_out_proj"].layout in imma and os.environ.get("RTNQ_ATTN_PLANES") == "1" \
            else None
        # non-finite activations (InvalidInputError, gemm.cpp:13-19) are flagged asynchronously
        # by the int8 kernels' planes pass; the stack checks the flag after a step
        self.err = None
        self.attn_ws = None  # split-merge scratch of decode_attention (the stack's, or a default)

    @property
    def weight_bytes(self):
        return sum(q.weight_bytes for q in self.q.values())

    def _linear(self, module, a, planes, out, ws, stream, pdl):
        import paper_2505_15909_b200 as rq
        q = self.q[module]
        if planes is not None and q.layout in (rq.NATIVE_I4, rq.NATIVE_I8):
            return rq.linear_planes(planes, q, out, workspace=ws, stream=stream, pdl=pdl)
        return rq.linear(a, q, out=out, workspace=ws, stream=stream, pdl=pdl, err=self.err,
                         check=False)

    def _norm(self, x, weight, delta, peer, stream):
        import paper_2505_15909_b200 as rq
        if peer is not None:  # delta = sum of the ranks' partials of the current peer round
            peer.add_rmsnorm(x, weight, self.y, eps=self.shape.eps, stream=stream, planes=self.py)
        else:
            rq.add_rmsnorm(x, weight, self.y, delta=delta, eps=self.shape.eps, stream=stream,
                           planes=self.py)

    def _row_split(self, module, a, planes, out, ws, stream, pdl, peer):
        import paper_2505_15909_b200 as rq
        if peer is None:
            return self._linear(module, a, planes, out, ws, stream, pdl)
        q = self.q[module]
        if planes is not None and q.layout in (rq.NATIVE_I4, rq.NATIVE_I8):
            peer.linear(q, planes=planes, workspace=ws, stream=stream, pdl=pdl, err=self.err)
        else:
            peer.linear(q, a=a, workspace=ws, stream=stream, pdl=pdl, err=self.err)
        return None

    def attn_half(self, x, delta, ws, stream=None, pdl=False, peer=None, peer_in=False):
        """x += delta; y = rmsnorm(x); qkv; attention; o = partial attn_out_proj.
        ``peer`` (peer.PeerGroup): o goes to the peers' slots instead (returns None), and with
        ``peer_in`` the delta is the previous peer round's sum."""
        import paper_2505_15909_b200 as rq
        s = self.shape
        self._norm(x, self.attn_norm, delta, peer if peer_in else None, stream)
        self._linear("qkv_proj", self.y, self.py, self.qkv, ws, stream, pdl)
        rq.decode_attention(self.qkv, self.k_cache, self.v_cache, self.attn, self.dims.hq,
                            self.dims.hkv, self.pos, s.head_dim, s.rope_theta, stream=stream,
                            workspace=self.attn_ws, planes=self.pat)
        if peer is not None:
            return self._row_split("attn_out_proj", self.attn, self.pat, self.o, ws, stream, pdl, peer)
        self._linear("attn_out_proj", self.attn, self.pat, self.o, ws, stream, pdl)
        return self.o

    def mlp_half(self, x, o_sum, ws, stream=None, pdl=False, peer=None):
        """x += o_sum; y = rmsnorm(x); gate_up; silu*up; d = partial ffn_down.
        ``peer``: o_sum is the current peer round's sum and d goes to the peers (returns None)."""
        import paper_2505_15909_b200 as rq
        self._norm(x, self.ffn_norm, o_sum, peer, stream)
        self._linear("ffn_up", self.y, self.py, self.gu, ws, stream, pdl)
        rq.silu_mul(self.gu, self.act, stream=stream, planes=self.pa)
        if peer is not None:
            return self._row_split("ffn_down", self.act, self.pa, self.d, ws, stream, pdl, peer)
        self._linear("ffn_down", self.act, self.pa, self.d, ws, stream, pdl)
        return self.d


class TPDecodeStack:
    """All layers of one rank plus the step driver (NCCL allreduce between halves)."""

    def __init__(self, shape: LlamaShape, table, world: int, rank: int, batch: int,
                 max_len: int = 257, pos: int = 256, group: int = 128, layers=None, seed=0,
                 device="cuda", w8_per_channel=False, fuse_planes=True, collectives=True,
                 peer=None):
        """collectives=False builds ONE rank's shard stack of a TP=world model without a
        process group (the per-GPU work of that configuration on a single GPU; the allreduces
        are skipped).  collectives="peer": the allreduces run over peer memory, fused into
        the row-split linears and the following add+RMSNorm (peer.py); ``peer`` is this
        rank's PeerGroup (default: built over the default process group)."""
        import torch

        import paper_2505_15909_b200 as rq
        n = shape.layers if layers is None else layers
        self.world, self.rank, self.shape = world, rank, shape
        self.collectives = collectives
        self.layers = [TPDecodeLayer(shape, li, world, rank, module_bits(table, li), batch,
                                     max_len, pos, group, seed=seed, device=device,
                                     w8_per_channel=w8_per_channel, fuse_planes=fuse_planes)
                       for li in range(n)]
        self.x = torch.zeros(batch, shape.hidden, dtype=torch.bfloat16, device=device)
        self.ws = rq.Workspace(device=device)
        self.err = rq.error_flag(device)
        self.attn_ws = rq.Workspace(device=device)  # decode attention's split-merge scratch
        for layer in self.layers:
            layer.err = self.err
            layer.attn_ws = self.attn_ws
        self.peer = peer
        if collectives == "peer" and peer is None and world > 1:
            from paper_2505_15909_b200.peer import PeerGroup, slot_cap
            self.peer = PeerGroup.from_process_group(slot_cap(batch * shape.hidden), device=self.x.device)

    @property
    def weight_bytes(self):
        return sum(l.weight_bytes for l in self.layers)

    def _allreduce(self, t):
        if self.world > 1 and self.collectives:
            import torch.distributed as dist
            dist.all_reduce(t)
        return t

    def check(self, stream=None):
        """Raise InvalidInputError if a step since the last check saw a non-finite activation
        (synchronizes ``stream``)."""
        import paper_2505_15909_b200 as rq
        rq.check_flag(self.err, stream)

    def step(self, x0, stream=None, pdl=True):
        """One decode step for the batch; returns the residual stream after all layers.
        Asynchronous (capturable in a CUDA graph); :meth:`check` reports non-finite inputs."""
        if self.peer is not None:
            return step_peer([self], [x0], [stream], pdl)[0]
        self.x.copy_(x0)
        delta = None
        for layer in self.layers:
            o = self._allreduce(layer.attn_half(self.x, delta, self.ws, stream, pdl))
            delta = self._allreduce(layer.mlp_half(self.x, o, self.ws, stream, pdl))
        # fold the last layer's down-projection into the residual stream
        self.x.add_(delta)
        return self.x


def step_peer(stacks, x0s, streams=None, pdl=True):
    """One decode step of the ranks in ``stacks`` whose allreduces run over peer memory
    (each stack's ``peer``).  One stack per process (torchrun), or all ranks of a group driven
    by this process (PeerGroup.single_process): the ranks are issued half-layer by half-layer,
    so every consumer follows, in issue order, the producers it waits for."""
    streams = streams or [None] * len(stacks)
    for st, x0, stream in zip(stacks, x0s, streams):
        if stream is None:
            st.x.copy_(x0)
        else:
            import torch
            with torch.cuda.stream(stream):
                st.x.copy_(x0)
    for li in range(len(stacks[0].layers)):
        for st, stream in zip(stacks, streams):
            st.layers[li].attn_half(st.x, None, st.ws, stream, pdl, peer=st.peer, peer_in=li > 0)
        for st, stream in zip(stacks, streams):
            st.layers[li].mlp_half(st.x, None, st.ws, stream, pdl, peer=st.peer)
    for st, stream in zip(stacks, streams):  # fold the last down-projection into the residual
        st.peer.reduce(st.x, accumulate=True, stream=stream)
    return [st.x for st in stacks]
