"""GPU: the decode-layer kernels against plain-PyTorch fp32 references, and tensor
parallelism simulated on one GPU (rank shards run in turn, partials summed) against the
unsharded layer."""
import numpy as np
import pytest

import paper_2505_15909_b200 as rq
from paper_2505_15909_b200 import tp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def rel(x, ref):
    return ((x.double() - ref.double()).norm() / ref.double().norm()).item()


def test_add_rmsnorm_matches_torch():
    g = torch.Generator(device="cuda").manual_seed(0)
    for m, h in ((1, 4096), (16, 8192), (3, 512)):
        x = torch.randn(m, h, device="cuda", generator=g).to(torch.bfloat16)
        d = torch.randn(m, h, device="cuda", generator=g).to(torch.bfloat16)
        w = (1 + 0.1 * torch.rand(h, device="cuda", generator=g)).to(torch.bfloat16)
        xs = (x.float() + d.float()).to(torch.bfloat16)
        ref = xs.float() * torch.rsqrt(xs.float().pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
        out = torch.empty_like(x)
        rq.add_rmsnorm(x, w, out, delta=d)
        assert torch.equal(x, xs)                   # residual updated in place
        assert rel(out.float(), ref) < 4e-3         # one bf16 rounding
        out2 = torch.empty_like(x)
        rq.add_rmsnorm(x, w, out2)                  # no delta: plain rmsnorm
        assert torch.equal(out2, out)


def test_silu_mul_matches_torch():
    gu = torch.randn(16, 2 * 3584, device="cuda").to(torch.bfloat16)
    act = torch.empty(16, 3584, device="cuda", dtype=torch.bfloat16)
    rq.silu_mul(gu, act)
    g, u = gu[:, :3584].float(), gu[:, 3584:].float()
    assert rel(act.float(), torch.nn.functional.silu(g) * u) < 4e-3


def rope_ref(x, pos, theta):
    d = x.shape[-1]
    inv = theta ** (-2.0 * torch.arange(d // 2, device=x.device, dtype=torch.float64) / d)
    ang = pos * inv
    c, s = torch.cos(ang), torch.sin(ang)
    a, b = x[..., : d // 2].double(), x[..., d // 2:].double()
    return torch.cat([a * c - b * s, b * c + a * s], -1)


@pytest.mark.parametrize("hq,hkv,b,lmax,pos", [
    (32, 8, 3, 40, 33), (8, 1, 3, 40, 33), (4, 2, 3, 40, 33),
    # the tensor-core kernel's 64-position stages: context ends on / next to a stage edge, one
    # position, long splits (many stages per CTA, online softmax), batch 16 / 32
    (32, 8, 2, 200, 127), (32, 8, 2, 200, 128), (32, 8, 1, 8, 0), (8, 1, 2, 1300, 1200),
    (32, 8, 1, 4100, 4095), (32, 8, 16, 300, 256),
    # splits longer than 256 positions: the streaming kernel (stages of 64, online softmax)
    (32, 8, 32, 1100, 1023), (32, 8, 16, 1100, 1024), (32, 8, 64, 700, 600), (8, 1, 128, 800, 780)])
def test_decode_attention_matches_torch(hq, hkv, b, lmax, pos):
    d, theta = 128, 500000.0
    g = torch.Generator(device="cuda").manual_seed(hq)
    qkv = torch.randn(b, (hq + 2 * hkv) * d, device="cuda", generator=g).to(torch.bfloat16)
    kc = (torch.rand(b, lmax, hkv, d, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    vc = (torch.rand(b, lmax, hkv, d, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    k0, v0 = kc.clone(), vc.clone()
    out = torch.empty(b, hq * d, device="cuda", dtype=torch.bfloat16)
    rq.decode_attention(qkv, kc, vc, out, hq, hkv, pos, d, theta)
    q = qkv[:, : hq * d].view(b, hq, d)
    kn = qkv[:, hq * d:(hq + hkv) * d].view(b, hkv, d)
    vn = qkv[:, (hq + hkv) * d:].view(b, hkv, d)
    kref, vref = k0.double(), v0.double()
    kref[:, pos] = rope_ref(kn, pos, theta).to(torch.bfloat16).double()
    vref[:, pos] = vn.double()
    # rotated key: within one bf16 rounding of the f64 rotation plus the f32 angle's error
    # (pos * inv rounded: ~pos * 2^-24 rad); value copied verbatim
    atol = 1e-6 + (pos + 1) * 2.0 ** -22 * float(kn.abs().max())
    assert torch.allclose(kc[:, pos].double(), kref[:, pos], rtol=2 ** -7, atol=atol)
    assert torch.equal(vc[:, pos], vn)
    assert torch.equal(kc[:, :pos], k0[:, :pos])           # earlier positions untouched
    qr = rope_ref(q, pos, theta)                           # [b, hq, d]
    kk = kref[:, : pos + 1].repeat_interleave(hq // hkv, dim=2)  # [b, t, hq, d]
    vv = vref[:, : pos + 1].repeat_interleave(hq // hkv, dim=2)
    s = torch.einsum("bhd,bthd->bht", qr, kk) / d ** 0.5
    ref = torch.einsum("bht,bthd->bhd", torch.softmax(s, -1), vv).reshape(b, hq * d)
    assert rel(out.float(), ref) < 6e-3


TINY = tp.LlamaShape("tiny", hidden=512, heads=4, kv_heads=2, head_dim=128, ffn=1024, layers=2)


def _full_weights(shape):
    g = torch.Generator(device="cuda").manual_seed(5)
    d = shape.head_dim
    sizes = {"qkv_proj": ((shape.heads + 2 * shape.kv_heads) * d, shape.hidden),
             "attn_out_proj": (shape.hidden, shape.heads * d),
             "ffn_up": (2 * shape.ffn, shape.hidden), "ffn_down": (shape.hidden, shape.ffn)}
    return {m: ((torch.rand(*s, device="cuda", generator=g) * 2 - 1) * (3.0 / s[1]) ** 0.5
                ).to(torch.bfloat16) for m, s in sizes.items()}


@pytest.mark.parametrize("world", [2])
def test_tp_simulated_on_one_gpu_matches_unsharded(world):
    """Shards of every rank run in turn on cuda:0; the allreduce is a sum of the partials."""
    w = _full_weights(TINY)
    table = np.array([[4, 4, 4, 8], [8, 4, 4, 4]], np.uint8)  # selective precision per module
    b, lmax, pos = 3, 20, 17
    ref_layers = [tp.TPDecodeLayer(TINY, li, 1, 0, tp.module_bits(table, li), b, lmax, pos,
                                   weights=w) for li in range(2)]
    ranks = [[tp.TPDecodeLayer(TINY, li, world, r, tp.module_bits(table, li), b, lmax, pos,
                               weights=w) for li in range(2)] for r in range(world)]
    # same KV cache contents: the unsharded cache holds every rank's heads
    for li in range(2):
        hkv = TINY.kv_heads // world
        for r in range(world):
            ranks[r][li].k_cache.copy_(ref_layers[li].k_cache[:, :, r * hkv:(r + 1) * hkv])
            ranks[r][li].v_cache.copy_(ref_layers[li].v_cache[:, :, r * hkv:(r + 1) * hkv])
    x0 = torch.randn(b, TINY.hidden, device="cuda").to(torch.bfloat16)
    ws = rq.Workspace(device="cuda")
    # unsharded
    x = x0.clone()
    delta = None
    for layer in ref_layers:
        o = layer.attn_half(x, delta, ws).clone()
        delta = layer.mlp_half(x, o, ws).clone()
    x_ref = (x.float() + delta.float())
    # sharded: each rank keeps its own replica of the residual stream
    xs = [x0.clone() for _ in range(world)]
    delta = None
    for li in range(2):
        o = sum(ranks[r][li].attn_half(xs[r], delta, ws).float() for r in range(world))
        o = o.to(torch.bfloat16)
        d = sum(ranks[r][li].mlp_half(xs[r], o, ws).float() for r in range(world))
        delta = d.to(torch.bfloat16)
    for r in range(world):
        got = xs[r].float() + delta.float()
        assert rel(got, x_ref) < 2e-2, r   # bf16 partial outputs summed in another order


def test_tp_stack_step_runs_llama8b_two_layers():
    table, _ = rq.plan.resolve("explicit:0 modules:4", 2)
    st = tp.TPDecodeStack(tp.LLAMA_8B, table, world=1, rank=0, batch=4, layers=2)
    assert st.layers[0].bits["ffn_down"] == 8 and st.layers[1].bits["ffn_down"] == 4
    x = st.step(torch.randn(4, 4096, device="cuda").to(torch.bfloat16))
    torch.cuda.synchronize()
    assert torch.isfinite(x.float()).all()


@pytest.mark.parametrize("m", [1, 5, 16])
def test_fused_planes_match_the_planes_kernel(m):
    """add+RMSNorm and SiLU*up emit the int8 kernels' activation planes in the same kernel:
    bit-identical to the standalone planes kernel on their outputs, and the linear on them is
    bit-identical to the linear that computes its own planes."""
    g = torch.Generator(device="cuda").manual_seed(m)
    h, f = 4096, 1536
    x = (torch.randn(m, h, device="cuda", generator=g)).to(torch.bfloat16)
    w = (1 + 0.1 * torch.rand(h, device="cuda", generator=g)).to(torch.bfloat16)
    y = torch.empty_like(x)
    pf = rq.Planes(m, h)
    rq.add_rmsnorm(x.clone(), w, y, eps=1e-5, planes=pf)
    ps = rq.act_planes(y, rq.Planes(m, h))
    assert torch.equal(pf.planes, ps.planes) and torch.equal(pf.texp, ps.texp)
    gu = torch.randn(m, 2 * f, device="cuda", generator=g).to(torch.bfloat16)
    act = torch.empty(m, f, device="cuda", dtype=torch.bfloat16)
    pa = rq.Planes(m, f)
    rq.silu_mul(gu, act, planes=pa)
    act_ref = rq.silu_mul(gu, torch.empty_like(act))
    assert torch.equal(act, act_ref)
    pas = rq.act_planes(act, rq.Planes(m, f))
    assert torch.equal(pa.planes, pas.planes) and torch.equal(pa.texp, pas.texp)
    for bits, k, p, a in ((4, h, pf, y), (8, h, pf, y), (4, f, pa, act)):
        g_ = 128 if bits == 4 else 1 << (k - 1).bit_length()
        wq = rq.quantize_pack((torch.rand(1024, k, device="cuda") * 2 - 1).to(torch.bfloat16), bits, g_,
                              ragged=k % g_ != 0)
        o1 = rq.linear(a, wq, out_dtype=torch.float32)
        o2 = rq.linear_planes(p, wq, torch.empty(m, 1024, device="cuda", dtype=torch.float32))
        assert torch.equal(o1, o2), (bits, k)


def test_decode_step_fused_planes_is_bit_identical():
    table, _ = rq.plan.resolve("explicit:0 modules:4", 2)
    outs = []
    for fuse in (True, False):
        st = tp.TPDecodeStack(tp.LLAMA_8B, table, world=1, rank=0, batch=4, layers=2, fuse_planes=fuse)
        x0 = torch.randn(4, 4096, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3)
                         ).to(torch.bfloat16)
        outs.append(st.step(x0).clone())
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("batch,pos", [(1, 100), (2, 300), (16, 256), (1, 700), (16, 1100)])
def test_decode_attention_merge_paths(batch, pos):
    """The split-context merges (thread-block cluster over DSMEM on small grids, last-CTA global
    merge otherwise) agree with each other and with the single-CTA path's math."""
    import os
    hq, hkv, d = 32, 8, 128
    g = torch.Generator(device="cuda").manual_seed(batch * 1000 + pos)
    qkv = torch.randn(batch, (hq + 2 * hkv) * d, device="cuda", generator=g).to(torch.bfloat16)
    kc = torch.randn(batch, pos + 1, hkv, d, device="cuda", generator=g).to(torch.bfloat16)
    vc = torch.randn(batch, pos + 1, hkv, d, device="cuda", generator=g).to(torch.bfloat16)
    outs = []
    for no_cluster in ("", "1"):
        if no_cluster:
            os.environ["RTNQ_ATTN_NO_CLUSTER"] = "1"
        try:
            o = torch.empty(batch, hq * d, device="cuda", dtype=torch.bfloat16)
            rq.decode_attention(qkv, kc.clone(), vc.clone(), o, hq, hkv, pos)
            outs.append(o)
        finally:
            os.environ.pop("RTNQ_ATTN_NO_CLUSTER", None)
    torch.cuda.synchronize()
    assert rel(outs[0], outs[1].float()) < 1e-2


def test_default_workspaces_of_attention_and_linear_are_separate():
    """decode_attention and linear with no explicit workspace on the same stream: each kind gets
    its own default buffer (the attention's split-merge scratch once overwrote the linears'
    stream-K counters in a shared default buffer, and the next stream-K linear never finished)."""
    batch, hq, hkv, d, max_len, pos = 4, 32, 8, 128, 800, 700
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = (torch.rand(batch, (hq + 2 * hkv) * d, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    kc = (torch.rand(batch, max_len, hkv, d, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    vc = (torch.rand(batch, max_len, hkv, d, device="cuda", generator=g) - 0.5).to(torch.bfloat16)
    out = torch.empty(batch, hq * d, dtype=torch.bfloat16, device="cuda")
    w = ((torch.rand(12800, 1024, device="cuda", generator=g) * 2 - 1) * 0.05).to(torch.bfloat16)
    q = rq.quantize_pack(w, 4, 128)  # 100 row-blocks: stream-K over all SMs
    a = torch.empty(3, 1024, device="cuda").uniform_(-1, 1, generator=g).to(torch.bfloat16)
    ref = rq.linear(a, q, workspace=rq.Workspace(device="cuda"))
    for _ in range(3):
        rq.decode_attention(qkv, kc, vc, out, hq, hkv, pos)
        y = rq.linear(a, q)  # default workspace, synchronizing check
        assert torch.equal(y, ref)


@pytest.mark.parametrize("batch,pos,hq,hkv", [(1, 100, 32, 8), (2, 300, 32, 8), (16, 256, 32, 8), (1, 700, 32, 8),
                                              (3, 50, 64, 2), (32, 1023, 32, 8), (16, 1100, 32, 8)])
def test_decode_attention_emits_o_proj_planes(batch, pos, hq, hkv):
    """The attention's last CTA per token writes the o-projection's activation planes: bit-identical
    to the planes kernel on the attention output, on every merge path (one split, cluster DSMEM,
    global last-CTA), on the CUDA-core kernel (32 query heads per KV head) and on the streaming
    kernel (splits of more than 128 positions)."""
    import os
    d = 128
    g = torch.Generator(device="cuda").manual_seed(batch * 7 + pos)
    qkv = torch.randn(batch, (hq + 2 * hkv) * d, device="cuda", generator=g).to(torch.bfloat16)
    kc = torch.randn(batch, pos + 1, hkv, d, device="cuda", generator=g).to(torch.bfloat16)
    vc = torch.randn(batch, pos + 1, hkv, d, device="cuda", generator=g).to(torch.bfloat16)
    for no_cluster in ("", "1"):
        if no_cluster:
            os.environ["RTNQ_ATTN_NO_CLUSTER"] = "1"
        try:
            o_ref = torch.empty(batch, hq * d, device="cuda", dtype=torch.bfloat16)
            rq.decode_attention(qkv, kc.clone(), vc.clone(), o_ref, hq, hkv, pos)
            for rep in range(2):  # the per-token counters reset themselves
                o = torch.empty_like(o_ref)
                p = rq.Planes(batch, hq * d)
                rq.decode_attention(qkv, kc.clone(), vc.clone(), o, hq, hkv, pos, planes=p)
                ref = rq.act_planes(o, rq.Planes(batch, hq * d))
                torch.cuda.synchronize()
                assert torch.equal(o, o_ref)
                assert torch.equal(p.planes, ref.planes) and torch.equal(p.texp, ref.texp), (no_cluster, rep)
        finally:
            os.environ.pop("RTNQ_ATTN_NO_CLUSTER", None)


def test_attention_workspace_shared_across_batch_sizes():
    """One attention workspace for calls of different batch sizes (global-merge path): the
    self-resetting counters sit in a fixed region, so a smaller call's partials never land on a
    larger call's counters (a batch-dependent layout once broke the merge silently)."""
    import os
    hq, hkv, d = 32, 8, 128
    ws = rq.Workspace(device="cuda")
    os.environ["RTNQ_ATTN_NO_CLUSTER"] = "1"
    try:
        for batch, pos in ((1, 700), (2, 300), (16, 700), (1, 700), (16, 700)):
            g = torch.Generator(device="cuda").manual_seed(batch + pos)
            qkv = torch.randn(batch, (hq + 2 * hkv) * d, device="cuda", generator=g).to(torch.bfloat16)
            kc = torch.randn(batch, pos + 1, hkv, d, device="cuda", generator=g).to(torch.bfloat16)
            vc = torch.randn(batch, pos + 1, hkv, d, device="cuda", generator=g).to(torch.bfloat16)
            o = torch.empty(batch, hq * d, device="cuda", dtype=torch.bfloat16)
            o_fresh = torch.empty_like(o)
            rq.decode_attention(qkv, kc.clone(), vc.clone(), o, hq, hkv, pos, workspace=ws)
            rq.decode_attention(qkv, kc.clone(), vc.clone(), o_fresh, hq, hkv, pos,
                                workspace=rq.Workspace(device="cuda"))
            torch.cuda.synchronize()
            assert torch.equal(o, o_fresh), (batch, pos)
    finally:
        os.environ.pop("RTNQ_ATTN_NO_CLUSTER", None)
