"""GPU parity: every rtnq kernel against the oracle and the reference's golden vectors.

Bit-exact: quantize-and-pack (all layouts, f32/f16 scales), relayout, dequantize,
and the reference-exact GEMMs (gemm_fused / gemm_dequant / gemm_oracle / gemm_float)
through the host C-ABI.  The tensor-core linear is checked against the f64 oracle
within the tolerance stated in each test.
"""
import numpy as np
import pytest

import paper_2505_15909_b200 as rq
from oracle import KERNEL, NATIVE, ROW_MAJOR
from oracle import encode_native_i4, encode_native_i8

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def bf16_exact(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    return (x.view(np.uint32) & 0xFFFF0000).view(np.float32)


def rel_frob(x, ref):
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.sqrt((ref ** 2).sum())
    num = np.sqrt(((x - ref) ** 2).sum())
    return num if den == 0 else num / den


# ---- host C-ABI (reference-identical results) ------------------------------------------

def test_host_api_matches_golden(golden_qg):
    for name, z in golden_qg.items():
        rows, cols, bits, g, ragged, m, tr, tc = (int(v) for v in z["meta"])
        data, scales = rq.quantize_tensor(z["w"], bits, g, bool(ragged))
        assert np.array_equal(data, z["data"]), name
        assert np.array_equal(scales, z["scales"]), name
        k = rq.reshuffle(data, rq.layout(rq.ROW_MAJOR), rq.layout(rq.KERNEL_INTERLEAVED, tr, tc),
                         bits, rows, cols)
        assert np.array_equal(k, z["kernel"]), name
        back = rq.reshuffle(k, rq.layout(rq.KERNEL_INTERLEAVED, tr, tc), rq.layout(rq.ROW_MAJOR),
                            bits, rows, cols)
        assert np.array_equal(back, data), name
        klay = rq.layout(rq.KERNEL_INTERLEAVED, tr, tc)
        deq = rq.dequantize_tensor(k, klay, bits, rows, cols, g, scales, bool(ragged))
        assert np.array_equal(deq, z["deq"]), name
        a = z["a"]
        f = rq.gemm_fused(a, k, klay, bits, rows, g, scales, bool(ragged))
        assert np.array_equal(f.view(np.uint32), z["fused"].view(np.uint32)), name
        d = rq.gemm_dequant(a, data, rq.layout(rq.ROW_MAJOR), bits, rows, g, scales, bool(ragged))
        assert np.array_equal(d.view(np.uint32), z["dequant"].view(np.uint32)), name
        o = rq.gemm_oracle(a, data, rq.layout(rq.ROW_MAJOR), bits, rows, g, scales, bool(ragged))
        assert np.array_equal(o.view(np.uint32), z["oracle"].view(np.uint32)), name


def test_host_api_kats():
    # test_quant.cpp:33-91, test_packing.cpp:38-58, test_gemm.cpp:61-90
    assert rq.compute_scale([1.0, -2.0, 3.75], 4) == 0.5
    assert rq.compute_scale([-7.5], 4) == 1.0
    assert rq.compute_scale(np.zeros(64), 8) == 1.0
    for bad in ([], [1.0, np.nan], [np.inf]):
        with pytest.raises(rq.InvalidInputError):
            rq.compute_scale(bad, 4)
    codes, s = rq.quantize_group([1.0, -2.0, 3.75], 4)
    assert s == 0.5 and codes.tolist() == [2, -4, 7]
    codes, s = rq.quantize_group([-7.5], 4)
    assert s == 1.0 and codes.tolist() == [-8]
    assert rq.dequantize_group([2, -4, 7], 0.5, 4).tolist() == [1.0, -2.0, 3.5]
    with pytest.raises(rq.CorruptDataError):
        rq.dequantize_group([9], 1.0, 4)
    # hand products 15 / -5 through every path
    logical = np.array([[1, 2, 3, 4], [-4, -3, -2, -1]], np.int8)
    rm = np.array([0xA9, 0xCB, 0x54, 0x76], np.uint8)  # pack(logical, 4)
    klay = rq.layout(rq.KERNEL_INTERLEAVED)
    k = rq.reshuffle(rm, rq.layout(rq.ROW_MAJOR), klay, 4, 2, 4)
    sc = np.array([[0.5], [0.25]], np.float32)
    a = np.array([[1, 2, 3, 4]], np.float32)
    for out in (rq.gemm_fused(a, k, klay, 4, 2, 4, sc), rq.gemm_dequant(a, rm, rq.layout(), 4, 2, 4, sc),
                rq.gemm_oracle(a, rm, rq.layout(), 4, 2, 4, sc)):
        assert out.tolist() == [[15.0, -5.0]]
    del logical
    # error classes (test_gemm.cpp:174-190)
    with pytest.raises(rq.ShapeError):
        rq.gemm_fused(a, rm, rq.layout(), 4, 2, 4, sc)  # row-major into the fused path
    with pytest.raises(rq.InvalidInputError):
        rq.gemm_auto(a, k, klay, 4, 2, 4, sc, threshold=0)
    bad = a.copy()
    bad[0, 1] = np.nan
    with pytest.raises(rq.InvalidInputError):
        rq.gemm_fused(bad, k, klay, 4, 2, 4, sc)


def test_gemm_auto_dispatch():
    # test_gemm.cpp:151-172 / acceptance.cpp:290-307
    rng = np.random.default_rng(59)
    w = rng.uniform(-1, 1, (8, 32)).astype(np.float32)
    data, sc = rq.quantize_tensor(w, 4, 16)
    klay = rq.layout(rq.KERNEL_INTERLEAVED)
    k = rq.reshuffle(data, rq.layout(), klay, 4, 8, 32)
    a1 = rng.uniform(-1, 1, (1023, 32)).astype(np.float32)
    out, path = rq.gemm_auto(a1, k, klay, 4, 8, 16, sc, 1024)
    assert path == rq.PATH_FUSED and np.array_equal(out, rq.gemm_fused(a1, k, klay, 4, 8, 16, sc))
    a2 = rng.uniform(-1, 1, (1024, 32)).astype(np.float32)
    out, path = rq.gemm_auto(a2, k, klay, 4, 8, 16, sc, 1024)
    assert path == rq.PATH_DEQUANT_FIRST
    assert np.array_equal(out, rq.gemm_dequant(a2, k, klay, 4, 8, 16, sc))


def test_quantize_random_vs_oracle(oracle):
    """Bit-exact quantize for shapes on both the fused and the generic path."""
    rng = np.random.default_rng(7)
    for trial in range(40):
        bits = 4 if trial % 2 else 8
        g = int(2 ** rng.integers(0, 9))
        cols = int(max(g, 128) * rng.integers(1, 4)) if trial % 3 else int(rng.integers(1, 300))
        ragged = cols % g != 0
        rows = int(rng.integers(1, 70))
        amp = float(2.0 ** rng.integers(-20, 20))
        w = rng.uniform(-amp, amp, (rows, cols)).astype(np.float32)
        codes, scales = oracle.quantize(w, bits, g, ragged)
        data, s2 = rq.quantize_tensor(w, bits, g, ragged)
        assert np.array_equal(s2, scales)
        assert np.array_equal(data, oracle.pack(codes, bits))


@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "float16"])
@pytest.mark.parametrize("bits,g,rows,cols", [(4, 128, 300, 512), (8, 128, 64, 1024), (4, 32, 48, 256),
                                               (8, 4096, 40, 4096), (4, 64, 17, 200), (8, 1, 5, 9)])
def test_device_quantize_pack_all_layouts(oracle, dtype, bits, g, rows, cols):
    ragged = cols % g != 0
    tdt = getattr(torch, dtype)
    gen = torch.Generator(device="cuda").manual_seed(rows * cols + bits)
    w = (torch.rand(rows, cols, device="cuda", generator=gen) * 2 - 1).to(tdt)
    w[0, : min(cols, 3)] = 0  # partially-zero group
    if rows > 2:
        w[2] = 0  # all-zero groups -> scale 1.0
    q = rq.quantize_pack(w, bits, g, ragged, native=True, row_major=True, kernel=True,
                         scales_f32=True, scales_f16=True)
    wf = w.float().cpu().numpy()
    codes, scales = oracle.quantize(wf, bits, g, ragged)
    assert np.array_equal(q.scales_f32.cpu().numpy(), scales)
    s16 = oracle.f16_round(scales)
    assert np.array_equal(q.scales_f16.cpu().numpy().view(np.uint16), s16)
    assert np.array_equal(q.codes_row_major.cpu().numpy(), oracle.pack(codes, bits))
    assert np.array_equal(q.codes_kernel.cpu().numpy(), oracle.encode(codes, bits, KERNEL))
    assert np.array_equal(q.codes.cpu().numpy(), oracle.encode(codes, bits, NATIVE))
    gpr = scales.shape[1]
    assert np.array_equal(q.scales.cpu().numpy().view(np.uint16), oracle.native_scales(s16, rows, gpr))
    # device relayout row-major -> native equals the kernel's native output
    nat = rq.relayout(q.codes_row_major, rq.layout(rq.ROW_MAJOR), rq.layout(rq.NATIVE), bits, rows, cols)
    assert torch.equal(nat, q.codes)
    ns = rq.native_scales(q.scales_f32, rows, gpr)
    assert torch.equal(ns, q.scales)


def test_quantize_flags_non_finite():
    w = torch.ones(16, 128, device="cuda")
    w[3, 7] = float("nan")
    with pytest.raises(rq.InvalidInputError):
        rq.quantize_pack(w, 4, 128)
    w[3, 7] = float("inf")
    with pytest.raises(rq.InvalidInputError):
        rq.quantize_pack(w, 8, 32)


def test_dequantize_native_bf16(oracle):
    rows, cols, bits, g = 64, 256, 4, 64
    w = torch.randn(rows, cols, device="cuda")
    q = rq.quantize_pack(w, bits, g, scales_f32=True)
    out = rq.dequantize(q.codes, rq.layout(rq.NATIVE), bits, rows, cols, g, q.scales, rq.F16,
                        rq.SCALES_NATIVE, torch.float32)
    codes, scales = oracle.quantize(w.cpu().numpy(), bits, g)
    s16 = oracle.f16_round(scales).view(np.float16).astype(np.float32)
    assert np.array_equal(out.cpu().numpy(), oracle.dequantize(codes, s16, g))


# ---- tensor-core linear ------------------------------------------------------------------

def _make(oracle, n, k, bits, g, seed, ragged=False):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    w = ((torch.rand(n, k, device="cuda", generator=gen) * 2 - 1) * (3.0 / k) ** 0.5).to(torch.bfloat16)
    q = rq.quantize_pack(w, bits, g, ragged)
    codes, scales = oracle.quantize(w.float().cpu().numpy(), bits, g, ragged)
    s16w = oracle.f16_round(scales).view(np.float16).astype(np.float32)
    return q, codes, s16w


TOL = 1e-5  # rel. Frobenius vs the f64 oracle (reference gate 1e-4, acceptance.cpp:281-282)


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("m", [1, 3, 8, 16, 17, 32, 64, 80])
def test_linear_tensor_core_vs_oracle(oracle, bits, m):
    n, k, g = 528, 1024, 128
    q, codes, s16w = _make(oracle, n, k, bits, g, seed=m * 7 + bits)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    out = rq.linear(a, q, out_dtype=torch.float32)
    ref = oracle.gemm_oracle_f64(a.float().cpu().numpy(), codes, g, s16w)
    assert rel_frob(out.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("bits,g,k,act", [(4, 16, 256, "bfloat16"), (4, 32, 512, "float16"),
                                          (4, 64, 192, "bfloat16"), (8, 16, 96, "float16"),
                                          (8, 32, 320, "bfloat16"), (8, 8192, 4096, "bfloat16"),
                                          (4, 4096, 1024, "float16"), (8, 512, 1536, "float16")])
def test_linear_groups_dtypes(oracle, bits, g, k, act):
    n, m = 200, 5
    q, codes, s16w = _make(oracle, n, k, bits, g, seed=k + g, ragged=k % g != 0)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(getattr(torch, act))
    for odt in (torch.float32, torch.bfloat16, torch.float16):
        out = rq.linear(a, q, out_dtype=odt)
        ref = oracle.gemm_oracle_f64(a.float().cpu().numpy(), codes, g, s16w)
        tol = TOL if odt == torch.float32 else 8e-3  # one 16-bit output rounding
        assert rel_frob(out.float().cpu().numpy(), ref) <= tol, odt


def test_linear_deterministic_and_split_invariant(oracle, monkeypatch):
    n, k, bits, g, m = 4096, 4096, 4, 128, 16
    q, codes, s16w = _make(oracle, n, k, bits, g, seed=1)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    o1 = rq.linear(a, q, out_dtype=torch.float32)
    o2 = rq.linear(a, q, out_dtype=torch.float32)
    assert torch.equal(o1, o2)  # run-to-run bit identity (deterministic stream-K fixup)
    for ctas in ("1", "7", "64", "300"):
        monkeypatch.setenv("RTNQ_WGEMM_CTAS", ctas)
        ws = rq.Workspace(device="cuda")
        o3 = rq.linear(a, q, out_dtype=torch.float32, workspace=ws)
        assert rel_frob(o3.cpu().numpy(), o1.cpu().numpy()) <= 1e-6, ctas
    ref = oracle.gemm_oracle_f64(a.float().cpu().numpy(), codes, g, s16w)
    assert rel_frob(o1.cpu().numpy(), ref) <= TOL


LLAMA_8B = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}


@pytest.mark.parametrize("name", list(LLAMA_8B))
@pytest.mark.parametrize("bits", [4, 8])
def test_linear_llama_shapes_vs_dequant_reference(name, bits):
    """Full-size Llama-3.1-8B shapes: compare against a torch f64 GEMM over the
    exactly dequantized weights (size-independent check: same math, f64 sums)."""
    n, k = LLAMA_8B[name]
    g = 128 if bits == 4 else 1 << (k - 1).bit_length()  # W8 per-channel (configs[2])
    w = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
    q = rq.quantize_pack(w, bits, g, ragged=k % g != 0)
    wd = rq.dequantize(q.codes, rq.layout(q.layout), bits, n, k, g, q.scales, rq.F16,
                       rq.SCALES_NATIVE, torch.float32)
    for m in (1, 4, 16):
        a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
        out = rq.linear(a, q, out_dtype=torch.float32)
        ref = a.double() @ wd.double().t()
        err = ((out.double() - ref).norm() / ref.norm()).item()
        assert err <= TOL, (name, bits, m, err)


@pytest.mark.parametrize("n,k,bits,g,m", [(4096, 4096, 4, 128, 16), (512, 1024, 4, 128, 1),
                                          (4096, 14336, 8, 16384, 5), (1000, 2048, 8, 128, 33),
                                          (2304, 16384, 4, 128, 7)])
def test_cluster_split_k_matches_stream_k(oracle, monkeypatch, n, k, bits, g, m):
    """Small-N shapes run cluster split-K (DSMEM reduction); it must agree with the
    stream-K path and be run-to-run deterministic."""
    q, codes, s16w = _make(oracle, n, k, bits, g, seed=n + k, ragged=k % g != 0)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    o1 = rq.linear(a, q, out_dtype=torch.float32)
    o2 = rq.linear(a, q, out_dtype=torch.float32)
    assert torch.equal(o1, o2)
    monkeypatch.setenv("RTNQ_WGEMM_CLUSTER", "0")
    o3 = rq.linear(a, q, out_dtype=torch.float32, workspace=rq.Workspace(device="cuda"))
    assert rel_frob(o1.cpu().numpy(), o3.cpu().numpy()) <= 1e-6
    if n * k <= 4096 * 4096:
        ref = oracle.gemm_oracle_f64(a.float().cpu().numpy(), codes, g, s16w)
        assert rel_frob(o1.cpu().numpy(), ref) <= TOL


@pytest.mark.parametrize("n,k,m", [(4096, 4096, 1), (4096, 14336, 16), (6144, 4096, 64),
                                   (1000, 2048, 5), (200, 96, 33), (28672, 4096, 16)])
def test_w8_per_channel_int8_path(oracle, n, k, m):
    """W8 per-channel runs tcgen05 kind::i8 over the row-major codes with exact int8
    activation planes; against the f64 oracle (small) or an f64 GEMM over the exactly
    dequantized weights (large)."""
    g = 1 << (k - 1).bit_length()
    gen = torch.Generator(device="cuda").manual_seed(n + k + m)
    w = ((torch.rand(n, k, device="cuda", generator=gen) * 2 - 1) * (3.0 / k) ** 0.5).to(torch.bfloat16)
    q = rq.quantize_pack(w, 8, g, ragged=k % g != 0)
    assert q.layout == rq.NATIVE_I8
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1, generator=gen).to(torch.bfloat16)
    a[0, : k // 3] *= 1e-3  # a wide dynamic range inside one token
    out = rq.linear(a, q, out_dtype=torch.float32)
    assert torch.equal(out, rq.linear(a, q, out_dtype=torch.float32))  # deterministic
    wd = rq.dequantize(q.codes, rq.layout(rq.NATIVE_I8), 8, n, k, g, q.scales, rq.F16,
                       rq.SCALES_NATIVE, torch.float32)
    ref = a.double() @ wd.double().t()
    assert ((out.double() - ref).norm() / ref.norm()).item() <= TOL


@pytest.mark.parametrize("n,k,m,act", [(4096, 4096, 1, "bfloat16"), (4096, 14336, 16, "bfloat16"),
                                       (6144, 4096, 33, "float16"), (1000, 2048, 5, "bfloat16"),
                                       (200, 208, 17, "float16"), (28672, 4096, 16, "bfloat16"),
                                       (520, 1024, 80, "bfloat16"), (300, 4096, 64, "float16")])
def test_w4_group128_int8_path(oracle, n, k, m, act):
    """W4 group-128 runs tcgen05 kind::i8 over NATIVE_I4 nibble tiles (16 x code as s8,
    one TMEM accumulator per group) with exact int8 activation planes: packing bit-exact
    against the numpy restatement; output against the f64 oracle (small) or an f64 GEMM
    over the exactly dequantized weights (large)."""
    g = 128
    gen = torch.Generator(device="cuda").manual_seed(n * 3 + k + m)
    w = ((torch.rand(n, k, device="cuda", generator=gen) * 2 - 1) * (3.0 / k) ** 0.5).to(torch.bfloat16)
    q = rq.quantize_pack(w, 4, g, ragged=k % g != 0, row_major=True)
    assert q.layout == rq.NATIVE_I4
    logical = oracle.unpack(q.codes_row_major.cpu().numpy(), n * k, 4).reshape(n, k)
    assert np.array_equal(q.codes.cpu().numpy(), encode_native_i4(logical))
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1, generator=gen).to(getattr(torch, act))
    a[0, : k // 3] *= 1e-3  # a wide dynamic range inside one token
    out = rq.linear(a, q, out_dtype=torch.float32)
    assert torch.equal(out, rq.linear(a, q, out_dtype=torch.float32))  # deterministic
    if n * k <= 1 << 22:
        codes, scales = oracle.quantize(w.float().cpu().numpy(), 4, g, k % g != 0)
        assert np.array_equal(codes, logical)
        s16w = oracle.f16_round(scales).view(np.float16).astype(np.float32)
        ref = oracle.gemm_oracle_f64(a.float().cpu().numpy(), codes, g, s16w)
        assert rel_frob(out.cpu().numpy(), ref) <= TOL
    else:
        wd = rq.dequantize(q.codes, rq.layout(rq.NATIVE_I4), 4, n, k, g, q.scales, rq.F16,
                           rq.SCALES_NATIVE, torch.float32)
        ref = a.double() @ wd.double().t()
        assert ((out.double() - ref).norm() / ref.norm()).item() <= TOL


def test_int8_mma_codes_bit_exact(oracle):
    """The kind::i8 operands hold exactly the reference's codes, re-encoded (W8: two's
    complement in 128x128 swizzled tiles; W4: nibble pairs in 128x128 group tiles)."""
    for bits, g, enc, kind in ((8, 1024, encode_native_i8, rq.NATIVE_I8), (4, 128, encode_native_i4, rq.NATIVE_I4)):
        n, k = 333, 1024
        w = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.bfloat16)
        q = rq.quantize_pack(w, bits, g)
        assert q.layout == kind
        codes, _ = oracle.quantize(w.float().cpu().numpy(), bits, g, False)
        assert np.array_equal(q.codes.cpu().numpy(), enc(codes))


def test_w4_group128_tc_kernel_still_reachable(oracle):
    """native=True keeps W4 group-128 on the kind::f16 kernel (NATIVE layout); both
    kernels agree."""
    n, k, m = 1024, 2048, 7
    w = ((torch.rand(n, k, device="cuda") * 2 - 1) * (3.0 / k) ** 0.5).to(torch.bfloat16)
    q1 = rq.quantize_pack(w, 4, 128)
    q2 = rq.quantize_pack(w, 4, 128, native=True)
    assert (q1.layout, q2.layout) == (rq.NATIVE_I4, rq.NATIVE)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    o1, o2 = rq.linear(a, q1, out_dtype=torch.float32), rq.linear(a, q2, out_dtype=torch.float32)
    assert rel_frob(o1.cpu().numpy(), o2.cpu().numpy()) <= 2 * TOL


def test_graft_smoke_entry():
    """The driver's smoke() (one small W4 linear on cuda:0 checked against the oracle)."""
    import __graft_entry__
    __graft_entry__.smoke()


@pytest.mark.parametrize("bits,g,m", [(4, 128, 1), (4, 128, 300), (8, 4096, 64), (4, 64, 96), (8, 128, 130)])
def test_dequant_first_tensor_path(oracle, bits, g, m):
    """dequant-first on the tensor cores (exact hi + lo 16-bit weight split, both
    terms accumulated in one hand-written tcgen05 GEMM, dense_tc.cu), any codes layout, against
    the f64 oracle."""
    n, k = 520, 4096 if g == 4096 else 1024
    q, codes, s16w = _make(oracle, n, k, bits, g, seed=m + bits + g)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
    ref = oracle.gemm_oracle_f64(a.float().cpu().numpy(), codes, g, s16w)
    out = rq.linear(a, q, out_dtype=torch.float32, path=rq.PATH_DEQUANT_FIRST)
    assert rel_frob(out.cpu().numpy(), ref) <= TOL
    o16 = rq.linear(a, q, out_dtype=torch.bfloat16, path=rq.PATH_DEQUANT_FIRST)
    assert rel_frob(o16.float().cpu().numpy(), ref) <= 8e-3


@pytest.mark.parametrize("m,n,k,g,dt", [(257, 200, 1000, 128, torch.bfloat16),  # k % 8 != 0, ragged
                                         (130, 136, 520, 8, torch.float16),       # f16, odd tiles
                                         (1024, 384, 2048, 128, torch.bfloat16)])
def test_dense_tc_odd_shapes(oracle, m, n, k, g, dt):
    """The tcgen05 dequant-first GEMM on partial tiles (m, n not multiples of 128), rows not a
    multiple of 8 elements (padded copies for the TMA), f16 operands, every output type."""
    ragged = k % g != 0
    q, codes, s16w = _make(oracle, n, k, 4, g, seed=m + n, ragged=ragged)
    a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(dt)
    ref = oracle.gemm_oracle_f64(a.float().cpu().numpy(), codes, g, s16w)
    for odt, tol in ((torch.float32, TOL), (torch.bfloat16, 8e-3), (torch.float16, 1e-3)):
        out = rq.linear(a, q, out_dtype=odt, path=rq.PATH_DEQUANT_FIRST)
        assert rel_frob(out.float().cpu().numpy(), ref) <= tol, odt
    # deterministic
    o1 = rq.linear(a, q, out_dtype=torch.float32, path=rq.PATH_DEQUANT_FIRST)
    assert torch.equal(o1, rq.linear(a, q, out_dtype=torch.float32, path=rq.PATH_DEQUANT_FIRST))


def test_gemm_auto_dispatch_tensor_paths(oracle):
    """gemm_auto (gemm.cpp:100-109) on the tensor paths: m >= threshold takes dequant-first,
    below it the fused kernel; both agree with the oracle."""
    n, k, bits, g = 256, 1024, 4, 128
    q, codes, s16w = _make(oracle, n, k, bits, g, seed=77)
    for m, want in ((40, rq.PATH_FUSED), (64, rq.PATH_DEQUANT_FIRST), (200, rq.PATH_DEQUANT_FIRST)):
        a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
        out = rq.linear(a, q, out_dtype=torch.float32, path=rq.PATH_AUTO, threshold=64)
        ref = oracle.gemm_oracle_f64(a.float().cpu().numpy(), codes, g, s16w)
        assert rel_frob(out.cpu().numpy(), ref) <= TOL, m
        # the chosen path reproduces its own output exactly
        again = rq.linear(a, q, out_dtype=torch.float32, path=want)
        assert torch.equal(out, again), m


TP8_SHARDS = {"8b_qkv": (768, 4096), "8b_o": (4096, 512), "8b_down": (4096, 1792),
              "70b_o": (8192, 1024), "70b_down": (8192, 3584), "405b_qkv": (2304, 16384),
              "405b_o": (16384, 2048)}


@pytest.mark.parametrize("name", list(TP8_SHARDS))
@pytest.mark.parametrize("bits", [4, 8])
def test_linear_tp8_shard_shapes(name, bits):
    """The per-rank weight shards the 8-GPU tensor-parallel step runs,
    through the default kernels, against an f64 GEMM over the exactly dequantized weights."""
    n, k = TP8_SHARDS[name]
    g = 128 if bits == 4 else 1 << (k - 1).bit_length()
    w = ((torch.rand(n, k, device="cuda") * 2 - 1) * (3.0 / k) ** 0.5).to(torch.bfloat16)
    q = rq.quantize_pack(w, bits, g, ragged=k % g != 0)
    wd = rq.dequantize(q.codes, rq.layout(q.layout), bits, n, k, g, q.scales, rq.F16,
                       rq.SCALES_NATIVE, torch.float32)
    for m in (1, 16):
        a = torch.empty(m, k, device="cuda").uniform_(-1, 1).to(torch.bfloat16)
        out = rq.linear(a, q, out_dtype=torch.float32)
        ref = a.double() @ wd.double().t()
        assert ((out.double() - ref).norm() / ref.norm()).item() <= TOL, (name, bits, m)


@pytest.mark.parametrize("m", [1, 16])
def test_chained_linears_pdl_graph_identical(m):
    """Each linear consumes the previous one's output (W8 cluster, W4 cluster, W8 stream-K, W4
    stream-K, mixed shapes).  The planes kernel lets the next GEMM launch before the previous
    GEMM finishes (early PDL trigger) and the W8 cluster peers push without a handshake; the
    chain run back to back in one CUDA graph must equal the chain run one synchronized linear
    at a time, bit for bit."""
    gen = torch.Generator(device="cuda").manual_seed(7)
    shapes = [(4096, 4096, 8), (4096, 4096, 4), (28672, 4096, 8), (4096, 28672, 4),
              (6144, 4096, 8), (4096, 6144, 4)]
    qs = []
    for n, k, bits in shapes:
        w = ((torch.rand(n, k, device="cuda", generator=gen) * 2 - 1) * 0.05).to(torch.bfloat16)
        g = 128 if bits == 4 else 1 << (k - 1).bit_length()
        qs.append(rq.quantize_pack(w, bits, g, ragged=bits == 8))
    x = torch.empty(m, 4096, device="cuda").uniform_(-1, 1, generator=gen).to(torch.bfloat16)
    ws = rq.Workspace(device="cuda")
    outs = [torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for n, _, _ in shapes]
    st = torch.cuda.Stream()

    def chain(sync):
        a = x
        for q, o in zip(qs, outs):
            rq.linear(a, q, out=o, workspace=ws, stream=st, pdl=True, check=False)
            if sync:
                st.synchronize()
            a = o
        return [o.clone() for o in outs] if sync else None

    with torch.cuda.stream(st):
        ref = chain(True)
    for o in outs:
        o.zero_()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=st):
        chain(False)
    for _ in range(3):
        for o in outs:
            o.zero_()
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        for i, (o, r) in enumerate(zip(outs, ref)):
            assert torch.equal(o, r), f"linear {i} {shapes[i]} differs in the graph chain"
    # eager back to back, no synchronization between linears
    with torch.cuda.stream(st):
        chain(False)
    st.synchronize()
    for i, (o, r) in enumerate(zip(outs, ref)):
        assert torch.equal(o, r), f"linear {i} {shapes[i]} differs in the eager chain"
    assert all(torch.isfinite(r.float()).all() for r in ref)


@pytest.mark.parametrize("bits", [8, 4])
def test_405b_ffn_up_full_shape(bits):
    """The largest single-GPU linear of the BASELINE configs (Llama-3.1-405B ffn_up,
    106496 x 16384, 1.7 GB at W8) at batch 16 through the fused int8 path, against an f64
    product of the dequantized weights (the f16 scales the kernels use).  Bar: 1e-5 relative
    Frobenius (measured 7e-8 at W8, 2e-7 at W4)."""
    n, k, m = 106496, 16384, 16
    gen = torch.Generator(device="cuda").manual_seed(3)
    w = ((torch.rand(n, k, device="cuda", generator=gen) * 2 - 1) * 0.02).to(torch.bfloat16)
    g = k if bits == 8 else 128
    q = rq.quantize_pack(w, bits, g, ragged=bits == 8, scales_f16=True, row_major=True)
    del w
    x = torch.randn(m, k, device="cuda", generator=gen).to(torch.bfloat16)
    y = rq.linear(x, q, out_dtype=torch.float32)
    wd = rq.dequantize(q.codes_row_major, rq.layout(rq.ROW_MAJOR), bits, n, k, g, q.scales_f16, rq.F16,
                       rq.SCALES_REF)
    num = den = 0.0
    for i in range(0, n, 8192):
        r = x.double() @ wd[i:i + 8192].double().t()
        num += ((y[:, i:i + 8192].double() - r) ** 2).sum().item()
        den += (r ** 2).sum().item()
    del q, wd, y
    torch.cuda.empty_cache()
    assert (num / den) ** 0.5 < 1e-5


@pytest.mark.parametrize("bits,n,k,g,m", [(4, 40, 14336, 128, 3), (8, 24, 4096, 64, 5), (4, 16, 1001, 16, 1),
                                          (8, 33, 520, 8, 2)])
def test_dropin_gemm_fused_group_parallel_bit_exact(oracle, bits, n, k, g, m):
    """The drop-in gemm_fused on the reference's kernel layout runs the group-parallel exact
    kernel (one lane per group, block sums folded in group order) for <= 128 groups per row and
    the one-thread-per-output kernel beyond: both bit-identical to the C oracle (gemm.cpp:46-92),
    incl. ragged groups, odd row counts and 1..5 tokens."""
    ragged = k % g != 0
    rng = np.random.default_rng(n * k + m)
    w = (rng.standard_normal((n, k)) * 0.05).astype(np.float32)
    data, scales = rq.quantize_tensor(w, bits, g, ragged)
    klay = rq.layout(rq.KERNEL_INTERLEAVED)
    kern = rq.reshuffle(data, rq.layout(), klay, bits, n, k)
    a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    got = rq.gemm_fused(a, kern, klay, bits, n, g, scales, ragged)
    want = oracle.gemm_fused(a, kern, n, bits, g, scales)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
