"""Pin the CPU oracle (oracle/rtnq_oracle.c) before trusting it.

1. Known-answer tests copied as *values* from the reference's own unit tests
   (proj/tests/test_{quant,packing,gemm,f16}.cpp, cited per test).
2. Golden vectors produced by the unmodified reference library
   (tests/golden/make_golden.py -> tests/golden/*.npz): the oracle must be
   bit-identical on every one.
3. When the reference library itself is present (this container), randomized
   cross-checks oracle == reference.
"""
import numpy as np
import pytest

from oracle import KERNEL, NATIVE, ROW_MAJOR, OracleError, Ref


# ---- 1. the reference's own KATs -----------------------------------------------------

def test_scale_kats(oracle):
    # proj/tests/test_quant.cpp:35-39
    assert oracle.compute_scale([1.0, -2.0, 3.75], 4) == 0.5
    assert oracle.compute_scale([-7.5], 4) == 1.0
    # degenerate group -> 1.0 (test_quant.cpp:56-62)
    assert oracle.compute_scale(np.zeros(64), 8) == 1.0
    # empty / non-finite rejected (test_quant.cpp:64-73)
    for bad in ([], [1.0, np.nan], [np.inf]):
        with pytest.raises(OracleError):
            oracle.compute_scale(bad, 4)


def test_round_half_away_kats(oracle):
    # test_quant.cpp:75-91 and :249-254
    codes, s = oracle.quantize(np.array([[1.0, -2.0, 3.75]], np.float32), 4, 4, ragged=True)
    assert s[0, 0] == 0.5 and codes.tolist() == [[2, -4, 7]]
    codes, s = oracle.quantize(np.array([[-7.5]], np.float32), 4, 1)
    assert s[0, 0] == 1.0 and codes.tolist() == [[-8]]
    codes, s = oracle.quantize(np.array([[7.5, -7.0]], np.float32), 4, 2)
    assert s[0, 0] == 1.0 and codes.tolist() == [[7, -7]]


def test_row_independence_kat(oracle):
    # test_quant.cpp:197-213
    w = np.array([[1.0, -2.0, 3.75, 0.5], [10.0, -20.0, 37.5, 5.0]], np.float32)
    codes, s = oracle.quantize(w, 4, 4)
    assert s.ravel().tolist() == [0.5, 5.0]
    assert codes[0, 2] == 7 and codes[1, 1] == -4
    deq = oracle.dequantize(codes, s, 4)
    assert deq[0, 0] == 1.0 and deq[1, 2] == 35.0


def test_group_validation(oracle):
    # test_quant.cpp:176-195
    assert oracle.groups_per_row(128, False, 256) == 2
    with pytest.raises(OracleError):
        oracle.groups_per_row(128, False, 200)
    assert oracle.groups_per_row(128, True, 200) == 2
    for g in (96, 0):
        with pytest.raises(OracleError):
            oracle.groups_per_row(g, False, 256)


def test_pack_kats(oracle):
    # test_packing.cpp:38-58
    assert oracle.pack([-8, 7], 4).tolist() == [0xF0]
    assert oracle.pack([0], 8).tolist() == [0x80]
    assert oracle.pack([3], 4).tolist() == [0x0B]
    assert oracle.pack([], 4).size == 0
    with pytest.raises(OracleError):
        oracle.pack([8], 4)


def test_interleave_hand_traced(oracle):
    # test_packing.cpp:82-96: 2x4 matrix, 2x2 tiles
    order = [[0, 2, 4, 6], [1, 3, 5, 7]]
    for r in range(2):
        for c in range(4):
            assert oracle.layout_index(KERNEL, 4, 2, 4, r, c, tr=2, tc=2) == order[r][c]
    assert oracle.layout_index(ROW_MAJOR, 4, 2, 4, 1, 2) == 6
    # padding: layout_slots(kernel(16,4), 17, 5) == 32*8
    assert oracle.layout_bytes(KERNEL, 8, 17, 5) == 32 * 8


def test_golden_16x4_tile(oracle):
    # test_packing.cpp:98-123
    codes = np.array([[((4 * r + c) & 15) - 8 for c in range(4)] for r in range(16)], np.int8)
    expected = [0x40, 0xC8] * 4 + [0x51, 0xD9] * 4 + [0x62, 0xEA] * 4 + [0x73, 0xFB] * 4
    assert oracle.encode(codes, 4, KERNEL).tolist() == expected


def test_gemm_hand_products(oracle):
    # test_gemm.cpp:75-90: rows [1,2,3,4]*0.5 and [-4..-1]*0.25 against a=[1,2,3,4]
    logical = np.array([[1, 2, 3, 4], [-4, -3, -2, -1]], np.int8)
    scales = np.array([[0.5], [0.25]], np.float32)
    a = np.array([[1, 2, 3, 4]], np.float32)
    kern = oracle.encode(logical, 4, KERNEL)
    for out in (oracle.gemm_fused(a, kern, 2, 4, 4, scales),
                oracle.gemm_dequant(a, logical, 4, scales),
                oracle.gemm_oracle(a, logical, 4, scales)):
        assert out.tolist() == [[15.0, -5.0]]


def test_gemm_identity_exact(oracle):
    # test_gemm.cpp:61-73: diag(4) at scale 0.25 is the identity, bit for bit
    logical = (np.eye(4) * 4).astype(np.int8)
    scales = np.full((4, 1), 0.25, np.float32)
    a = np.random.default_rng(41).uniform(-2, 2, (3, 4)).astype(np.float32)
    kern = oracle.encode(logical, 4, KERNEL)
    assert np.array_equal(oracle.gemm_fused(a, kern, 4, 4, 4, scales), a)
    assert np.array_equal(oracle.gemm_oracle(a, logical, 4, scales), a)


def test_f16_kats(oracle):
    # proj/tests/test_f16.cpp:17-57
    kats = [(0.0, 0x0000), (-0.0, 0x8000), (1.0, 0x3C00), (-2.0, 0xC000), (0.5, 0x3800),
            (65504.0, 0x7BFF), (2.0 ** -14, 0x0400), (2.0 ** -24, 0x0001),
            (1023 * 2.0 ** -24, 0x03FF), (1 + 2.0 ** -11, 0x3C00), (1 + 1.5 * 2.0 ** -10, 0x3C02),
            (2.0 ** -25, 0x0000), (1.5 * 2.0 ** -25, 0x0001), (2047 * 2.0 ** -25, 0x0400),
            (65520.0, 0x7C00), (1e9, 0x7C00), (-1e9, 0xFC00), (2.0 ** -26, 0), (-(2.0 ** -26), 0x8000),
            (float("inf"), 0x7C00), (float("-inf"), 0xFC00)]
    for x, h in kats:
        assert oracle.f32_to_f16(x) == h, (x, h)
    assert oracle.f32_to_f16(float(np.nextafter(np.float32(65520), np.float32(0)))) == 0x7BFF
    h = oracle.f32_to_f16(float("nan"))
    assert (h & 0x7C00) == 0x7C00 and (h & 0x3FF) != 0
    assert oracle.f16_to_f32(0x0001) == 2.0 ** -24 and oracle.f16_to_f32(0x7BFF) == 65504.0


# ---- 2. golden vectors from the reference --------------------------------------------

def test_f16_golden(oracle, golden_f16):
    widened = golden_f16["widened"].view(np.float32)
    for h in range(0, 65536, 7):
        got = np.float32(oracle.f16_to_f32(h))
        assert got.view(np.uint32) == widened[h].view(np.uint32) or (np.isnan(got) and np.isnan(widened[h]))
    for x, h in zip(golden_f16["xs"], golden_f16["narrowed"]):
        assert oracle.f32_to_f16(float(x)) == int(h)
    # numpy's f16 cast (used by f16_round) agrees with the reference on all of them
    assert np.array_equal(oracle.f16_round(golden_f16["xs"]), golden_f16["narrowed"])


def test_quant_gemm_golden(oracle, golden_qg):
    for name, z in golden_qg.items():
        rows, cols, bits, g, ragged, m, tr, tc = (int(v) for v in z["meta"])
        codes, scales = oracle.quantize(z["w"], bits, g, bool(ragged))
        assert np.array_equal(scales, z["scales"]), name
        assert np.array_equal(oracle.pack(codes, bits), z["data"]), name
        kern = oracle.encode(codes, bits, KERNEL, tr, tc)
        assert np.array_equal(kern, z["kernel"]), name
        assert np.array_equal(oracle.decode(kern, rows, cols, bits, KERNEL, tr, tc), codes), name
        assert np.array_equal(oracle.dequantize(codes, scales, g), z["deq"]), name
        assert np.array_equal(oracle.f16_round(scales), z["scales_f16"]), name
        a = z["a"]
        f = oracle.gemm_fused(a, kern, rows, bits, g, scales, tr, tc)
        assert np.array_equal(f.view(np.uint32), z["fused"].view(np.uint32)), name
        d = oracle.gemm_dequant(a, codes, g, scales)
        assert np.array_equal(d.view(np.uint32), z["dequant"].view(np.uint32)), name
        o = oracle.gemm_oracle(a, codes, g, scales)
        assert np.array_equal(o.view(np.uint32), z["oracle"].view(np.uint32)), name
        s16 = oracle.f16_round(scales).view(np.float16).astype(np.float32)
        o16 = oracle.gemm_oracle(a, codes, g, s16)
        assert np.array_equal(o16.view(np.uint32), z["oracle_s16"].view(np.uint32)), name


# ---- native layout is a bijection (this repo's own kind) -----------------------------

@pytest.mark.parametrize("bits", [4, 8])
def test_native_layout_bijection(oracle, bits):
    rng = np.random.default_rng(3)
    for rows, cols in [(16, 64), (33, 96), (5, 7), (48, 320)]:
        codes = rng.integers(-(1 << (bits - 1)), 1 << (bits - 1), (rows, cols)).astype(np.int8)
        nat = oracle.encode(codes, bits, NATIVE)
        assert nat.size == oracle.layout_bytes(NATIVE, bits, rows, cols)
        assert np.array_equal(oracle.decode(nat, rows, cols, bits, NATIVE), codes)
        # padding decodes to 0 (offset-binary 0x8 / 0x80)
        slots = oracle.unpack(nat, nat.size * 8 // bits, bits)
        used = np.zeros(slots.size, bool)
        for r in range(rows):
            for c in range(cols):
                used[oracle.layout_index(NATIVE, bits, rows, cols, r, c)] = True
        assert used.sum() == rows * cols and np.all(slots[~used] == 0)


# ---- 3. randomized oracle == reference (only where the reference was built) ----------

@pytest.mark.skipif(not Ref.available(), reason="reference library not built here")
def test_oracle_matches_reference_random(oracle):
    ref = Ref()
    rng = np.random.default_rng(11)
    for trial in range(60):
        bits = 4 if trial % 2 else 8
        g = int(2 ** rng.integers(0, 8))
        cols = int(g * rng.integers(1, 5) + (rng.integers(0, g) if trial % 3 == 0 else 0))
        ragged = cols % g != 0
        rows = int(rng.integers(1, 40))
        amp = float(2.0 ** rng.integers(-12, 12))
        w = (rng.uniform(-amp, amp, (rows, cols))).astype(np.float32)
        data, scales = ref.quantize(w, bits, g, ragged)
        codes, s2 = oracle.quantize(w, bits, g, ragged)
        assert np.array_equal(scales, s2)
        assert np.array_equal(oracle.pack(codes, bits), data)
        m = int(rng.integers(1, 9))
        a = rng.uniform(-2, 2, (m, cols)).astype(np.float32)
        kern = ref.reshuffle(data, rows, cols, bits, g, scales, ROW_MAJOR, KERNEL, ragged=ragged)
        assert np.array_equal(oracle.encode(codes, bits, KERNEL), kern)
        fr, _ = ref.gemm("fused", a, kern, rows, bits, g, scales, KERNEL, ragged=ragged)
        assert np.array_equal(oracle.gemm_fused(a, kern, rows, bits, g, scales), fr)
        orr, _ = ref.gemm("oracle", a, data, rows, bits, g, scales, ROW_MAJOR, ragged=ragged)
        assert np.array_equal(oracle.gemm_oracle(a, codes, g, scales), orr)


def test_oracle_f32_tie_quantize_matches_reference(oracle, golden_ties):
    """The C restatement on f32 weights a third of which sit on, or one ulp beside, a rounding
    tie (not truncated to bf16): bytes and scales equal the reference's (quant.cpp:24-29,49-68)."""
    for name, z in golden_ties.items():
        rows, cols, bits, g, ragged = (int(v) for v in z["meta"])
        codes, scales = oracle.quantize(z["w"], bits, g, bool(ragged))
        assert np.array_equal(scales, z["scales"]), name
        assert np.array_equal(oracle.pack(codes, bits), z["data"]), name
        assert np.array_equal(oracle.f16_round(scales), z["scales_f16"]), name


def test_oracle_gemm_float_matches_reference(oracle, golden_gemm_float):
    """gemm_float (gemm.cpp:111-119), bit-exact."""
    for name, z in golden_gemm_float.items():
        m, k, n, block = (int(v) for v in z["meta"])
        out = oracle.gemm_float(z["a"], z["w"], block)
        assert np.array_equal(out.view(np.uint32), z["out"].view(np.uint32)), name
