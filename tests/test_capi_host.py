"""CPU-side checks of the product library: it loads without a GPU, exports every
symbol include/rtnq_capi.h declares, its geometry helpers agree with the oracle,
the selective-precision plan logic matches the reference, and compute entry
points fail loudly (no CPU fallback) when there is no device."""
import os
import re

import numpy as np
import pytest

import paper_2505_15909_b200 as rq
from conftest import ROOT, has_gpu
from oracle import KERNEL, NATIVE, ROW_MAJOR
from oracle import encode_native_i4, encode_native_i8


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "rtnq_capi.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)  # declarations only, not comments
    return sorted(set(re.findall(r"^[a-z0-9_ ]+\**\s*\**(rtnq_[a-z0-9_]+)\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    lib = rq.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_geometry_matches_oracle(oracle):
    rng = np.random.default_rng(5)
    for kind, ok in ((rq.ROW_MAJOR, ROW_MAJOR), (rq.KERNEL_INTERLEAVED, KERNEL), (rq.NATIVE, NATIVE)):
        for bits in (4, 8):
            for rows, cols in ((16, 64), (17, 5), (33, 96), (300, 520)):
                lay = rq.layout(kind)
                assert rq.layout_bytes(lay, bits, rows, cols) == oracle.layout_bytes(ok, bits, rows, cols)
                for _ in range(50):
                    r, c = int(rng.integers(rows)), int(rng.integers(cols))
                    assert rq.layout_index(lay, bits, rows, cols, r, c) == \
                        oracle.layout_index(ok, bits, rows, cols, r, c)
    with pytest.raises(rq.ShapeError):
        rq.layout_index(rq.layout(rq.ROW_MAJOR), 4, 2, 2, 2, 0)
    assert rq.groups_per_row(128, False, 256) == 2
    with pytest.raises(rq.ShapeError):
        rq.groups_per_row(128, False, 200)
    with pytest.raises(rq.InvalidInputError):
        rq.groups_per_row(96, False, 192)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_compute_fails_loudly_without_gpu():
    with pytest.raises(rq.CudaError):
        rq.quantize_tensor(np.ones((2, 4), np.float32), 4, 4)


# ---- selective precision (plan.hpp); the reference's test_plan.cpp cases -------------

def test_plan_golden(golden_plan):
    z = golden_plan
    for text, canon, status, offset, table in zip(z["texts"], z["canon"], z["status"],
                                                  z["offset"], z["tables"]):
        text = str(text)
        if status == 0:
            t, c = rq.plan.resolve(text, 80)
            assert c == str(canon), text
            assert np.array_equal(t.ravel(), table), text
        elif status == 4:
            with pytest.raises(rq.PlanError) as e:
                rq.plan.resolve(text, 80)
            want = None if offset == -1 else int(offset)
            assert e.value.offset == want, (text, e.value.offset, want)
        else:
            with pytest.raises(rq.Error):
                rq.plan.resolve(text, 80)


def test_plan_kats():
    # proj/tests/test_plan.cpp:112-153
    t, _ = rq.plan.resolve("first:1 modules:1+3+4", 80)
    assert t[0].tolist() == [8, 4, 8, 8] and (t == 8).sum() == 3
    t, _ = rq.plan.resolve("middle:2", 6)
    assert [list(r) for r in t] == [[4] * 4, [4] * 4, [8] * 4, [8] * 4, [4] * 4, [4] * 4]
    t, _ = rq.plan.resolve("last:3", 10)
    assert (t == 8).sum() == 12 and t[6, 3] == 4 and t[7, 0] == 8
    with pytest.raises(rq.PlanError):
        rq.plan.resolve("first:7", 6)
    with pytest.raises(rq.PlanError):
        rq.plan.resolve("explicit:4", 4)
    # canonical rendering round trip (test_plan.cpp:90-110)
    for text in ("first:0 modules:1+2+3+4 base:4 high:8", "middle:2 modules:2 base:4 high:8",
                 "last:7 modules:none base:4 high:8", "explicit:0,5,7 modules:3+4 base:4 high:8"):
        assert rq.plan.canonical(text) == text
    assert rq.plan.canonical("explicit:7,0,5") == "explicit:0,5,7 modules:1+2+3+4 base:4 high:8"


def test_effective_bits(golden_plan):
    # uniform manifest: exact 4 / 6 / 5 bits (test_plan.cpp:155-174)
    rows4, cols4 = [64] * 4, [64] * 4
    for text, want in (("first:0", 4.0), ("first:8", 8.0), ("first:4", 6.0), ("middle:2", 5.0)):
        t, _ = rq.plan.resolve(text, 8)
        assert rq.plan.effective_bits(t, rows4, cols4, 32) == want
    t, _ = rq.plan.resolve("first:0", 8)
    assert rq.plan.effective_bits(t, rows4, cols4, 32, include_scales=True) == 4.5
    # 70B manifest (plan.cpp:275-286): explicit:0 modules:4 and first:1 modules:1+3+4
    r70 = [8192 + 2048, 8192, 2 * 28672, 8192]
    c70 = [8192, 8192, 8192, 28672]
    eff = golden_plan["eff"]
    t, _ = rq.plan.resolve("explicit:0 modules:4", 80)
    assert rq.plan.effective_bits(t, r70, c70, 128) == eff[0]
    assert rq.plan.effective_bits(t, r70, c70, 128, include_scales=True) == eff[1]
    t, _ = rq.plan.resolve("first:1 modules:1+3+4", 80)
    e1 = rq.plan.effective_bits(t, r70, c70, 128)
    assert e1 == eff[2] and abs((e1 - 4.0) - 47.0 / 1020.0) < 1e-12


def test_f16_conversions_match_reference_golden(golden_f16):
    # f16.cpp:8-63 through the C-ABI, against the reference-generated fixture
    # (tests/golden/f16.npz: narrowed xs, and every one of the 65536 encodings widened)
    xs = golden_f16["xs"].astype(np.float32)
    assert np.array_equal(rq.f32_to_f16(xs), golden_f16["narrowed"].astype(np.uint16))
    allbits = np.arange(65536, dtype=np.uint16)
    widened = rq.f16_to_f32(allbits)
    ref = golden_f16["widened"].view(np.float32)  # stored as f32 bit patterns
    same = widened.view(np.uint32) == ref.view(np.uint32)
    assert np.all(same | (np.isnan(widened) & np.isnan(ref)))


@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("rows,cols", [(130, 208), (128, 128), (5, 96), (256, 384)])
def test_int8_mma_layouts_match_numpy_restatement(bits, rows, cols):
    """NATIVE_I8 / NATIVE_I4 (the kind::i8 kernels' operands): the host layout index of
    every sampled code agrees with the numpy restatement's encoding, sizes included."""
    rng = np.random.default_rng(rows * cols + bits)
    lo, hi = (-128, 127) if bits == 8 else (-8, 7)
    codes = rng.integers(lo, hi + 1, (rows, cols)).astype(np.int8)
    kind, enc = (rq.NATIVE_I8, encode_native_i8) if bits == 8 else (rq.NATIVE_I4, encode_native_i4)
    e = enc(codes)
    lay = rq.layout(kind)
    assert e.size == rq.layout_bytes(lay, bits, rows, cols)
    for r, c in zip(rng.integers(0, rows, 400), rng.integers(0, cols, 400)):
        idx = rq.layout_index(lay, bits, rows, cols, int(r), int(c))
        if bits == 8:
            v = int(e[idx].astype(np.int8))
        else:
            b = int(e[idx >> 1])
            v = (((b >> 4) if idx & 1 else (b & 15)) ^ 8) - 8
        assert v == int(codes[r, c]), (r, c)


def test_peer_abi_validates_before_touching_a_device():
    """The tensor-parallel peer C-ABI: buffer sizing, and argument errors reported
    as statuses before any CUDA call (so they hold without a GPU)."""
    import ctypes as C
    L = rq.lib()
    # header 256 B + [2 parities][8 ranks][cap] bf16 slots
    assert L.rtnq_peer_buffer_bytes(8) == 256 + 2 * 8 * 8 * 2
    assert L.rtnq_peer_buffer_bytes(4096 * 16) == 256 + 2 * 8 * 4096 * 16 * 2
    assert L.rtnq_peer_buffer_bytes(-1) == 0
    bufs = (C.c_void_p * 2)(None, None)
    lay = rq.layout(rq.NATIVE_I4)
    # null peer buffer -> InvalidInputError
    st = L.rtnq_dev_linear_peer(C.c_void_p(16), None, None, 4, 128, C.c_void_p(16), lay, 4, 128, 128, 0,
                                C.c_void_p(16), rq.F16, rq.SCALES_NATIVE, bufs, 2, 0, 4096, None, None, 0,
                                None, 0)
    assert st == 1 and b"peer" in L.rtnq_last_error()
    # both activations and planes given -> InvalidInputError
    st = L.rtnq_dev_linear_peer(C.c_void_p(16), C.c_void_p(16), C.c_void_p(16), 4, 128, C.c_void_p(16), lay, 4,
                                128, 128, 0, C.c_void_p(16), rq.F16, rq.SCALES_NATIVE, bufs, 2, 0, 4096, None,
                                None, 0, None, 0)
    assert st == 1
    # world outside 1..8, capacity not a multiple of 8
    assert L.rtnq_dev_peer_reduce(C.c_void_p(256), 9, 4096, C.c_void_p(16), 8, 0, None) == 1
    assert L.rtnq_dev_peer_reduce(C.c_void_p(256), 2, 4097, C.c_void_p(16), 8, 0, None) == 1
    assert L.rtnq_dev_add_rmsnorm_peer(C.c_void_p(16), C.c_void_p(256), 2, 4096, C.c_void_p(16), C.c_void_p(16),
                                       2, 100, 1e-5, None, None, None) == 2  # h % 16 != 0: ShapeError
