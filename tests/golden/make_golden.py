"""Generate the golden parity fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/librtnq_ref.so, i.e.
``make -C oracle`` with /root/reference present):

    python tests/golden/make_golden.py

Every array stored here is an output of the reference library itself
(proj/core/src/{quant,packing,gemm,f16,plan}.cpp via oracle/ref_shim.cpp) on
seeded inputs; the inputs are stored next to the outputs so the fixtures are
self-contained on the GPU box, where /root/reference does not exist.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import KERNEL, ROW_MAJOR, Ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def tie_rich(rng, rows, cols, g, bits):
    """Weights where many elements sit exactly on, or one ulp beside, a rounding tie."""
    w = rng.uniform(-1, 1, size=(rows, cols)).astype(np.float32)
    div = 7.5 if bits == 4 else 127.5
    for r in range(rows):
        for j in range(0, cols, g):
            amp = np.float32(div * 2.0 ** rng.integers(-6, 3))
            grp = w[r, j:j + g]
            grp *= amp
            grp[0] = amp if rng.integers(2) else -amp  # S = amp/div exactly
            s = np.float32(amp / np.float32(div))
            for i in range(1, len(grp), 3):
                t = np.float32((rng.integers(0, int(div)) + 0.5) * s)
                grp[i] = [t, np.nextafter(t, np.float32(0)), np.nextafter(t, np.float32(9e9))][i % 3] \
                    * (1 if rng.integers(2) else -1)
    return w


def main():
    ref = Ref()
    ref.set_threads(4)
    rng = np.random.default_rng(20250515)

    # ---- quantize / layouts / dequantize / GEMMs --------------------------------
    cases = [
        # name, rows, cols, bits, g, ragged, m, tile
        ("q_16x4_g4_b4", 16, 4, 4, 4, False, 3, (16, 4)),
        ("q_2x4_g4_b4", 2, 4, 4, 4, False, 1, (16, 4)),
        ("q_18x12_g4_b4", 18, 12, 4, 4, False, 5, (16, 4)),
        ("q_17x5_g4r_b8", 17, 5, 8, 4, True, 2, (16, 4)),
        ("q_37x256_g64_b4", 37, 256, 4, 64, False, 7, (16, 4)),
        ("q_37x256_g64_b8", 37, 256, 8, 64, False, 7, (16, 4)),
        ("q_2x200_g128r_b4", 2, 200, 4, 128, True, 3, (16, 4)),
        ("q_24x128_g32_b4", 24, 128, 4, 32, False, 17, (16, 4)),
        ("q_64x512_g128_b4", 64, 512, 4, 128, False, 16, (16, 4)),
        ("q_64x512_g128_b8", 64, 512, 8, 128, False, 16, (16, 4)),
        ("q_48x320_g512r_b8", 48, 320, 8, 512, True, 9, (16, 4)),   # per-channel style
        ("q_10x64_g32_b8_t22", 10, 64, 8, 32, False, 6, (2, 2)),
        ("q_33x96_g16_b4_t84", 33, 96, 4, 16, False, 4, (8, 4)),
    ]
    arrays = {}
    names = []
    for name, rows, cols, bits, g, ragged, m, (tr, tc) in cases:
        if rows * cols >= 1024 and "g4" not in name:
            w = tie_rich(rng, rows, cols, g, bits)
        else:
            w = rng.uniform(-2, 2, size=(rows, cols)).astype(np.float32)
        # exact-bf16 weights and activations (the GPU fast path consumes bf16)
        w = (w.view(np.uint32) & 0xFFFF0000).view(np.float32)
        data, scales = ref.quantize(w, bits, g, ragged)
        kern = ref.reshuffle(data, rows, cols, bits, g, scales, ROW_MAJOR, KERNEL, tr, tc, ragged)
        back = ref.reshuffle(kern, rows, cols, bits, g, scales, KERNEL, ROW_MAJOR, tr, tc, ragged)
        assert np.array_equal(back, data)
        deq = ref.dequantize(kern, rows, cols, bits, g, scales, KERNEL, tr, tc, ragged)
        a = rng.uniform(-1, 1, size=(m, cols)).astype(np.float32)
        a = (a.view(np.uint32) & 0xFFFF0000).view(np.float32)
        fused, _ = ref.gemm("fused", a, kern, rows, bits, g, scales, KERNEL, tr, tc, ragged)
        dequant, _ = ref.gemm("dequant", a, data, rows, bits, g, scales, ROW_MAJOR, tr, tc, ragged)
        orac, _ = ref.gemm("oracle", a, data, rows, bits, g, scales, ROW_MAJOR, tr, tc, ragged)
        s16 = np.array([ref.f32_to_f16(float(x)) for x in scales.ravel()],
                       np.uint16).reshape(scales.shape)
        s16w = np.array([ref.f16_to_f32(int(h)) for h in s16.ravel()],
                        np.float32).reshape(scales.shape)
        orac16, _ = ref.gemm("oracle", a, data, rows, bits, g, s16w, ROW_MAJOR, tr, tc, ragged)
        meta = np.array([rows, cols, bits, g, int(ragged), m, tr, tc], np.int64)
        for key, val in dict(meta=meta, w=w, data=data, scales=scales, scales_f16=s16,
                             kernel=kern, deq=deq, a=a, fused=fused, dequant=dequant,
                             oracle=orac, oracle_s16=orac16).items():
            arrays[f"{name}/{key}"] = val
        names.append(name)
    arrays["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "quant_gemm.npz"), **arrays)

    # ---- f16 ------------------------------------------------------------------------
    allh = np.arange(65536, dtype=np.uint32)
    widened = np.array([ref.f16_to_f32(int(h)) for h in allh], np.float32)
    xs = np.concatenate([
        rng.uniform(-70000, 70000, 3000), rng.uniform(-1e-4, 1e-4, 3000),
        rng.uniform(-2, 2, 2000), np.ldexp(1.0, np.arange(-30, 18)).astype(np.float64),
    ]).astype(np.float32)
    narrowed = np.array([ref.f32_to_f16(float(x)) for x in xs], np.uint16)
    np.savez_compressed(os.path.join(OUT, "f16.npz"), widened=widened.view(np.uint32),
                        xs=xs, narrowed=narrowed)

    # ---- plans ----------------------------------------------------------------------
    texts = ["first:1 modules:1+3+4", "first:0", "middle:3 modules:1+2+3+4", "last:2 base:4 high:8",
             "explicit:7,0,5", "  first:1   modules:2  ", "first:1 modules:none", "middle:2",
             "last:3", "explicit:0,2", "middle:1", "explicit:0 modules:4", "first:80",
             "", "frist:1", "first", "first:x", "first:1x", "first:-1", "first:1 modules:5",
             "first:1 modules:0", "first:1 modules:1+1", "first:1 modules:", "first:2 base:8",
             "first:2 high:4", "first:2 base:4 high:4", "first:2 base:5", "middle:1 junk:3",
             "first:1 first:2", "first:1 base:4 modules:2", "explicit:", "explicit:3,3",
             "explicit:1,-2", "first:81", "explicit:80"]
    layers_for = 80
    plan_rows = []
    tables = np.zeros((len(texts), layers_for * 4), np.uint8)
    for i, t in enumerate(texts):
        try:
            tab, canon = ref.resolve_plan(t, layers_for)
            tables[i] = tab
            plan_rows.append((t, canon, 0, -2))
        except Exception as e:  # PlanError / InvalidInput from resolution
            try:
                _, canon = ref.resolve_plan(t, 0)
            except Exception:
                canon = ""
            plan_rows.append((t, canon, int(e.status), int(getattr(e, "offset", -2))))
    t70 = ref.resolve_plan("explicit:0 modules:4", 80)[0]
    eff70 = ref.effective_bits(t70, 80, 1)
    eff70s = ref.effective_bits(t70, 80, 1, include_scales=True)
    t1 = ref.resolve_plan("first:1 modules:1+3+4", 80)[0]
    eff1 = ref.effective_bits(t1, 80, 1)
    np.savez_compressed(
        os.path.join(OUT, "plan.npz"), texts=np.array([r[0] for r in plan_rows]),
        canon=np.array([r[1] for r in plan_rows]), status=np.array([r[2] for r in plan_rows]),
        offset=np.array([r[3] for r in plan_rows]), tables=tables,
        eff=np.array([eff70, eff70s, eff1]))
    for f in ("quant_gemm.npz", "f16.npz", "plan.npz"):
        print(f, os.path.getsize(os.path.join(OUT, f)), "bytes")


if __name__ == "__main__":
    main()
