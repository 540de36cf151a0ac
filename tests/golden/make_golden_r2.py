"""Round-2 golden fixtures from the UNMODIFIED reference (oracle/_ref/librtnq_ref.so).

    python tests/golden/make_golden_r2.py

* ``quant_f32ties.npz`` -- f32 weights where a third of every group sits exactly on a
  rounding tie or one f32 ulp to either side of it (make_golden.tie_rich), NOT truncated to
  bf16: the reference's quantize_tensor (quant.cpp:100-141) bytes and f32 scales.  These
  exercise the f32-input quantize path's tie handling (common.cuh quantize_one), which the
  bf16-truncated fixtures of make_golden.py cannot reach.
* ``gemm_float.npz`` -- the reference's dense blocked f32 baseline gemm_float
  (gemm.cpp:111-119) on seeded inputs at several block sizes, for the GPU kernel's bit-exact
  test.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, HERE)
from make_golden import tie_rich  # noqa: E402
from oracle import Ref  # noqa: E402


def main():
    ref = Ref()
    ref.set_threads(4)
    rng = np.random.default_rng(20251017)
    arrays, names = {}, []
    for name, rows, cols, bits, g, ragged in [
            ("t_64x512_g128_b4", 64, 512, 4, 128, False),
            ("t_48x1024_g128_b8", 48, 1024, 8, 128, False),
            ("t_40x384_g32_b4", 40, 384, 4, 32, False),
            ("t_33x300_g512r_b8", 33, 300, 8, 512, True),
            ("t_16x4096_g4096_b8", 16, 4096, 8, 4096, False),
            ("t_20x256_g64_b4", 20, 256, 4, 64, False)]:
        w = tie_rich(rng, rows, cols, g, bits)
        data, scales = ref.quantize(w, bits, g, ragged)
        s16 = np.array([ref.f32_to_f16(float(x)) for x in scales.ravel()], np.uint16).reshape(scales.shape)
        for key, val in dict(meta=np.array([rows, cols, bits, g, int(ragged)], np.int64), w=w,
                             data=data, scales=scales, scales_f16=s16).items():
            arrays[f"{name}/{key}"] = val
        names.append(name)
    arrays["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "quant_f32ties.npz"), **arrays)

    gf, gnames = {}, []
    for name, m, k, n, block in [("f_3x256x40_b64", 3, 256, 40, 64), ("f_5x1000x17_b128", 5, 1000, 17, 128),
                                 ("f_1x4096x64_b4096", 1, 4096, 64, 4096), ("f_7x96x33_b1", 7, 96, 33, 1),
                                 ("f_16x512x128_b100", 16, 512, 128, 100)]:
        a = rng.uniform(-1, 1, (m, k)).astype(np.float32)
        w = rng.uniform(-1, 1, (n, k)).astype(np.float32)
        out = ref.gemm_float(a, w, block)
        for key, val in dict(meta=np.array([m, k, n, block], np.int64), a=a, w=w, out=out).items():
            gf[f"{name}/{key}"] = val
        gnames.append(name)
    gf["names"] = np.array(gnames)
    np.savez_compressed(os.path.join(HERE, "gemm_float.npz"), **gf)
    for f in ("quant_f32ties.npz", "gemm_float.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")


if __name__ == "__main__":
    main()
