"""Generates the RTNCKPT1 fixtures with the reference's own writer (oracle/_ref/make_ckpt, built by
`make -C oracle _ref/make_ckpt` from /root/reference sources):

  tests/golden/toy_q.rtnckpt     3-layer toy model (dim 128, ffn 256, g=128), plan
                                 'explicit:0 modules:4' (layer 0 ffn_down q8, the rest q4)
  tests/golden/toy_f32.rtnckpt   the same model in f32 (quantize-on-load input)
  tests/golden/toy_q_expect.npz  what the reference loader reads back from toy_q.rtnckpt:
                                 per tensor the logical codes and the f32 (f16-widened) scales
"""
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
PLAN = "explicit:0 modules:4"


def main():
    exe = os.path.join(ROOT, "oracle", "_ref", "make_ckpt")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "_ref/make_ckpt"], check=True)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run([exe, d, PLAN], check=True)
        for f in ("toy_q.rtnckpt", "toy_f32.rtnckpt"):
            with open(os.path.join(d, f), "rb") as src, open(os.path.join(HERE, f), "wb") as dst:
                dst.write(src.read())
        raw = open(os.path.join(d, "toy_q.expect"), "rb").read()
    out, off, i = {}, 0, 0
    while off < len(raw):
        rows, cols, bits = np.frombuffer(raw, np.int64, 3, off)
        off += 24
        codes = np.frombuffer(raw, np.int8, rows * cols, off).reshape(rows, cols)
        off += rows * cols
        gpr = -(-cols // 128)
        scales = np.frombuffer(raw, np.float32, rows * gpr, off).reshape(rows, gpr)
        off += rows * gpr * 4
        out[f"t{i}_codes"], out[f"t{i}_scales"], out[f"t{i}_bits"] = codes, scales, np.int64(bits)
        i += 1
    out["plan"] = np.array(PLAN)
    np.savez_compressed(os.path.join(HERE, "toy_q_expect.npz"), **out)
    print(f"{i} tensors", file=sys.stderr)


if __name__ == "__main__":
    main()
