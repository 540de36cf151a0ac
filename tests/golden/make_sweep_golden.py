"""Generates the eval-harness fixtures with the reference's own eval.cpp (oracle/_ref/make_sweep,
built by `make -C oracle _ref/make_sweep` from /root/reference sources) on the default toy
decoder (toy.hpp: 8 layers, dim 64, 4 heads, ffn 256, seq 32, group 64, seed 0), 2 inputs:

  tests/golden/toy_sweeps.csv   horizontal_sweep first/middle/last + vertical_sweep rows
                                (sweep_to_csv format, eval.cpp:226-243)
  tests/golden/toy_compare.txt  compare() reports (eval.cpp:147-182) for four plans + self
  tests/golden/toy_probe.txt    first values of every toy weight tensor and input (PRNG pin)
"""
import os
import shutil
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
N_INPUTS = 2


def main():
    exe = os.path.join(ROOT, "oracle", "_ref", "make_sweep")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "_ref/make_sweep"], check=True)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run([exe, d, str(N_INPUTS)], check=True)
        for f in ("toy_sweeps.csv", "toy_compare.txt", "toy_probe.txt"):
            shutil.copyfile(os.path.join(d, f), os.path.join(HERE, f))


if __name__ == "__main__":
    main()
