"""RTNCKPT1 -> GPU against fixtures written and read back by the reference's own
store.cpp (tests/golden/make_ckpt_golden.py): header parsing and validation on CPU; on the GPU,
load_quantized reproduces the reference loader's codes and scales bit for bit, and
quantize_on_load of the f32 checkpoint reproduces the reference's quantized checkpoint."""
import os
import shutil
import struct

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2505_15909_b200 import checkpoint as ck

QF = os.path.join(GOLDEN, "toy_q.rtnckpt")
FF = os.path.join(GOLDEN, "toy_f32.rtnckpt")


def expect():
    return np.load(os.path.join(GOLDEN, "toy_q_expect.npz"))


def test_read_info_matches_reference_header():
    info = ck.read_info(QF)
    assert info.manifest["layers"] == 3 and info.group == 128 and not info.ragged
    assert len(info.records) == 12
    z = expect()
    for i, r in enumerate(info.records):
        assert (r.layer, r.module) == (i // 4, i % 4 + 1)
        assert r.dtype == ("q8" if int(z[f"t{i}_bits"]) == 8 else "q4")
        assert info.shape(r.module) == z[f"t{i}_codes"].shape
    assert all(r.dtype == "f32" for r in ck.read_info(FF).records)


@pytest.mark.parametrize("damage", ["magic", "truncate", "mlen", "align", "order"])
def test_corrupt_checkpoints_are_rejected(tmp_path, damage):
    p = tmp_path / "bad.rtnckpt"
    shutil.copy(QF, p)
    raw = bytearray(open(p, "rb").read())
    if damage == "magic":
        raw[0:8] = b"RTNCKPT2"
    elif damage == "truncate":
        raw = raw[: len(raw) - 1000]
    elif damage == "mlen":
        raw[8:16] = struct.pack("<Q", len(raw))
    else:
        (mlen,) = struct.unpack("<Q", raw[8:16])
        text = raw[16:16 + mlen].decode()
        text = (text.replace('"data_off":25344', '"data_off":25345') if damage == "align"
                else text.replace('"layer":0,"module":1', '"layer":0,"module":2', 1))
        assert len(text) == mlen
        raw[16:16 + mlen] = text.encode()
    open(p, "wb").write(bytes(raw))
    with pytest.raises(ck.CorruptDataError):
        ck.read_info(str(p))


@pytest.mark.gpu
def test_load_quantized_matches_reference_loader(oracle):
    import torch

    import paper_2505_15909_b200 as rq
    z = expect()
    qs = ck.load_quantized(QF)
    for i, q in enumerate(qs):
        codes, scales = z[f"t{i}_codes"], z[f"t{i}_scales"]
        wd = rq.dequantize(q.codes, rq.layout(q.layout), q.bits, q.rows, q.cols, q.group, q.scales, rq.F16,
                           rq.SCALES_NATIVE, torch.float32).cpu().numpy()
        ref = codes.astype(np.float32) * np.repeat(scales, 128, axis=1)[:, : q.cols]
        assert np.array_equal(wd, ref), i  # code * f16-widened scale, one f32 rounding: exact


@pytest.mark.gpu
def test_quantize_on_load_matches_reference_checkpoint(oracle):
    import torch

    import paper_2505_15909_b200 as rq
    z = expect()
    table = np.array([[int(z[f"t{4 * l + m}_bits"]) for m in range(4)] for l in range(3)])
    qs = ck.quantize_on_load(FF, table)
    for i, q in enumerate(qs):
        wd = rq.dequantize(q.codes, rq.layout(q.layout), q.bits, q.rows, q.cols, q.group, q.scales, rq.F16,
                           rq.SCALES_NATIVE, torch.float32).cpu().numpy()
        ref = z[f"t{i}_codes"].astype(np.float32) * np.repeat(z[f"t{i}_scales"], 128, axis=1)[:, : q.cols]
        assert np.array_equal(wd, ref), i
