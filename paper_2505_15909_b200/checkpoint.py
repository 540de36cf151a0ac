"""RTNCKPT1 checkpoints -> GPU kernel operands.

The reference's container (store.hpp:16-31, store.cpp:201-306):

    bytes 0..7   magic "RTNCKPT1"
    bytes 8..15  u64 manifest length (little-endian)
    manifest     sorted-key JSON: format, name, layers, group {g, ragged}, layout, modules
                 [{id, rows, cols}], optional plan / toy, tensors [{layer, module, dtype,
                 data_off, data_len, scales_off, scales_len}] (layer-major, module order 1..4)
    payload      64-byte aligned from 16 + manifest length; blob offsets are relative to it

Quantized tensors ("q4"/"q8") hold offset-binary codes in logical row-major order plus IEEE
half scales; "f32" tensors hold raw row-major weights.  ``read_info`` parses and validates the
header exactly as ``open_checkpoint`` does (same checks, same failure classes as
CorruptDataError); ``load_quantized`` streams one tensor at a time into the GPU kernels'
layout (the row-major bytes are uploaded and relaid out on the device, the f16 scales go to
the native order); ``quantize_on_load`` quantizes an f32 checkpoint on the GPU under a
selective-precision plan (store.cpp:394-422), also one tensor at a time.
"""
from __future__ import annotations

import json
import os
import struct
from dataclasses import dataclass, field

import numpy as np

MAGIC = b"RTNCKPT1"
BLOB_ALIGN = 64
MODULES = ("qkv_proj", "attn_out_proj", "ffn_up", "ffn_down")  # ModuleId 1..4


class CorruptDataError(ValueError):
    """The reference's CorruptDataError (error.hpp): the file is not a valid RTNCKPT1."""


@dataclass(frozen=True)
class TensorRecord:
    layer: int
    module: int  # ModuleId 1..4
    dtype: str   # "f32" | "q8" | "q4"
    data_off: int
    data_len: int
    scales_off: int
    scales_len: int


@dataclass
class CheckpointInfo:
    manifest: dict
    records: list = field(default_factory=list)
    payload_base: int = 0
    file_bytes: int = 0

    @property
    def group(self) -> int:
        return int(self.manifest["group"]["g"])

    @property
    def ragged(self) -> bool:
        return bool(self.manifest["group"]["ragged"])

    def shape(self, module: int):
        for m in self.manifest["modules"]:
            if m["id"] == module:
                return int(m["rows"]), int(m["cols"])
        raise CorruptDataError("module id out of range in manifest")


def _align(n: int, a: int = BLOB_ALIGN) -> int:
    return (n + a - 1) // a * a


def _groups_per_row(g: int, ragged: bool, cols: int) -> int:
    if g < 1 or g & (g - 1):
        raise CorruptDataError("group size must be a positive power of two")
    if cols % g and not ragged:
        raise CorruptDataError("cols is not a multiple of the group size")
    return -(-cols // g)


def _data_length(rows: int, cols: int, dtype: str) -> int:  # store.cpp data_length
    n = rows * cols
    if dtype == "f32":
        return 4 * n
    if dtype == "q8":
        return n
    if dtype == "q4":
        return (n + 1) // 2
    raise CorruptDataError(f"unknown dtype '{dtype}'")


def read_info(path: str) -> CheckpointInfo:
    """Parse and validate the header (store.cpp:201-270); no tensor bytes are read."""
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(16)
        if len(head) < 16 or head[:8] != MAGIC:
            raise CorruptDataError("bad checkpoint magic")
        (mlen,) = struct.unpack("<Q", head[8:16])
        if 16 + mlen > size:
            raise CorruptDataError("manifest length exceeds file size")
        try:
            j = json.loads(f.read(mlen).decode("utf-8"))
            if j["format"] != 1:
                raise CorruptDataError("unsupported checkpoint format version")
            layers, mods = int(j["layers"]), j["modules"]
            g, ragged = int(j["group"]["g"]), bool(j["group"]["ragged"])
        except (KeyError, TypeError, ValueError, UnicodeDecodeError) as e:
            if isinstance(e, CorruptDataError):
                raise
            raise CorruptDataError(f"malformed manifest: {e}") from e
    if not isinstance(mods, list) or len(mods) != 4 or sorted(m.get("id") for m in mods) != [1, 2, 3, 4]:
        raise CorruptDataError("manifest must list exactly four modules")
    if layers < 1:
        raise CorruptDataError("manifest needs at least one layer")
    info = CheckpointInfo(j, [], _align(16 + mlen), size)
    for m in mods:
        if int(m["rows"]) < 1 or int(m["cols"]) < 1:
            raise CorruptDataError("module has empty shape")
        _groups_per_row(g, ragged, int(m["cols"]))
    if info.payload_base > size:
        raise CorruptDataError("missing payload")
    payload = size - info.payload_base
    recs = j.get("tensors")
    if not isinstance(recs, list) or len(recs) != layers * 4:
        raise CorruptDataError("checkpoint must hold exactly layers x 4 tensor records")
    for i, r in enumerate(recs):
        try:
            rec = TensorRecord(int(r["layer"]), int(r["module"]), str(r["dtype"]), int(r["data_off"]),
                               int(r["data_len"]), int(r["scales_off"]), int(r["scales_len"]))
        except (KeyError, TypeError, ValueError) as e:
            raise CorruptDataError(f"malformed tensor record: {e}") from e
        if not 1 <= rec.module <= 4:
            raise CorruptDataError("module id out of range in tensor record")
        if rec.layer != i // 4 or rec.module - 1 != i % 4:
            raise CorruptDataError("tensor records out of canonical order")
        rows, cols = info.shape(rec.module)
        if rec.data_len != _data_length(rows, cols, rec.dtype):
            raise CorruptDataError("tensor data length does not match its shape")
        want_scales = 0 if rec.dtype == "f32" else rows * _groups_per_row(g, ragged, cols) * 2
        if rec.scales_len != want_scales:
            raise CorruptDataError("scale blob length does not match the group spec")
        if rec.data_off % BLOB_ALIGN or rec.scales_off % BLOB_ALIGN:
            raise CorruptDataError("unaligned blob offset")
        if rec.data_off + rec.data_len > payload or rec.scales_off + rec.scales_len > payload:
            raise CorruptDataError("blob extends past end of file")
        info.records.append(rec)
    return info


def _blob(path: str, info: CheckpointInfo, off: int, n: int, dtype) -> np.ndarray:
    return np.fromfile(path, dtype=dtype, count=n // np.dtype(dtype).itemsize,
                       offset=info.payload_base + off)


def load_quantized(path: str, device="cuda", stream=None):
    """All quantized tensors of a q4/q8 checkpoint as device QuantWeights (layer-major, module
    order 1..4), each in its kernel's layout: one tensor's host bytes resident at a time."""
    import torch

    import paper_2505_15909_b200 as rq
    info = read_info(path)
    out = []
    for rec in info.records:
        if rec.dtype == "f32":
            raise CorruptDataError("load_quantized needs a quantized checkpoint (use quantize_on_load)")
        rows, cols = info.shape(rec.module)
        bits = 4 if rec.dtype == "q4" else 8
        codes = torch.from_numpy(_blob(path, info, rec.data_off, rec.data_len, np.uint8)).to(device)
        s16 = torch.from_numpy(_blob(path, info, rec.scales_off, rec.scales_len, np.int16)).to(device)
        out.append(rq.from_row_major(codes, s16, rows, cols, bits, info.group, info.ragged, stream=stream))
    return out


def quantize_on_load(path: str, table, device="cuda", stream=None):
    """Quantize an f32 checkpoint on the GPU under a per-(layer, module) bit table
    (plan.resolve), one tensor at a time (store.cpp:394-422)."""
    import torch

    import paper_2505_15909_b200 as rq
    info = read_info(path)
    out = []
    for rec in info.records:
        if rec.dtype != "f32":
            raise CorruptDataError("quantize_on_load needs an f32 checkpoint")
        rows, cols = info.shape(rec.module)
        w = torch.from_numpy(_blob(path, info, rec.data_off, rec.data_len, np.float32)).to(device)
        bits = int(table[rec.layer][rec.module - 1])
        out.append(rq.quantize_pack(w.view(rows, cols), bits, info.group, info.ragged, stream=stream))
    return out
