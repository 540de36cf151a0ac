"""numpy/ctypes front end for the parity checkers.

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline leg and ``--impl reference``) -- never from the product
package.  Two checkers live here:

* ``Oracle`` -- the C restatement in oracle/rtnq_oracle.c (always available; it
  is rebuilt with gcc on demand if the .so is missing).
* ``Ref``    -- the unmodified reference library compiled by oracle/Makefile
  into oracle/_ref/librtnq_ref.so (available where it was built; it travels to
  the GPU box with the repo snapshot).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "librtnq_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librtnq_ref.so")

ROW_MAJOR, KERNEL, NATIVE = 0, 1, 2

_i64, _i32, _u64 = C.c_int64, C.c_int, C.c_uint64
_p = C.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _build_oracle():
    subprocess.run(["make", "-s", "-C", HERE, "_build/librtnq_oracle.so"], check=True)


# ---- the int8-MMA native layouts (numpy restatement of common.cuh i8_slot / i4_slot) ----------
# These are the product's own tensor-core operand orders, not reference
# formats: a fixed permutation (plus re-encoding) of the reference's logical codes.

def _pad128(codes):
    rows, cols = codes.shape
    R, Cc = -(-rows // 128) * 128, -(-cols // 128) * 128
    out = np.zeros((R, Cc), np.int8)
    out[:rows, :cols] = codes
    return out


def encode_native_i8(codes):
    """Signed codes -> NATIVE_I8 bytes: 128x128 tiles (row-blocks outer), byte (r, k) of a
    tile at r*128 + ((k/16) ^ (r%8))*16 + k%16, two's complement."""
    t = _pad128(np.asarray(codes, np.int8))
    R, Cc = t.shape
    t = t.reshape(R // 128, 128, Cc // 128, 128).transpose(0, 2, 1, 3)  # [rb][kt][r][k]
    t = t.reshape(R // 128, Cc // 128, 128, 8, 16)                       # k = 16 * chunk + i
    r = np.arange(128)[:, None]
    phys = np.arange(8)[None, :] ^ (r & 7)                               # [r][chunk] -> slot
    out = np.zeros_like(t)
    out[:, :, r, phys, :] = t[:, :, r, np.arange(8)[None, :], :]
    return out.view(np.uint8).ravel()


def encode_native_i4(codes):
    """Signed 4-bit codes -> NATIVE_I4 bytes: one 8 KiB tile per 128 rows x 128-code group
    (row-blocks outer); row r is 64 bytes, byte p = (code(r, p) << 4) | (code(r, 64 + p) & 15)
    stored at 16 * ((p/16) ^ ((r/2) % 4)) + p % 16."""
    t = _pad128(np.asarray(codes, np.int8))
    R, Cc = t.shape
    nib = (t.astype(np.int16) & 15).astype(np.uint8)
    nib = nib.reshape(R // 128, 128, Cc // 128, 128).transpose(0, 2, 1, 3)
    byte = (nib[..., :64] << 4) | nib[..., 64:]                          # [rb][kt][r][p]
    byte = byte.reshape(R // 128, Cc // 128, 128, 4, 16)
    r = np.arange(128)[:, None]
    phys = np.arange(4)[None, :] ^ ((r >> 1) & 3)
    out = np.zeros_like(byte)
    out[:, :, r, phys, :] = byte[:, :, r, np.arange(4)[None, :], :]
    return out.ravel()


class OracleError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"status {status}: {msg}")
        self.status = status


class Oracle:
    """The C restatement (rtnq_oracle.c)."""

    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            _build_oracle()
        L = self.lib = C.CDLL(ORACLE_SO)
        L.ro_f32_to_f16.restype = C.c_uint16
        L.ro_f32_to_f16.argtypes = [C.c_float]
        L.ro_f16_to_f32.restype = C.c_float
        L.ro_f16_to_f32.argtypes = [C.c_uint16]
        L.ro_compute_scale.argtypes = [_p, _i64, _i32, _p]
        L.ro_quantize_tensor.argtypes = [_p, _i64, _i64, _i32, _i64, _i32, _p, _p]
        L.ro_groups_per_row.restype = _i64
        L.ro_groups_per_row.argtypes = [_i64, _i32, _i64]
        L.ro_packed_size.restype = _i64
        L.ro_packed_size.argtypes = [_i64, _i32]
        L.ro_pack.argtypes = [_p, _i64, _i32, _p]
        L.ro_unpack.argtypes = [_p, _i64, _i32, _p]
        L.ro_layout_index.restype = _i64
        L.ro_layout_index.argtypes = [_i32, _i32, _i32, _i32, _i64, _i64, _i64, _i64]
        L.ro_layout_slots.restype = _i64
        L.ro_layout_slots.argtypes = [_i32, _i32, _i32, _i32, _i64, _i64]
        L.ro_layout_bytes.restype = _i64
        L.ro_layout_bytes.argtypes = [_i32, _i32, _i32, _i32, _i64, _i64]
        L.ro_encode_layout.argtypes = [_p, _i64, _i64, _i32, _i32, _i32, _i32, _p]
        L.ro_decode_layout.argtypes = [_p, _i64, _i64, _i32, _i32, _i32, _i32, _p]
        L.ro_native_scale_count.restype = _i64
        L.ro_native_scale_count.argtypes = [_i64, _i64]
        L.ro_native_scales.argtypes = [_p, _i64, _i64, _p]
        L.ro_dequantize.argtypes = [_p, _p, _i64, _i64, _i64, _p]
        L.ro_gemm_fused.argtypes = [_p, _i64, _i64, _p, _i32, _i32, _i32, _i64, _i64, _p, _p]
        L.ro_gemm_dequant.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _p, _p]
        L.ro_gemm_oracle.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _p, _p]
        L.ro_gemm_oracle_f64.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _p, _p]
        L.ro_gemm_float.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _p]
        L.ro_xoshiro_fill_unit.argtypes = [_u64, _u64, _p, _i64, C.c_float]

    # -- scalars -------------------------------------------------------------
    def f32_to_f16(self, x: float) -> int:
        return int(self.lib.ro_f32_to_f16(C.c_float(x)))

    def f16_to_f32(self, h: int) -> float:
        return float(self.lib.ro_f16_to_f32(C.c_uint16(h)))

    def f16_round(self, s: np.ndarray) -> np.ndarray:
        """f32 -> f16 bits (vectorised through numpy; checked equal to ro_f32_to_f16)."""
        with np.errstate(over="ignore"):
            return np.ascontiguousarray(s, dtype=np.float32).astype(np.float16).view(np.uint16)

    def compute_scale(self, v, bits):
        v = np.ascontiguousarray(v, dtype=np.float32)
        out = np.zeros(1, np.float32)
        st = self.lib.ro_compute_scale(_ptr(v), v.size, bits, _ptr(out))
        if st:
            raise OracleError(st)
        return float(out[0])

    def groups_per_row(self, g, ragged, cols):
        r = self.lib.ro_groups_per_row(g, int(ragged), cols)
        if r < 0:
            raise OracleError(-r)
        return int(r)

    # -- quantize / pack -----------------------------------------------------
    def quantize(self, w, bits, g, ragged=False):
        """-> (logical int8 codes [rows, cols], f32 scales [rows, gpr])."""
        w = np.ascontiguousarray(w, dtype=np.float32)
        rows, cols = w.shape
        gpr = self.groups_per_row(g, ragged, cols)
        codes = np.zeros((rows, cols), np.int8)
        scales = np.zeros((rows, gpr), np.float32)
        st = self.lib.ro_quantize_tensor(_ptr(w), rows, cols, bits, g, int(ragged),
                                         _ptr(codes), _ptr(scales))
        if st:
            raise OracleError(st)
        return codes, scales

    def pack(self, codes, bits):
        codes = np.ascontiguousarray(codes, dtype=np.int8).ravel()
        out = np.zeros(self.lib.ro_packed_size(codes.size, bits), np.uint8)
        st = self.lib.ro_pack(_ptr(codes), codes.size, bits, _ptr(out))
        if st:
            raise OracleError(st)
        return out

    def unpack(self, data, n, bits):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        out = np.zeros(n, np.int8)
        self.lib.ro_unpack(_ptr(data), n, bits, _ptr(out))
        return out

    def layout_bytes(self, kind, bits, rows, cols, tr=16, tc=4):
        return int(self.lib.ro_layout_bytes(kind, tr, tc, bits, rows, cols))

    def layout_index(self, kind, bits, rows, cols, r, c, tr=16, tc=4):
        return int(self.lib.ro_layout_index(kind, tr, tc, bits, rows, cols, r, c))

    def encode(self, logical, bits, kind, tr=16, tc=4):
        logical = np.ascontiguousarray(logical, dtype=np.int8)
        rows, cols = logical.shape
        out = np.zeros(self.layout_bytes(kind, bits, rows, cols, tr, tc), np.uint8)
        self.lib.ro_encode_layout(_ptr(logical), rows, cols, bits, kind, tr, tc, _ptr(out))
        return out

    def decode(self, data, rows, cols, bits, kind, tr=16, tc=4):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        out = np.zeros((rows, cols), np.int8)
        self.lib.ro_decode_layout(_ptr(data), rows, cols, bits, kind, tr, tc, _ptr(out))
        return out

    def native_scales(self, scales_f16_bits, rows, gpr):
        s = np.ascontiguousarray(scales_f16_bits, dtype=np.uint16)
        out = np.zeros(self.lib.ro_native_scale_count(rows, gpr), np.uint16)
        self.lib.ro_native_scales(_ptr(s), rows, gpr, _ptr(out))
        return out

    def dequantize(self, logical, scales, g):
        logical = np.ascontiguousarray(logical, dtype=np.int8)
        scales = np.ascontiguousarray(scales, dtype=np.float32)
        rows, cols = logical.shape
        out = np.zeros((rows, cols), np.float32)
        self.lib.ro_dequantize(_ptr(logical), _ptr(scales), rows, cols, g, _ptr(out))
        return out

    # -- GEMMs ---------------------------------------------------------------
    def gemm_fused(self, a, kernel_bytes, n, bits, g, scales, tr=16, tc=4):
        a = np.ascontiguousarray(a, dtype=np.float32)
        m, k = a.shape
        kb = np.ascontiguousarray(kernel_bytes, dtype=np.uint8)
        s = np.ascontiguousarray(scales, dtype=np.float32)
        out = np.zeros((m, n), np.float32)
        self.lib.ro_gemm_fused(_ptr(a), m, k, _ptr(kb), bits, tr, tc, n, g, _ptr(s), _ptr(out))
        return out

    def _g3(self, fn, a, logical, g, scales, dtype=np.float32):
        a = np.ascontiguousarray(a, dtype=np.float32)
        logical = np.ascontiguousarray(logical, dtype=np.int8)
        s = np.ascontiguousarray(scales, dtype=np.float32)
        m, k = a.shape
        n = logical.shape[0]
        out = np.zeros((m, n), dtype)
        fn(_ptr(a), m, k, _ptr(logical), n, g, _ptr(s), _ptr(out))
        return out

    def gemm_dequant(self, a, logical, g, scales):
        return self._g3(self.lib.ro_gemm_dequant, a, logical, g, scales)

    def gemm_oracle(self, a, logical, g, scales):
        return self._g3(self.lib.ro_gemm_oracle, a, logical, g, scales)

    def gemm_oracle_f64(self, a, logical, g, scales):
        return self._g3(self.lib.ro_gemm_oracle_f64, a, logical, g, scales, np.float64)

    def gemm_float(self, a, w, block):
        a = np.ascontiguousarray(a, dtype=np.float32)
        w = np.ascontiguousarray(w, dtype=np.float32)
        out = np.zeros((a.shape[0], w.shape[0]), np.float32)
        self.lib.ro_gemm_float(_ptr(a), a.shape[0], a.shape[1], _ptr(w), w.shape[0], block,
                               _ptr(out))
        return out

    def xoshiro(self, seed, stream, n, mult=1.0):
        out = np.zeros(n, np.float32)
        self.lib.ro_xoshiro_fill_unit(seed, stream, _ptr(out), n, mult)
        return out


class Ref:
    """The unmodified reference library (oracle/_ref/librtnq_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        L = self.lib = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_f32_to_f16.restype = C.c_uint16
        L.ref_f32_to_f16.argtypes = [C.c_float]
        L.ref_f16_to_f32.restype = C.c_float
        L.ref_f16_to_f32.argtypes = [C.c_uint16]
        L.ref_compute_scale.argtypes = [_p, _i64, _i32, _p]
        L.ref_quantize_group.argtypes = [_p, _i64, _i32, _p, _p]
        L.ref_quantize_tensor.argtypes = [_p, _i64, _i64, _i32, _i64, _i32, _p, _p]
        L.ref_layout_slots.restype = _i64
        L.ref_layout_slots.argtypes = [_i32, _i32, _i32, _i64, _i64]
        L.ref_reshuffle.argtypes = [_p, _i64, _i64, _i64, _i32, _i64, _i32, _i32, _i32, _i32,
                                    _i32, _p, _p]
        L.ref_dequantize.argtypes = [_p, _i64, _i64, _i64, _i32, _i64, _i32, _i32, _i32, _i32,
                                     _p, _p]
        L.ref_gemm.argtypes = [_i32, _p, _i64, _i64, _p, _i64, _i64, _i32, _i64, _i32, _i32,
                               _i32, _i32, _p, _i64, _p, _p]
        L.ref_gemm_float.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _p]
        L.ref_resolve_plan.argtypes = [C.c_char_p, _i64, _p, _p, C.c_char_p, _i64]
        L.ref_effective_bits.argtypes = [_p, _i64, _i32, _i64, _i64, _i64, _i32, _p]
        L.ref_set_threads.argtypes = [_i32]

    def _chk(self, st):
        if st:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def set_threads(self, n):
        self.lib.ref_set_threads(n)

    def threads(self):
        return int(self.lib.ref_threads())

    def f32_to_f16(self, x):
        return int(self.lib.ref_f32_to_f16(C.c_float(x)))

    def f16_to_f32(self, h):
        return float(self.lib.ref_f16_to_f32(C.c_uint16(h)))

    def compute_scale(self, v, bits):
        v = np.ascontiguousarray(v, dtype=np.float32)
        out = np.zeros(1, np.float32)
        self._chk(self.lib.ref_compute_scale(_ptr(v), v.size, bits, _ptr(out)))
        return float(out[0])

    def quantize(self, w, bits, g, ragged=False):
        """-> (row-major packed bytes, f32 scales [rows, gpr])."""
        w = np.ascontiguousarray(w, dtype=np.float32)
        rows, cols = w.shape
        gpr = -(-cols // g)
        data = np.zeros((rows * cols * bits + 7) // 8, np.uint8)
        scales = np.zeros((rows, gpr), np.float32)
        self._chk(self.lib.ref_quantize_tensor(_ptr(w), rows, cols, bits, g, int(ragged),
                                               _ptr(data), _ptr(scales)))
        return data, scales

    def reshuffle(self, data, rows, cols, bits, g, scales, frm, to, tr=16, tc=4, ragged=False):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        s = np.ascontiguousarray(scales, dtype=np.float32)
        slots = self.lib.ref_layout_slots(to, tr, tc, rows, cols)
        out = np.zeros((slots * bits + 7) // 8, np.uint8)
        self._chk(self.lib.ref_reshuffle(_ptr(data), data.size, rows, cols, bits, g,
                                         int(ragged), frm, to, tr, tc, _ptr(s), _ptr(out)))
        return out

    def dequantize(self, data, rows, cols, bits, g, scales, layout, tr=16, tc=4, ragged=False):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        s = np.ascontiguousarray(scales, dtype=np.float32)
        out = np.zeros((rows, cols), np.float32)
        self._chk(self.lib.ref_dequantize(_ptr(data), data.size, rows, cols, bits, g,
                                          int(ragged), layout, tr, tc, _ptr(s), _ptr(out)))
        return out

    def gemm(self, which, a, data, n, bits, g, scales, layout, tr=16, tc=4, ragged=False,
             threshold=1024):
        """which: 'fused' | 'dequant' | 'oracle' | 'auto' -> (out, chosen)."""
        w = {"fused": 0, "dequant": 1, "oracle": 2, "auto": 3}[which]
        a = np.ascontiguousarray(a, dtype=np.float32)
        data = np.ascontiguousarray(data, dtype=np.uint8)
        s = np.ascontiguousarray(scales, dtype=np.float32)
        m, k = a.shape
        out = np.zeros((m, n), np.float32)
        chosen = C.c_int(-1)
        self._chk(self.lib.ref_gemm(w, _ptr(a), m, k, _ptr(data), data.size, n, bits, g,
                                    int(ragged), layout, tr, tc, _ptr(s), threshold,
                                    C.byref(chosen), _ptr(out)))
        return out, chosen.value

    def gemm_float(self, a, w, block):
        a = np.ascontiguousarray(a, dtype=np.float32)
        w = np.ascontiguousarray(w, dtype=np.float32)
        out = np.zeros((a.shape[0], w.shape[0]), np.float32)
        self._chk(self.lib.ref_gemm_float(_ptr(a), a.shape[0], a.shape[1], _ptr(w), w.shape[0],
                                          block, _ptr(out)))
        return out

    def resolve_plan(self, text, layers):
        """-> (table uint8[layers*4] or None, canonical text); raises OracleError(4) with .offset."""
        table = np.zeros(max(layers, 0) * 4, np.uint8)
        off = C.c_int64(-2)
        canon = C.create_string_buffer(512)
        st = self.lib.ref_resolve_plan(text.encode(), layers, _ptr(table), C.byref(off), canon,
                                       512)
        if st:
            e = OracleError(st, self.lib.ref_last_error().decode())
            e.offset = off.value
            raise e
        return (table if layers > 0 else None), canon.value.decode()

    def effective_bits(self, table, layers, kind, rows=0, cols=0, g=128, include_scales=False):
        t = np.ascontiguousarray(table, dtype=np.uint8)
        out = C.c_double(0)
        self._chk(self.lib.ref_effective_bits(_ptr(t), layers, kind, rows, cols, g,
                                              int(include_scales), C.byref(out)))
        return out.value
