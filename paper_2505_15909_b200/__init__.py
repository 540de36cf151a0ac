"""B200-native rtnq: RTN quantize-and-pack + W4A16/W8A16 weight-only GEMM (sm_100a).

Python is a binding here, not the product: everything below calls the C-ABI of
``librtnq_b200.so`` (include/rtnq_capi.h) through ctypes.  Two surfaces:

* device API (torch CUDA tensors in, torch CUDA tensors out, async on the
  current stream): :func:`quantize_pack`, :class:`QuantWeight`, :func:`linear`,
  :func:`relayout`, :func:`dequantize` -- the performance path;
* host API (numpy in/out, synchronous), named after the reference functions in
  proj/core/include/rtnq/{quant,packing,gemm}.hpp: :func:`quantize_tensor`,
  :func:`reshuffle`, :func:`dequantize_tensor`, :func:`gemm_fused`,
  :func:`gemm_dequant`, :func:`gemm_auto`, :func:`gemm_oracle`,
  :func:`gemm_float`, :func:`compute_scale`, :func:`quantize_group`,
  :func:`dequantize_group`.

There is no CPU fallback: if the library or a GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import plan  # noqa: F401  (selective-precision table, host logic)
from .errors import (CorruptDataError, CudaError, Error, InvalidInputError, PlanError,
                     ShapeError, UnsupportedError, raise_for)

PKG = os.path.dirname(os.path.abspath(__file__))
# RTNQ_LIB: an alternative build of the same library (e.g. the RTNQ_KERNEL_DEBUG profiling build)
LIB_PATH = os.environ.get("RTNQ_LIB") or os.path.join(PKG, "librtnq_b200.so")

F32, F16, BF16 = 0, 1, 2
ROW_MAJOR, KERNEL_INTERLEAVED, NATIVE, NATIVE_I8, NATIVE_I4 = 0, 1, 2, 3, 4
SCALES_REF, SCALES_NATIVE = 0, 1
PATH_FUSED, PATH_DEQUANT_FIRST, PATH_AUTO, PATH_ORACLE = 0, 1, 2, 3
DEFAULT_THRESHOLD = 1024  # kDefaultGemmThreshold, gemm.hpp:16


class Layout(C.Structure):
    _fields_ = [("kind", C.c_int32), ("tile_rows", C.c_int32), ("tile_cols", C.c_int32)]

    def __repr__(self):
        return f"Layout(kind={self.kind}, tile_rows={self.tile_rows}, tile_cols={self.tile_cols})"


def layout(kind=ROW_MAJOR, tile_rows=16, tile_cols=4) -> Layout:
    return Layout(kind, tile_rows, tile_cols)


_lib = None
_i64, _i32, _p, _sz = C.c_int64, C.c_int, C.c_void_p, C.c_size_t


def lib():
    """Load librtnq_b200.so (built in-tree by paper_2505_15909_b200/build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2505_15909_b200.build`")
    L = C.CDLL(LIB_PATH)
    L.rtnq_last_error.restype = C.c_char_p
    L.rtnq_groups_per_row.restype = _i64
    L.rtnq_groups_per_row.argtypes = [_i64, _i32, _i64]
    L.rtnq_layout_slots.restype = _i64
    L.rtnq_layout_slots.argtypes = [Layout, _i32, _i64, _i64]
    L.rtnq_layout_bytes.restype = _i64
    L.rtnq_layout_bytes.argtypes = [Layout, _i32, _i64, _i64]
    L.rtnq_layout_index.restype = _i64
    L.rtnq_layout_index.argtypes = [Layout, _i32, _i64, _i64, _i64, _i64]
    L.rtnq_native_scale_count.restype = _i64
    L.rtnq_native_scale_count.argtypes = [_i64, _i64]
    L.rtnq_dev_quantize_workspace_bytes.restype = _sz
    L.rtnq_dev_quantize_workspace_bytes.argtypes = [_i64, _i64, _i32, _i64, _i32]
    L.rtnq_dev_quantize_pack.argtypes = [_p, _i32, _i64, _i64, _i32, _i64, _i32, _p, _p, _p, _p,
                                         _p, _p, _p, _p, _sz, _p]
    L.rtnq_dev_quantize_workspace_bytes_ex.restype = _sz
    L.rtnq_dev_quantize_workspace_bytes_ex.argtypes = [_i64, _i64, _i32, _i64, _i32, _i32]
    L.rtnq_dev_quantize_pack_ex.argtypes = [_p, _i32, _i64, _i64, _i32, _i64, _i32, _i32, _p, _p, _p,
                                            _p, _p, _p, _p, _p, _sz, _p]
    L.rtnq_dev_relayout.argtypes = [_p, Layout, _p, Layout, _i32, _i64, _i64, _p]
    L.rtnq_dev_native_scales.argtypes = [_p, _i32, _i64, _i64, _p, _p]
    L.rtnq_dev_dequantize.argtypes = [_p, Layout, _i32, _i64, _i64, _i64, _p, _i32, _i32, _p,
                                      _i32, _p]
    L.rtnq_dev_linear_workspace_bytes.restype = _sz
    L.rtnq_dev_linear_workspace_bytes.argtypes = [_i64, _i64, _i64, _i32, _i64, _i32, Layout]
    L.rtnq_dev_linear.argtypes = [_p, _i32, _i64, _i64, _p, Layout, _i32, _i64, _i64, _i32, _p,
                                  _i32, _i32, _p, _i32, _i32, _i64, _p, _p, _p, _sz, _p]
    L.rtnq_dev_linear_ex.argtypes = [_p, _i32, _i64, _i64, _p, Layout, _i32, _i64, _i64, _i32,
                                     _p, _i32, _i32, _p, _i32, _i32, _i64, _p, _p, _p, _sz, _p,
                                     C.c_uint]
    L.rtnq_dev_gemm_float.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _p, _p]
    L.rtnq_dev_check_flag.argtypes = [_p, _p]
    L.rtnq_device_info.argtypes = [_p, _p, _p]
    L.rtnq_compute_scale.argtypes = [_p, _i64, _i32, _p]
    L.rtnq_quantize_group.argtypes = [_p, _i64, _i32, _p, _p, _p]
    L.rtnq_dequantize_group.argtypes = [_p, _i64, C.c_float, _i32, _p]
    L.rtnq_quantize_tensor.argtypes = [_p, _i64, _i64, _i32, _i64, _i32, _p, _p]
    L.rtnq_reshuffle.argtypes = [_p, _i64, Layout, Layout, _i32, _i64, _i64, _p]
    L.rtnq_dequantize_tensor.argtypes = [_p, _i64, Layout, _i32, _i64, _i64, _i64, _i32, _p, _p]
    L.rtnq_gemm.argtypes = [_i32, _p, _i64, _i64, _p, _i64, Layout, _i32, _i64, _i64, _i32, _p,
                            _i64, _p, _p]
    L.rtnq_gemm_float.argtypes = [_p, _i64, _i64, _p, _i64, _i64, _p]
    L.rtnq_dev_add_rmsnorm.argtypes = [_p, _p, _p, _p, _i64, _i64, C.c_float, _p]
    L.rtnq_dev_silu_mul.argtypes = [_p, _p, _i64, _i64, _p]
    L.rtnq_dev_add_rmsnorm_planes.argtypes = [_p, _p, _p, _p, _i64, _i64, C.c_float, _p, _p, _p]
    L.rtnq_dev_silu_mul_planes.argtypes = [_p, _p, _i64, _i64, _p, _p, _p]
    L.rtnq_dev_act_planes.argtypes = [_p, _i32, _i64, _i64, _p, _p, _p]
    L.rtnq_dev_linear_planes.argtypes = [_p, _p, _i64, _i64, _p, Layout, _i32, _i64, _i64, _i32, _p,
                                         _i32, _i32, _p, _i32, _p, _sz, _p, C.c_uint]
    L.rtnq_dev_decode_attention.argtypes = [_p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64,
                                            C.c_float, _p]
    L.rtnq_dev_decode_attention_workspace_bytes.restype = _sz
    L.rtnq_dev_decode_attention_workspace_bytes.argtypes = [_i64, _i64, _i64, _i64]
    L.rtnq_dev_decode_attention_ws.argtypes = [_p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64,
                                               C.c_float, _p, _sz, _p]
    L.rtnq_dev_decode_attention_planes.argtypes = [_p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64, _i64,
                                                   C.c_float, _p, _p, _p, _sz, _p]
    L.rtnq_peer_buffer_bytes.restype = _sz
    L.rtnq_peer_buffer_bytes.argtypes = [_i64]
    L.rtnq_peer_alloc.argtypes = [_i64, C.POINTER(_p)]
    L.rtnq_peer_free.argtypes = [_p]
    L.rtnq_ipc_get_handle.argtypes = [_p, _p]
    L.rtnq_ipc_open.argtypes = [_p, C.POINTER(_p)]
    L.rtnq_ipc_close.argtypes = [_p]
    L.rtnq_peer_enable.argtypes = [_i32, _i32]
    L.rtnq_dev_linear_peer.argtypes = [_p, _p, _p, _i64, _i64, _p, Layout, _i32, _i64, _i64, _i32, _p,
                                       _i32, _i32, _p, _i32, _i32, _i64, _p, _p, _sz, _p, C.c_uint]
    L.rtnq_dev_add_rmsnorm_peer.argtypes = [_p, _p, _i32, _i64, _p, _p, _i64, _i64, C.c_float, _p, _p,
                                            _p]
    L.rtnq_dev_peer_reduce.argtypes = [_p, _i32, _i64, _p, _i64, _i32, _p]
    L.rtnq_f32_to_f16.argtypes = [_p, _i64, _p]
    L.rtnq_f16_to_f32.argtypes = [_p, _i64, _p]
    L.rtnq_plan_resolve.argtypes = [C.c_char_p, _i64, _p, C.c_char_p, _i64, _p]
    L.rtnq_effective_bits.argtypes = [_p, _i64, _p, _p, _i64, _i32, _p]
    _lib = L
    return L


def _check(status):
    if status:
        raise_for(status, lib().rtnq_last_error().decode())


def _np(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---- geometry --------------------------------------------------------------------------

def groups_per_row(g: int, ragged: bool, cols: int) -> int:
    r = lib().rtnq_groups_per_row(g, int(ragged), cols)
    if r < 0:
        _check(-r)
    return int(r)


def layout_bytes(lay: Layout, bits: int, rows: int, cols: int) -> int:
    r = lib().rtnq_layout_bytes(lay, bits, rows, cols)
    if r < 0:
        _check(-r)
    return int(r)


def layout_index(lay: Layout, bits: int, rows: int, cols: int, r: int, c: int) -> int:
    v = lib().rtnq_layout_index(lay, bits, rows, cols, r, c)
    if v < 0:
        _check(-v)
    return int(v)


def native_scale_count(rows: int, gpr: int) -> int:
    return int(lib().rtnq_native_scale_count(rows, gpr))


def device_info():
    sm, ma, mi = C.c_int(), C.c_int(), C.c_int()
    _check(lib().rtnq_device_info(C.byref(sm), C.byref(ma), C.byref(mi)))
    return sm.value, ma.value, mi.value


# ---- device API (torch) --------------------------------------------------------------------

def _torch():
    import torch
    return torch


def _dt(t) -> int:
    torch = _torch()
    return {torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16}[t.dtype]


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


@dataclass
class QuantWeight:
    """A device-resident quantized weight (the B200 counterpart of QuantTensor,
    quant.hpp:26-46).  ``codes``/``scales`` are in the native (tensor-core) order
    unless noted; ``rows`` are output channels, ``cols`` input features."""
    rows: int
    cols: int
    bits: int
    group: int
    ragged: bool
    codes: "object"            # uint8 codes in `layout` (native, or row-major for W8 per-channel)
    scales: "object"           # f16 bits (int16 tensor) in native order
    layout: int = NATIVE       # NATIVE: tcgen05 kind::f16 kernel; NATIVE_I8/I4: kind::i8 kernels
    codes_row_major: "object" = None
    codes_kernel: "object" = None
    scales_f32: "object" = None  # reference order
    scales_f16: "object" = None  # reference order

    @property
    def gpr(self):
        return groups_per_row(self.group, self.ragged, self.cols)

    @property
    def weight_bytes(self):
        """Algorithmic bytes the GEMM must stream: packed codes + f16 scales."""
        return self.rows * self.cols * self.bits // 8 + self.rows * self.gpr * 2


_qflags = {}


def _quant_flag(device, checked: bool):
    """Persistent per-device error flags of quantize_pack (no memset per call): the checked one
    is read and cleared by every check (so it is zero at the next call); the unchecked one only
    accumulates and is never read."""
    torch = _torch()
    key = (str(device), checked)
    f = _qflags.get(key)
    if f is None:
        f = _qflags[key] = torch.zeros(1, dtype=torch.int32, device=device)
    return f


def quantize_pack(w, bits: int, group: int, ragged: bool = False, *, native=None,
                  row_major=False, kernel=False, scales_f32=False, scales_f16=False,
                  check=True, stream=None) -> QuantWeight:
    """RTN quantize-and-pack on the GPU (rtnq_dev_quantize_pack_ex).

    The linear's operand is ``codes`` in ``out.layout``.  With ``native=None`` that is the
    layout of the fastest kernel for the shape: NATIVE_I8 for W8 per-channel and group-128 and
    NATIVE_I4 for W4 group-128 (tcgen05 kind::i8 kernels; one quantize kernel writes their
    tiles directly), else NATIVE (tcgen05 kind::f16 kernel).  ``native=True`` forces NATIVE."""
    torch = _torch()
    assert w.is_cuda and w.dim() == 2 and w.is_contiguous()
    rows, cols = w.shape
    gpr = groups_per_row(group, ragged, cols)
    dev = w.device
    u8 = dict(dtype=torch.uint8, device=dev)
    out = QuantWeight(rows, cols, bits, group, ragged, None, None)
    # default operand: W8 per-channel -> NATIVE_I8, W4 group-128 -> NATIVE_I4 (kind::i8
    # kernels, from the row-major bytes), else NATIVE (kind::f16 kernel)
    imma = None
    if native is None:
        if bits == 8 and (group >= cols or group == 128):
            imma = NATIVE_I8
        elif bits == 4 and group == 128:
            imma = NATIVE_I4
    native = (imma is None) if native is None else native
    if imma is not None:  # one kernel writes the int8-MMA tiles (rtnq_dev_quantize_pack_ex)
        native = False
        out.layout = imma
        out.codes = torch.empty(layout_bytes(layout(imma), bits, rows, cols), **u8)
        out.scales = torch.empty(native_scale_count(rows, gpr), dtype=torch.int16, device=dev)
    if native:
        out.codes = torch.empty(layout_bytes(layout(NATIVE), bits, rows, cols), **u8)
        out.scales = torch.empty(native_scale_count(rows, gpr), dtype=torch.int16, device=dev)
    if row_major:
        out.codes_row_major = torch.empty(layout_bytes(layout(ROW_MAJOR), bits, rows, cols), **u8)
    if kernel:
        out.codes_kernel = torch.empty(layout_bytes(layout(KERNEL_INTERLEAVED), bits, rows, cols),
                                       **u8)
    if scales_f32:
        out.scales_f32 = torch.empty(rows, gpr, dtype=torch.float32, device=dev)
    if scales_f16:
        out.scales_f16 = torch.empty(rows, gpr, dtype=torch.int16, device=dev)
    kind = imma if imma is not None else NATIVE
    wsb = lib().rtnq_dev_quantize_workspace_bytes_ex(rows, cols, bits, group, int(ragged), kind)
    ws = torch.empty(max(wsb, 1), **u8)
    err = _quant_flag(dev, check)
    st = _stream(stream)
    _check(lib().rtnq_dev_quantize_pack_ex(
        _ptr(w), _dt(w), rows, cols, bits, group, int(ragged), kind, _ptr(out.codes_row_major),
        _ptr(out.codes_kernel), _ptr(out.codes), _ptr(out.scales_f32), _ptr(out.scales_f16),
        _ptr(out.scales), _ptr(err), _ptr(ws), wsb, st))
    if check:
        _check(lib().rtnq_dev_check_flag(_ptr(err), st))
    return out


def from_row_major(codes_rm, scales_f16, rows: int, cols: int, bits: int, group: int,
                   ragged: bool = False, stream=None) -> QuantWeight:
    """A QuantWeight from the reference's file form (checkpoint.py): row-major offset-binary
    codes and per-(row, group) IEEE-half scale bits, both already on the device.  The codes
    are relaid out into the layout quantize_pack would pick (NATIVE_I4 / NATIVE_I8 / NATIVE)
    and the scales reordered into the native order."""
    gpr = groups_per_row(group, ragged, cols)
    kind = NATIVE
    if bits == 8 and (group >= cols or group == 128):
        kind = NATIVE_I8
    elif bits == 4 and group == 128:
        kind = NATIVE_I4
    out = QuantWeight(rows, cols, bits, group, ragged, None, None)
    out.layout = kind
    out.codes = relayout(codes_rm, layout(ROW_MAJOR), layout(kind), bits, rows, cols, stream=stream)
    out.scales = native_scales(scales_f16, rows, gpr, stream=stream)
    return out


class Workspace:
    """Zero-initialised scratch for rtnq_dev_linear (stream-K partials and the
    self-resetting per-row-block counters).  Reuse one per stream."""

    def __init__(self, nbytes: int = 0, device="cuda"):
        torch = _torch()
        self.device = device
        self._retired = []
        self.buf = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)

    def ensure(self, nbytes: int):
        torch = _torch()
        if self.buf.numel() < nbytes:
            # keep the old buffer alive: a CUDA graph captured earlier still launches kernels
            # whose stream-K counters and partials live in it
            self._retired.append(self.buf)
            self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        return self.buf


_default_ws = {}


FLAG_PDL = 1


def _default_workspace(device, stream, nbytes, kind="linear"):
    """The per-(kind, device, stream) default workspace: its self-resetting counters and partials
    must not be shared by two streams at once, nor by two kinds of kernel with different
    layouts of the buffer (the linears' stream-K counters vs the attention's split merge)."""
    key = (kind, str(device), _stream(stream).value)
    ws = _default_ws.get(key)
    if ws is None:
        ws = _default_ws[key] = Workspace(nbytes, device)
    return ws


_err_flags = {}


def error_flag(device):
    """A zeroed device int32 flag for the ``err=`` argument of the device API."""
    torch = _torch()
    return torch.zeros(1, dtype=torch.int32, device=device)


def check_flag(err, stream=None):
    """Synchronize ``stream`` and raise InvalidInputError if ``err`` was set (then clear it)
    (rtnq_dev_check_flag)."""
    _check(lib().rtnq_dev_check_flag(_ptr(err), _stream(stream)))


def linear(a, qw: QuantWeight, out=None, out_dtype=None, *, path=PATH_FUSED,
           threshold=DEFAULT_THRESHOLD, workspace: Workspace | None = None, stream=None,
           pdl=False, err=None, check=None):
    """out[m, n] = a[m, k] @ W^T with W = codes * scales (rtnq_dev_linear_ex).

    The tensor-core path runs for bf16/f16 ``a`` against the native layout.
    ``pdl=True`` lets the weight prefetch overlap the previous kernel (the caller
    asserts that kernel does not write this weight).

    Non-finite activations are the reference's InvalidInputError (gemm.cpp:13-19).  With
    ``err`` (a device int32 flag, :func:`error_flag`) the kernels OR 1 into it asynchronously
    and the caller checks it later (:func:`check_flag`, e.g. once per decode step); without it
    (``check`` defaults to True outside CUDA-graph capture) the call synchronizes and raises."""
    torch = _torch()
    assert a.is_cuda and a.dim() == 2 and a.is_contiguous() and a.shape[1] == qw.cols
    m = a.shape[0]
    if out is None:
        out = torch.empty(m, qw.rows, dtype=out_dtype or a.dtype, device=a.device)
    if check is None:
        check = err is None and not torch.cuda.is_current_stream_capturing()
    if check and err is None:
        err = _err_flags.get(str(a.device))
        if err is None:
            err = _err_flags[str(a.device)] = error_flag(a.device)
    lay = layout(qw.layout)
    wsb = lib().rtnq_dev_linear_workspace_bytes(m, qw.rows, qw.cols, qw.bits, qw.group, path, lay)
    if workspace is None:
        workspace = _default_workspace(a.device, stream, wsb)
    buf = workspace.ensure(wsb)
    chosen = C.c_int(-1)
    _check(lib().rtnq_dev_linear_ex(
        _ptr(a), _dt(a), m, qw.cols, _ptr(qw.codes), lay, qw.bits, qw.rows, qw.group,
        int(qw.ragged), _ptr(qw.scales), F16, SCALES_NATIVE, _ptr(out), _dt(out), path,
        threshold, C.byref(chosen), _ptr(err), _ptr(buf), buf.numel(), _stream(stream),
        FLAG_PDL if pdl else 0))
    if check:
        check_flag(err, stream)
    return out


def linear_raw(a, a_dtype, m, k, codes, lay, bits, n, g, ragged, scales, s_dtype, s_order, out,
               out_dtype, path=PATH_FUSED, threshold=DEFAULT_THRESHOLD, err=None, ws=None,
               ws_bytes=0, stream=None):
    """Direct rtnq_dev_linear binding (pointers as torch tensors or None)."""
    chosen = C.c_int(-1)
    _check(lib().rtnq_dev_linear(_ptr(a), a_dtype, m, k, _ptr(codes), lay, bits, n, g,
                                 int(ragged), _ptr(scales), s_dtype, s_order, _ptr(out),
                                 out_dtype, path, threshold, C.byref(chosen), _ptr(err),
                                 _ptr(ws), ws_bytes, _stream(stream)))
    return chosen.value


class Planes:
    """The int8 kernels' activation planes of an [m, k] activation: int8
    [3, m, k] and int32 exponents [m], filled by act_planes or by the fused producers."""

    def __init__(self, m: int, k: int, device="cuda"):
        torch = _torch()
        self.m, self.k = m, k
        self.planes = torch.empty(3, m, k, dtype=torch.int8, device=device)
        self.texp = torch.empty(m, dtype=torch.int32, device=device)


def act_planes(a, planes: Planes, stream=None):
    m, k = a.shape
    _check(lib().rtnq_dev_act_planes(_ptr(a), _dt(a), m, k, _ptr(planes.planes), _ptr(planes.texp),
                                     _stream(stream)))
    return planes


def add_rmsnorm(x, weight, out, delta=None, eps=1e-5, stream=None, planes: Planes | None = None):
    """x += delta (if given); out = rmsnorm(x) * weight.  bf16 [m, h] (rtnq_dev_add_rmsnorm).
    With ``planes`` the same kernel also writes the activation planes of ``out``."""
    m, h = x.shape
    if planes is not None:
        _check(lib().rtnq_dev_add_rmsnorm_planes(_ptr(x), _ptr(delta), _ptr(weight), _ptr(out), m, h,
                                                 eps, _ptr(planes.planes), _ptr(planes.texp),
                                                 _stream(stream)))
        return out
    _check(lib().rtnq_dev_add_rmsnorm(_ptr(x), _ptr(delta), _ptr(weight), _ptr(out), m, h, eps,
                                      _stream(stream)))
    return out


def silu_mul(gate_up, act, stream=None, planes: Planes | None = None):
    """act[m, f] = silu(gate_up[:, :f]) * gate_up[:, f:] (rtnq_dev_silu_mul).  With ``planes``
    the same kernel also writes the activation planes of ``act``."""
    m, f = act.shape
    if planes is not None:
        _check(lib().rtnq_dev_silu_mul_planes(_ptr(gate_up), _ptr(act), m, f, _ptr(planes.planes),
                                              _ptr(planes.texp), _stream(stream)))
        return act
    _check(lib().rtnq_dev_silu_mul(_ptr(gate_up), _ptr(act), m, f, _stream(stream)))
    return act


def linear_planes(planes: Planes, qw: QuantWeight, out, *, workspace: Workspace | None = None,
                  stream=None, pdl=False):
    """The int8 tensor-core linear (NATIVE_I4 / NATIVE_I8 weights) on precomputed planes
    (rtnq_dev_linear_planes): no planes kernel of its own."""
    m, k = planes.m, planes.k
    assert k == qw.cols and qw.layout in (NATIVE_I4, NATIVE_I8)
    wsb = lib().rtnq_dev_linear_workspace_bytes(m, qw.rows, qw.cols, qw.bits, qw.group, PATH_FUSED,
                                                layout(qw.layout))
    if workspace is None:
        workspace = _default_workspace(out.device, stream, wsb)
    buf = workspace.ensure(wsb)
    _check(lib().rtnq_dev_linear_planes(
        _ptr(planes.planes), _ptr(planes.texp), m, k, _ptr(qw.codes), layout(qw.layout), qw.bits, qw.rows,
        qw.group, int(qw.ragged), _ptr(qw.scales), F16, SCALES_NATIVE, _ptr(out), _dt(out), _ptr(buf),
        buf.numel(), _stream(stream), FLAG_PDL if pdl else 0))
    return out


def decode_attention(qkv, k_cache, v_cache, out, hq, hkv, pos, head_dim=128, theta=500000.0,
                     stream=None, workspace: Workspace | None = None, planes: Planes | None = None):
    """GQA decode attention with RoPE over a KV cache (rtnq_dev_decode_attention_planes).  The
    split-merge scratch comes from ``workspace`` (one per stream; the default per (device,
    stream)).  With ``planes`` the kernel also writes the activation planes of ``out`` for the
    int8 o-projection (linear_planes)."""
    batch, max_len = k_cache.shape[0], k_cache.shape[1]
    wsb = lib().rtnq_dev_decode_attention_workspace_bytes(batch, hq, hkv, max_len)
    if workspace is None:
        workspace = _default_workspace(qkv.device, stream, wsb, kind="attention")
    buf = workspace.ensure(wsb)
    _check(lib().rtnq_dev_decode_attention_planes(
        _ptr(qkv), _ptr(k_cache), _ptr(v_cache), _ptr(out), batch, hq, hkv, head_dim, max_len, pos, theta,
        None if planes is None else _ptr(planes.planes), None if planes is None else _ptr(planes.texp),
        _ptr(buf), buf.numel(), _stream(stream)))
    return out


def relayout(src, frm: Layout, to: Layout, bits, rows, cols, stream=None):
    torch = _torch()
    out = torch.empty(layout_bytes(to, bits, rows, cols), dtype=torch.uint8, device=src.device)
    _check(lib().rtnq_dev_relayout(_ptr(src), frm, _ptr(out), to, bits, rows, cols,
                                   _stream(stream)))
    return out


def native_scales(scales, rows, gpr, stream=None):
    torch = _torch()
    out = torch.empty(native_scale_count(rows, gpr), dtype=torch.int16, device=scales.device)
    dt = F32 if scales.dtype == torch.float32 else F16
    _check(lib().rtnq_dev_native_scales(_ptr(scales), dt, rows, gpr, _ptr(out), _stream(stream)))
    return out


def dequantize(codes, lay: Layout, bits, rows, cols, g, scales, s_dtype, s_order,
               out_dtype=None, stream=None):
    torch = _torch()
    out_dtype = out_dtype or torch.float32
    out = torch.empty(rows, cols, dtype=out_dtype, device=codes.device)
    _check(lib().rtnq_dev_dequantize(_ptr(codes), lay, bits, rows, cols, g, _ptr(scales),
                                     s_dtype, s_order, _ptr(out), _dt(out), _stream(stream)))
    return out


# ---- host API (numpy; the reference's function names) --------------------------------------

def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


def compute_scale(values, bits: int) -> float:
    v = _f32(values).ravel()
    out = C.c_float()
    _check(lib().rtnq_compute_scale(_np(v), v.size, bits, C.byref(out)))
    return out.value


def quantize_group(values, bits: int, scale: float | None = None):
    """-> (codes int8, scale).  scale=None computes it (quant.hpp:55-57)."""
    v = _f32(values).ravel()
    codes = np.zeros(v.size, np.int8)
    sin = None if scale is None else C.byref(C.c_float(scale))
    sout = C.c_float()
    _check(lib().rtnq_quantize_group(_np(v), v.size, bits, sin, C.byref(sout), _np(codes)))
    return codes, sout.value


def dequantize_group(codes, scale: float, bits: int):
    c = np.ascontiguousarray(codes, dtype=np.int8).ravel()
    out = np.zeros(c.size, np.float32)
    _check(lib().rtnq_dequantize_group(_np(c), c.size, C.c_float(scale), bits, _np(out)))
    return out


def quantize_tensor(w, bits: int, g: int = 128, ragged: bool = False):
    """-> (row-major packed bytes, f32 scales [rows, gpr]) (quant.hpp:64-67)."""
    w = _f32(w)
    rows, cols = w.shape
    gpr = groups_per_row(g, ragged, cols)
    data = np.zeros((rows * cols * bits + 7) // 8, np.uint8)
    scales = np.zeros((rows, gpr), np.float32)
    _check(lib().rtnq_quantize_tensor(_np(w), rows, cols, bits, g, int(ragged), _np(data),
                                      _np(scales)))
    return data, scales


def reshuffle(data, frm: Layout, to: Layout, bits, rows, cols):
    d = np.ascontiguousarray(data, dtype=np.uint8)
    out = np.zeros(layout_bytes(to, bits, rows, cols), np.uint8)
    _check(lib().rtnq_reshuffle(_np(d), d.size, frm, to, bits, rows, cols, _np(out)))
    return out


def dequantize_tensor(data, lay: Layout, bits, rows, cols, g, scales, ragged=False):
    d = np.ascontiguousarray(data, dtype=np.uint8)
    s = _f32(scales)
    out = np.zeros((rows, cols), np.float32)
    _check(lib().rtnq_dequantize_tensor(_np(d), d.size, lay, bits, rows, cols, g, int(ragged),
                                        _np(s), _np(out)))
    return out


def _gemm(path, a, data, lay, bits, n, g, scales, ragged=False, threshold=DEFAULT_THRESHOLD):
    a = _f32(a)
    m, k = a.shape
    d = np.ascontiguousarray(data, dtype=np.uint8)
    s = _f32(scales)
    out = np.zeros((m, n), np.float32)
    chosen = C.c_int(-1)
    _check(lib().rtnq_gemm(path, _np(a), m, k, _np(d), d.size, lay, bits, n, g, int(ragged),
                           _np(s), threshold, C.byref(chosen), _np(out)))
    return out, chosen.value


def gemm_fused(a, data, lay, bits, n, g, scales, ragged=False):
    return _gemm(PATH_FUSED, a, data, lay, bits, n, g, scales, ragged)[0]


def gemm_dequant(a, data, lay, bits, n, g, scales, ragged=False):
    return _gemm(PATH_DEQUANT_FIRST, a, data, lay, bits, n, g, scales, ragged)[0]


def gemm_oracle(a, data, lay, bits, n, g, scales, ragged=False):
    return _gemm(PATH_ORACLE, a, data, lay, bits, n, g, scales, ragged)[0]


def gemm_auto(a, data, lay, bits, n, g, scales, threshold=DEFAULT_THRESHOLD, ragged=False):
    """-> (out, chosen path: 0 fused / 1 dequant_first) (gemm.hpp:38-40)."""
    return _gemm(PATH_AUTO, a, data, lay, bits, n, g, scales, ragged, threshold)


def f32_to_f16(values):
    """f32 -> binary16 bits, RNE (f16.cpp:8-41)."""
    v = _f32(values).ravel()
    out = np.zeros(v.size, np.uint16)
    _check(lib().rtnq_f32_to_f16(_np(v), v.size, _np(out)))
    return out


def f16_to_f32(bits):
    """binary16 bits -> f32, exact (f16.cpp:43-63)."""
    b = np.ascontiguousarray(bits, dtype=np.uint16).ravel()
    out = np.zeros(b.size, np.float32)
    _check(lib().rtnq_f16_to_f32(_np(b), b.size, _np(out)))
    return out


def gemm_float(a, w, block: int):
    a, w = _f32(a), _f32(w)
    out = np.zeros((a.shape[0], w.shape[0]), np.float32)
    _check(lib().rtnq_gemm_float(_np(a), a.shape[0], a.shape[1], _np(w), w.shape[0], block,
                                 _np(out)))
    return out
