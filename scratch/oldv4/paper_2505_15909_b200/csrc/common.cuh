// common.cuh -- shared device helpers: element types, the reference's scalar
// quantization rules, and the three code layouts.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/rtnq_capi.h"

namespace rtnq_b200 {

// ---- element loads/stores ------------------------------------------------------------
__device__ __forceinline__ float load_elem(const void* p, int dtype, int64_t i) {
    if (dtype == RTNQ_F32) return static_cast<const float*>(p)[i];
    if (dtype == RTNQ_F16) return __half2float(static_cast<const __half*>(p)[i]);
    return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}

__device__ __forceinline__ void store_elem(void* p, int dtype, int64_t i, float v) {
    if (dtype == RTNQ_F32) static_cast<float*>(p)[i] = v;
    else if (dtype == RTNQ_F16) static_cast<__half*>(p)[i] = __float2half_rn(v);
    else static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
}

// ---- the reference's scalar rules --------------------------------------------------------
__device__ __forceinline__ int qmin_of(int bits) { return -(1 << (bits - 1)); }
__device__ __forceinline__ int qmax_of(int bits) { return (1 << (bits - 1)) - 1; }

// compute_scale's last step (quant.cpp:64-67): the f64 quotient absmax/divisor,
// rounded upward to f32.  __double2float_ru(x) == the reference's
// "static_cast<float>, then nextafter upward if it rounded down".
__device__ __forceinline__ float scale_from_absmax(float absmax, int bits) {
    if (absmax == 0.0f) return 1.0f;  // quant.cpp:58
    const double div = bits == 4 ? 7.5 : 127.5;
    return __double2float_ru(__ddiv_rn(static_cast<double>(absmax), div));
}

// quantize_one (quant.cpp:24-29) without f64 arithmetic per element.  The
// reference computes round_half_away(RN64(v / S)).  For f32 v and S the exact
// quotient is either exactly a half-integer or at least ~2^-33 (relative) away
// from one, so RN64 neither creates nor crosses a tie and the reference equals
// round_half_away(exact v/S).  We compute that exactly in f32:
//   k = floor(RN32(|v| / S))        -- correct or one too high only when the
//                                      exact quotient is just below an integer,
//                                      where rounding returns k anyway;
//   n = k + (|v| - (k + 0.5) * S >= 0)  evaluated with one FMA (exact sign).
// Verified bit-exact against the reference by tests/test_gpu_quant.py on
// tie-rich inputs (every element on or one ulp beside a tie).
__device__ __forceinline__ int quantize_one(float v, float s, int bits) {
    const float a = fabsf(v);
    const float q = __fdiv_rn(a, s);
    float k = floorf(q);
    const float r = __fmaf_rn(-(k + 0.5f), s, a);
    if (r >= 0.0f) k += 1.0f;
    const int hi = qmax_of(bits), lo = qmin_of(bits);
    int n = static_cast<int>(fminf(k, 256.0f));
    int c = v < 0.0f ? -n : n;
    return c < lo ? lo : (c > hi ? hi : c);
}

// ---- layouts -----------------------------------------------------------------------------
struct Layout {
    int kind;  // RTNQ_ROW_MAJOR / RTNQ_KERNEL_INTERLEAVED / RTNQ_NATIVE_SM100
    int tr, tc;
};

__host__ __device__ __forceinline__ int64_t native_kblock(int bits) { return bits == 4 ? 64 : 32; }

// Native layout.  Rows form 16-row strips (one mma.m16n8k16 A
// tile); 16 strips form a 256-row row-block.  Columns form k-blocks of 64 (4-bit)
// or 32 (8-bit) codes = 16 bytes per lane.  Byte order:
//   [row-block][k-block][strip in block][lane 0..31][16 bytes]
// so every row-block's codes are one contiguous run along K (a GEMM CTA streams
// contiguous memory) and one (row-block, k-block) is a contiguous 8 KiB tile.
// The last row-block may hold fewer than 16 strips.  Inside a lane's 16 bytes each
// k16 step is one word of the A fragment (a0..a7), in the order the register
// dequantizer consumes it.
constexpr int kNativeBlockStrips = 16;

__host__ __device__ __forceinline__ int64_t native_chunk(int64_t ns, int64_t kblk, int64_t strip,
                                                         int64_t b) {
    const int64_t rb = strip / kNativeBlockStrips, sl = strip % kNativeBlockStrips;
    const int64_t in_rb = ns - rb * kNativeBlockStrips < kNativeBlockStrips
                              ? ns - rb * kNativeBlockStrips : kNativeBlockStrips;
    return rb * kNativeBlockStrips * kblk + b * in_rb + sl;  // index of the 512-byte chunk
}

__host__ __device__ __forceinline__ int64_t native_slot(int bits, int64_t rows, int64_t cols,
                                                        int64_t r, int64_t c) {
    const int64_t ns = (rows + 15) / 16, kb = native_kblock(bits);
    const int64_t kblk = (cols + kb - 1) / kb;
    const int64_t s = r >> 4, rr = r & 15, b = c / kb, cc = c % kb;
    const int64_t j = cc >> 4, kk = cc & 15;
    const int64_t gid = rr & 7, hi_row = rr >> 3, tig = (kk & 7) >> 1, hi_k = kk >> 3,
                  lo = kk & 1;
    const int64_t lane = 4 * gid + tig;
    const int64_t e = 4 * hi_k + 2 * hi_row + lo;
    const int64_t base = native_chunk(ns, kblk, s, b) * 32 + lane;
    if (bits == 4) return base * 32 + j * 8 + (e & 1) * 4 + (e >> 1);
    return base * 16 + j * 8 + (e >> 2) * 4 + (e & 1) * 2 + ((e >> 1) & 1);
}

// Inverse of native_slot: slot -> (r, c); returns false for padding slots.
__host__ __device__ __forceinline__ bool native_coords(int bits, int64_t rows, int64_t cols,
                                                       int64_t slot, int64_t* r, int64_t* c) {
    const int64_t ns = (rows + 15) / 16, kb = native_kblock(bits);
    const int64_t kblk = (cols + kb - 1) / kb;
    int64_t e, j, rest;
    if (bits == 4) {
        const int64_t nib = slot & 7;
        j = (slot >> 3) & 3;
        rest = slot >> 5;
        e = 2 * (nib & 3) + (nib >> 2);
    } else {
        const int64_t byte = slot & 7;
        j = (slot >> 3) & 1;
        rest = slot >> 4;
        const int64_t b2 = byte & 3;
        e = (byte >> 2) * 4 + (b2 & 1) * 2 + (b2 >> 1);
    }
    const int64_t lane = rest & 31;
    const int64_t chunk = rest >> 5;
    const int64_t per_rb = int64_t(kNativeBlockStrips) * kblk;
    const int64_t rb = chunk / per_rb, off = chunk % per_rb;
    const int64_t in_rb = ns - rb * kNativeBlockStrips < kNativeBlockStrips
                              ? ns - rb * kNativeBlockStrips : kNativeBlockStrips;
    const int64_t b = off / in_rb, s = rb * kNativeBlockStrips + off % in_rb;
    const int64_t gid = lane >> 2, tig = lane & 3;
    const int64_t hi_k = e >> 2, hi_row = (e >> 1) & 1, lo = e & 1;
    *r = 16 * s + gid + 8 * hi_row;
    *c = b * kb + j * 16 + 2 * tig + 8 * hi_k + lo;
    return *r < rows && *c < cols;
}

__host__ __device__ __forceinline__ int64_t layout_slot(const Layout& L, int bits, int64_t rows,
                                                        int64_t cols, int64_t r, int64_t c) {
    if (L.kind == RTNQ_ROW_MAJOR) return r * cols + c;
    if (L.kind == RTNQ_NATIVE_SM100) return native_slot(bits, rows, cols, r, c);
    const int64_t tpr = (cols + L.tc - 1) / L.tc;  // packing.cpp:62-65
    const int64_t tile = (r / L.tr) * tpr + c / L.tc;
    return tile * L.tr * L.tc + (c % L.tc) * L.tr + r % L.tr;
}

__host__ __device__ __forceinline__ bool layout_coords(const Layout& L, int bits, int64_t rows,
                                                       int64_t cols, int64_t slot, int64_t* r,
                                                       int64_t* c) {
    if (L.kind == RTNQ_ROW_MAJOR) {
        *r = slot / cols;
        *c = slot % cols;
        return *r < rows;
    }
    if (L.kind == RTNQ_NATIVE_SM100) return native_coords(bits, rows, cols, slot, r, c);
    const int64_t tt = int64_t(L.tr) * L.tc, tpr = (cols + L.tc - 1) / L.tc;
    const int64_t tile = slot / tt, within = slot % tt;
    *r = (tile / tpr) * L.tr + within % L.tr;
    *c = (tile % tpr) * L.tc + within / L.tr;
    return *r < rows && *c < cols;
}

__host__ __device__ __forceinline__ int64_t layout_slots_of(const Layout& L, int bits,
                                                            int64_t rows, int64_t cols) {
    if (L.kind == RTNQ_ROW_MAJOR) return rows * cols;
    if (L.kind == RTNQ_NATIVE_SM100) {
        const int64_t kb = native_kblock(bits);
        return ((rows + 15) / 16 * 16) * ((cols + kb - 1) / kb * kb);
    }
    return ((rows + L.tr - 1) / L.tr * L.tr) * ((cols + L.tc - 1) / L.tc * L.tc);
}

// Signed code at a storage slot (offset-binary, packing.cpp:19-30).
__device__ __forceinline__ int code_at_slot(const uint8_t* data, int bits, int64_t slot) {
    if (bits == 8) return int(data[slot]) - 128;
    const uint8_t b = data[slot >> 1];
    return int((slot & 1) ? (b >> 4) : (b & 0x0F)) - 8;
}

// Native scale order [row-block][group][strip in block][gid][half], f16, with
// row = 16*strip + 8*half + gid: a row-block's scales are one contiguous run
// along K, like its codes.  Padded rows hold 0.
__host__ __device__ __forceinline__ int64_t native_scale_index(int64_t rows, int64_t gpr,
                                                               int64_t r, int64_t group) {
    const int64_t ns = (rows + 15) / 16;
    return (native_chunk(ns, gpr, r >> 4, group) * 8 + (r & 7)) * 2 + ((r >> 3) & 1);
}

__device__ __forceinline__ float load_scale(const void* scales, int dtype, int order,
                                            int64_t rows, int64_t gpr, int64_t r,
                                            int64_t group) {
    const int64_t i = order == RTNQ_SCALES_NATIVE ? native_scale_index(rows, gpr, r, group)
                                                  : r * gpr + group;
    return load_elem(scales, dtype, i);
}

}  // namespace rtnq_b200
