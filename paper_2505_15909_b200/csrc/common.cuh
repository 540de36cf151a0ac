// common.cuh -- shared device helpers: element types, the reference's scalar
// quantization rules, and the three code layouts.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/rtnq_capi.h"

namespace rtnq_b200 {

// Bit of the current CUDA device in a per-process "done on this device" mask (kernel attributes
// and launch caches are per device; a process may drive several GPUs).
inline unsigned long long current_device_bit() {
    int dev = 0;
    cudaGetDevice(&dev);
    return 1ull << (dev & 63);
}
inline int current_device_index() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev & 63;
}

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
// Verified bit-exact against the reference by tests/test_gpu_full_shapes.py
// (test_quantize_f32_ties_bit_exact: f32 weights on or one ulp beside a tie).
__device__ __forceinline__ int quantize_one(float v, float s, int bits) {
    float a = fabsf(v);
    if (s < 5.421010862427522e-20f) {  // S < 2^-64: scale both by 2^64 (exact) so the tie
        a *= 18446744073709551616.0f;  // test below never underflows into -0
        s *= 18446744073709551616.0f;
    }
    const float q = __fdiv_rn(a, s);
    float k = floorf(q);
    const float r = __fmaf_rn(-(k + 0.5f), s, a);
    if (r >= 0.0f) k += 1.0f;
    const int hi = qmax_of(bits), lo = qmin_of(bits);
    int n = static_cast<int>(fminf(k, 256.0f));
    int c = v < 0.0f ? -n : n;
    return c < lo ? lo : (c > hi ? hi : c);
}

// quantize_one without a division (the load-path kernels, quant_native.cu).  inv is any
// approximation of 1/S good to ~2^-20 (MUFU.RCP): n0 = rint(|v| * inv) is then the reference's
// code magnitude n = round_half_away(|v| / S) or one off, and only next to a half-integer.  Two
// FMAs with exact signs fix it: |v| - (n0 - 0.5) S < 0  ->  n0 - 1,  |v| - (n0 + 0.5) S >= 0  ->
// n0 + 1 (ties go away from zero, quant.cpp:24-29).  |v| / S <= 7.5 (4-bit) or 127.5 (8-bit)
// by construction of S, so only the positive side needs the qmax clamp.
// Checked bit-exact on tie-rich f32 inputs (tests/test_gpu_full_shapes.py).
// Callers pass S >= 2^-64 (else v and S pre-scaled by 2^64, exact: quant_scale_prep), so the
// remainders of the tie test are far above the subnormal range and never round to -0.
template <int BITS>
__device__ __forceinline__ int quantize_fast(float v, float s, float inv) {
    const float a = fabsf(v);
    const float b = __fmaf_rn(a, inv, 12582912.0f);  // 1.5 * 2^23 + rint(a * inv)
    const float n0 = __fsub_rn(b, 12582912.0f);
    int n = __float_as_int(b) - 0x4B400000;
    n -= __fmaf_rn(-__fsub_rn(n0, 0.5f), s, a) < 0.0f;
    n += __fmaf_rn(-__fadd_rn(n0, 0.5f), s, a) >= 0.0f;
    return v < 0.0f ? -n : min(n, (1 << (BITS - 1)) - 1);
}

struct QuantScale {
    float s;    // the scale the tie test uses (S, or S * 2^64 for S < 2^-64)
    float inv;  // ~1 / s
    float pre;  // 1, or 2^64: multiply v by it
};
__device__ __forceinline__ QuantScale quant_scale_prep(float S) {
    const bool tiny = S < 5.421010862427522e-20f;
    const float s = tiny ? S * 18446744073709551616.0f : S;
    return {s, __frcp_rn(s), tiny ? 18446744073709551616.0f : 1.0f};
}

// ---- layouts -----------------------------------------------------------------------------
struct Layout {
    int kind;  // RTNQ_ROW_MAJOR / RTNQ_KERNEL_INTERLEAVED / RTNQ_NATIVE_SM100
    int tr, tc;
};

// Native layout: the tcgen05 A-operand order.  Rows form
// 128-row row-blocks (one M=128 UMMA tile; the last block may be shorter);
// columns form k-blocks of 64 codes (zero-padded).  Each (row-block, k-block)
// tile stores, for each 16-byte chunk c of a row (2 chunks per row for 4-bit,
// 4 for 8-bit), the chunks of all rows of the block consecutively:
//   byte = ((rb_base + (kb * CPR + c) * rows(rb) + row) * 16 + byte_in_chunk
// so a row-block is one contiguous run along K (a GEMM CTA streams contiguous
// memory), and a warp reading chunk c of 32 consecutive rows issues one
// conflict-free 512-byte LDS.128.  Inside a chunk, every 32-bit word holds 8
// (4-bit) or 4 (8-bit) codes of one k16 step in the order the register
// dequantizer emits TMEM columns {k, k+1}:
//   4-bit word: nibble j = code (j < 4 ? 2j : 2(j-4)+1) of its 8-code group
//   8-bit word: byte b   = code 2(b&1) + (b>>1)        of its 4-code group
constexpr int kNativeRows = 128;  // rows per row-block (UMMA M)
constexpr int kNativeKB = 64;     // codes per k-block

__host__ __device__ __forceinline__ int64_t native_kblock(int bits) {
    (void)bits;
    return kNativeKB;
}
__host__ __device__ __forceinline__ int native_cpr(int bits) { return bits == 4 ? 2 : 4; }

__host__ __device__ __forceinline__ int64_t native_rows_in(int64_t rows, int64_t rb) {
    const int64_t left = rows - rb * kNativeRows;
    return left < kNativeRows ? left : kNativeRows;
}

// 16-byte chunk index of (row r, k-block kb, chunk c).
__host__ __device__ __forceinline__ int64_t native_chunk(int bits, int64_t rows, int64_t kblk,
                                                         int64_t r, int64_t kb, int64_t c) {
    const int64_t rb = r / kNativeRows, cpr = native_cpr(bits);
    return rb * kNativeRows * kblk * cpr + (kb * cpr + c) * native_rows_in(rows, rb) +
           r % kNativeRows;
}

__host__ __device__ __forceinline__ int64_t native_slot(int bits, int64_t rows, int64_t cols,
                                                        int64_t r, int64_t c) {
    const int64_t kblk = (cols + kNativeKB - 1) / kNativeKB;
    const int64_t kb = c / kNativeKB, kk = c % kNativeKB;
    if (bits == 4) {
        const int64_t ch = kk >> 5, cc = kk & 31;  // chunk, code within chunk
        const int64_t w = cc >> 3, q = cc & 7;     // word, code within the word's group
        const int64_t j = (q & 1) ? 4 + (q >> 1) : (q >> 1);
        return native_chunk(4, rows, kblk, r, kb, ch) * 32 + w * 8 + j;
    }
    const int64_t ch = kk >> 4, cc = kk & 15;
    const int64_t w = cc >> 2, q = cc & 3;
    return native_chunk(8, rows, kblk, r, kb, ch) * 16 + w * 4 + 2 * (q & 1) + (q >> 1);
}

// Inverse of native_slot: slot -> (r, c); returns false for padding slots.
__host__ __device__ __forceinline__ bool native_coords(int bits, int64_t rows, int64_t cols,
                                                       int64_t slot, int64_t* r, int64_t* c) {
    const int64_t kblk = (cols + kNativeKB - 1) / kNativeKB, cpr = native_cpr(bits);
    int64_t chunk, cc;
    if (bits == 4) {
        chunk = slot >> 5;
        const int64_t within = slot & 31, w = within >> 3, j = within & 7;
        cc = w * 8 + (j < 4 ? 2 * j : 2 * (j - 4) + 1);
    } else {
        chunk = slot >> 4;
        const int64_t within = slot & 15, w = within >> 2, b = within & 3;
        cc = w * 4 + 2 * (b & 1) + (b >> 1);
    }
    const int64_t per_rb = int64_t(kNativeRows) * kblk * cpr;
    const int64_t rb = chunk / per_rb, off = chunk % per_rb;
    const int64_t rin = native_rows_in(rows, rb);
    if (rin <= 0) return false;
    const int64_t kbc = off / rin, row = off % rin;
    const int64_t kb = kbc / cpr, ch = kbc % cpr;
    *r = rb * kNativeRows + row;
    *c = kb * kNativeKB + ch * (bits == 4 ? 32 : 16) + cc;
    return *r < rows && *c < cols;
}

// Native int8-MMA layout (RTNQ_NATIVE_I8): 128-row x 128-code tiles, row-blocks
// outer and k-tiles inner (a row-block is one contiguous run along K), each tile stored
// exactly as a 128-byte-swizzled UMMA K-major operand: code (r, k) of a tile sits at
// r * 128 + ((k / 16) ^ (r % 8)) * 16 + k % 16.  Codes are two's-complement bytes (code_at_slot);
// padding (rows to 128, K to 128) is code 0.
constexpr int kI8Tile = 128;
__host__ __device__ __forceinline__ int64_t i8_slot(int64_t cols, int64_t r, int64_t c) {
    const int64_t kt = (cols + kI8Tile - 1) / kI8Tile;
    const int64_t tile = (r / kI8Tile) * kt + c / kI8Tile;
    const int64_t rr = r % kI8Tile, kk = c % kI8Tile;
    return tile * (kI8Tile * kI8Tile) + rr * kI8Tile + ((((kk >> 4) ^ (rr & 7)) << 4) | (kk & 15));
}
__host__ __device__ __forceinline__ bool i8_coords(int64_t rows, int64_t cols, int64_t slot,
                                                   int64_t* r, int64_t* c) {
    const int64_t kt = (cols + kI8Tile - 1) / kI8Tile;
    const int64_t tile = slot / (kI8Tile * kI8Tile), within = slot % (kI8Tile * kI8Tile);
    const int64_t rr = within / kI8Tile, pos = within % kI8Tile;
    const int64_t kk = ((((pos >> 4) ^ (rr & 7))) << 4) | (pos & 15);
    *r = (tile / kt) * kI8Tile + rr;
    *c = (tile % kt) * kI8Tile + kk;
    return *r < rows && *c < cols;
}

// Native W4 int8-MMA layout (RTNQ_NATIVE_I4): one 8 KiB tile per 128 rows x one
// 128-code group, row-blocks outer and groups inner.  Row r of a tile is 64 bytes; byte p
// holds code (r, p) in its high nibble and code (r, 64 + p) in its low nibble, as 4-bit two's
// complement, so (byte & 0xF0) and (byte << 4 & 0xF0) are the s8 values 16 * code.  The four
// 16-byte chunks of a row are XOR-swizzled by (r / 2) % 4 (conflict-free 16-byte reads of 8
// consecutive rows).  Padding is code 0.
constexpr int kI4Tile = 128;
__host__ __device__ __forceinline__ int64_t i4_slot(int64_t cols, int64_t r, int64_t c) {
    const int64_t kt = (cols + kI4Tile - 1) / kI4Tile;
    const int64_t tile = (r / kI4Tile) * kt + c / kI4Tile;
    const int64_t rr = r % kI4Tile, kk = c % kI4Tile, pos = kk & 63;
    const int64_t byte = tile * (kI4Tile * 64) + rr * 64 + ((((pos >> 4) ^ ((rr >> 1) & 3))) << 4) + (pos & 15);
    return 2 * byte + (kk < 64 ? 1 : 0);  // odd slot = high nibble
}
__host__ __device__ __forceinline__ bool i4_coords(int64_t rows, int64_t cols, int64_t slot,
                                                   int64_t* r, int64_t* c) {
    const int64_t kt = (cols + kI4Tile - 1) / kI4Tile;
    const int64_t byte = slot >> 1, tile = byte / (kI4Tile * 64), within = byte % (kI4Tile * 64);
    const int64_t rr = within / 64, off = within % 64;
    const int64_t pos = ((((off >> 4) ^ ((rr >> 1) & 3))) << 4) | (off & 15);
    *r = (tile / kt) * kI4Tile + rr;
    *c = (tile % kt) * kI4Tile + ((slot & 1) ? pos : 64 + pos);
    return *r < rows && *c < cols;
}

__host__ __device__ __forceinline__ int64_t layout_slot(const Layout& L, int bits, int64_t rows,
                                                        int64_t cols, int64_t r, int64_t c) {
    if (L.kind == RTNQ_ROW_MAJOR) return r * cols + c;
    if (L.kind == RTNQ_NATIVE_I8) return i8_slot(cols, r, c);
    if (L.kind == RTNQ_NATIVE_I4) return i4_slot(cols, r, c);
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
    if (L.kind == RTNQ_NATIVE_I8) return i8_coords(rows, cols, slot, r, c);
    if (L.kind == RTNQ_NATIVE_I4) return i4_coords(rows, cols, slot, r, c);
    const int64_t tt = int64_t(L.tr) * L.tc, tpr = (cols + L.tc - 1) / L.tc;
    const int64_t tile = slot / tt, within = slot % tt;
    *r = (tile / tpr) * L.tr + within % L.tr;
    *c = (tile % tpr) * L.tc + within / L.tr;
    return *r < rows && *c < cols;
}

__host__ __device__ __forceinline__ int64_t layout_slots_of(const Layout& L, int bits,
                                                            int64_t rows, int64_t cols) {
    if (L.kind == RTNQ_ROW_MAJOR) return rows * cols;
    if (L.kind == RTNQ_NATIVE_SM100)
        return rows * ((cols + kNativeKB - 1) / kNativeKB * kNativeKB);
    if (L.kind == RTNQ_NATIVE_I8 || L.kind == RTNQ_NATIVE_I4)
        return (rows + kI8Tile - 1) / kI8Tile * kI8Tile * ((cols + kI8Tile - 1) / kI8Tile * kI8Tile);
    return ((rows + L.tr - 1) / L.tr * L.tr) * ((cols + L.tc - 1) / L.tc * L.tc);
}

// Signed code at a storage slot (offset-binary, packing.cpp:19-30).  RTNQ_NATIVE_I8 stores the
// 8-bit code as a two's-complement byte instead (the s8 operand of the int8 MMA, no offset).
__device__ __forceinline__ int code_at_slot(const uint8_t* data, int bits, int64_t slot,
                                            int kind = RTNQ_ROW_MAJOR) {
    if (bits == 8) return kind == RTNQ_NATIVE_I8 ? int(int8_t(data[slot])) : int(data[slot]) - 128;
    const uint8_t b = data[slot >> 1];
    const int v = (slot & 1) ? (b >> 4) : (b & 0x0F);
    return kind == RTNQ_NATIVE_I4 ? ((v ^ 8) - 8) : v - 8;  // two's complement / offset-binary
}
__device__ __forceinline__ uint32_t code_nib4(int code, int kind) {
    return kind == RTNQ_NATIVE_I4 ? uint32_t(code) & 0xFu : uint32_t(code + 8);
}
__device__ __forceinline__ uint8_t code_byte8(int code, int kind) {
    return kind == RTNQ_NATIVE_I8 ? uint8_t(int8_t(code)) : uint8_t(code + 128);
}

// Native scale order: per 128-row row-block, [group][row] with the row count
// padded to 8 (so a block's scales for consecutive groups are one contiguous,
// 16-byte-aligned run); padded rows hold 0.
__host__ __device__ __forceinline__ int64_t native_scale_rows8(int64_t rows, int64_t rb) {
    return (native_rows_in(rows, rb) + 7) / 8 * 8;
}
__host__ __device__ __forceinline__ int64_t native_scale_index(int64_t rows, int64_t gpr,
                                                               int64_t r, int64_t group) {
    const int64_t rb = r / kNativeRows;
    return rb * kNativeRows * gpr + group * native_scale_rows8(rows, rb) + r % kNativeRows;
}

__device__ __forceinline__ float load_scale(const void* scales, int dtype, int order,
                                            int64_t rows, int64_t gpr, int64_t r,
                                            int64_t group) {
    const int64_t i = order == RTNQ_SCALES_NATIVE ? native_scale_index(rows, gpr, r, group)
                                                  : r * gpr + group;
    return load_elem(scales, dtype, i);
}

}  // namespace rtnq_b200
