/*
 * rtnq_oracle.c -- CPU restatement of the reference rtnq hot path (C99).
 *
 * TEST INFRASTRUCTURE ONLY (see rtnq_oracle.h).  Compiled by oracle/Makefile
 * with -O2 -ffp-contract=off so every float operation is a separately rounded
 * IEEE op, which is what the reference's default x86-64 build does (no FMA
 * contraction without -march=native; RTNQ_NATIVE is OFF by default,
 * proj/CMakeLists.txt:12-19).
 *
 * Every function cites the reference file:line it restates.  The reference is
 * single-process CPU C++20; its thread partitioning never changes results
 * (proj/core/include/rtnq/threading.hpp:14-18), so this port is sequential.
 */
#include "rtnq_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- f16 (proj/core/src/f16.cpp) ------------------------------------------------ */

static uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* Round-to-nearest-even narrowing; f16.cpp:8-41. */
uint16_t ro_f32_to_f16(float value) {
    uint32_t x = f2u(value);
    uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
    uint32_t mag = x & 0x7FFFFFFFu;
    if (mag >= 0x7F800000u) /* inf or nan; nan stays quiet (f16.cpp:14-17) */
        return (uint16_t)(sign | 0x7C00u | (mag > 0x7F800000u ? 0x0200u : 0u));
    if (mag >= 0x47800000u) return (uint16_t)(sign | 0x7C00u); /* >= 2^16 -> inf (:18-19) */
    if (mag < 0x38800000u) {                                 /* below 2^-14 (:21-33) */
        if (mag < 0x33000000u) return sign;                  /* < 2^-25 -> +-0 */
        int sh = 126 - (int)(mag >> 23);                     /* 14..24 */
        uint32_t m = (mag & 0x7FFFFFu) | 0x800000u;
        uint32_t q = m >> sh, r = m & ((1u << sh) - 1u), h = 1u << (sh - 1);
        if (r > h || (r == h && (q & 1u))) q++;
        return (uint16_t)(sign | q);
    }
    /* normal: rebias, RNE on 13 dropped bits; carry may reach inf (:35-40) */
    uint32_t q = (((mag >> 23) - 112u) << 10) | ((mag >> 13) & 0x3FFu);
    uint32_t r = mag & 0x1FFFu;
    if (r > 0x1000u || (r == 0x1000u && (q & 1u))) q++;
    return (uint16_t)(sign | q);
}

/* Exact widening; f16.cpp:43-63. */
float ro_f16_to_f32(uint16_t h) {
    uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    uint32_t e = (h >> 10) & 0x1Fu, m = h & 0x3FFu;
    if (e == 0x1Fu) return u2f(sign | 0x7F800000u | (m << 13));
    if (e == 0) {
        if (m == 0) return u2f(sign);
        /* subnormal: value = m * 2^-24, exact in f32 */
        float v = (float)m * 0x1p-24f;
        return sign ? -v : v;
    }
    return u2f(sign | ((e + 112u) << 23) | (m << 13));
}

/* ---- scalar grid (proj/core/include/rtnq/types.hpp:12-21) ------------------------ */

float ro_scale_divisor(int bits) { return (float)(1 << (bits - 1)) - 0.5f; }
int ro_qmin(int bits) { return -(1 << (bits - 1)); }
int ro_qmax(int bits) { return (1 << (bits - 1)) - 1; }

/* GroupSpec::groups_per_row, types.hpp:30-38. */
int64_t ro_groups_per_row(int64_t g, int ragged, int64_t cols) {
    if (g <= 0 || (g & (g - 1)) != 0) return -RO_INVALID;
    if (cols % g != 0 && !ragged) return -RO_SHAPE;
    return (cols + g - 1) / g;
}

/* compute_scale, proj/core/src/quant.cpp:49-68: f32 absmax, f64 quotient
 * rounded *up* to f32; 1.0 for an all-zero group; non-finite -> invalid. */
int ro_compute_scale(const float* v, int64_t n, int bits, float* out) {
    if (n <= 0) return RO_INVALID;
    float amax = 0.0f;
    for (int64_t i = 0; i < n; ++i) {
        float a = fabsf(v[i]);
        if (!(a <= FLT_MAX)) return RO_INVALID;
        if (a > amax) amax = a;
    }
    if (amax == 0.0f) { *out = 1.0f; return RO_OK; }
    double q = (double)amax / (double)ro_scale_divisor(bits);
    float s = (float)q;
    if ((double)s < q) s = nextafterf(s, INFINITY);
    *out = s;
    return RO_OK;
}

/* quantize_one, quant.cpp:24-29: round half away from zero of the f64
 * quotient, clamp to [qmin, qmax]. */
int8_t ro_quantize_one(float v, float scale, int bits) {
    double q = round((double)v / (double)scale);
    double lo = ro_qmin(bits), hi = ro_qmax(bits);
    if (q < lo) q = lo;
    if (q > hi) q = hi;
    return (int8_t)q;
}

/* quantize_tensor, quant.cpp:100-141 (logical codes before pack()). */
int ro_quantize_tensor(const float* w, int64_t rows, int64_t cols, int bits, int64_t g,
                       int ragged, int8_t* codes, float* scales) {
    int64_t gpr = ro_groups_per_row(g, ragged, cols);
    if (gpr < 0) return (int)-gpr;
    for (int64_t r = 0; r < rows; ++r) {
        const float* row = w + r * cols;
        for (int64_t j = 0; j < gpr; ++j) {
            int64_t c0 = j * g, len = (g < cols - c0) ? g : cols - c0;
            float s;
            int st = ro_compute_scale(row + c0, len, bits, &s);
            if (st != RO_OK) return st;
            scales[r * gpr + j] = s;
            for (int64_t i = 0; i < len; ++i)
                codes[r * cols + c0 + i] = ro_quantize_one(row[c0 + i], s, bits);
        }
    }
    return RO_OK;
}

/* ---- packing (proj/core/src/packing.cpp) ---------------------------------------- */

int64_t ro_packed_size(int64_t len, int bits) { return (len * bits + 7) / 8; }

/* pack, packing.cpp:6-32: offset-binary, 4-bit low nibble = even index. */
int ro_pack(const int8_t* codes, int64_t n, int bits, uint8_t* out) {
    for (int64_t i = 0; i < n; ++i)
        if (codes[i] < ro_qmin(bits) || codes[i] > ro_qmax(bits)) return RO_INVALID;
    memset(out, 0, (size_t)ro_packed_size(n, bits));
    if (bits == 8) {
        for (int64_t i = 0; i < n; ++i) out[i] = (uint8_t)(codes[i] + 128);
        return RO_OK;
    }
    for (int64_t i = 0; i < n; ++i) {
        uint8_t u = (uint8_t)(codes[i] + 8);
        out[i >> 1] |= (uint8_t)((i & 1) ? (u << 4) : u);
    }
    return RO_OK;
}

/* unpack, packing.cpp:34-55 (length validation is the caller's job here). */
void ro_unpack(const uint8_t* bytes, int64_t n, int bits, int8_t* out) {
    for (int64_t i = 0; i < n; ++i) {
        if (bits == 8) {
            out[i] = (int8_t)((int)bytes[i] - 128);
        } else {
            uint8_t b = bytes[i >> 1];
            out[i] = (int8_t)((int)((i & 1) ? (b >> 4) : (b & 0x0F)) - 8);
        }
    }
}

/* Native layout (this repository's GEMM operand order): the
 * tcgen05 A-operand order.  Rows form 128-row row-blocks (the last may be
 * shorter); columns form k-blocks of 64 codes (zero-padded).  Each row owns
 * 16-byte chunks (2 per k-block for 4-bit, 4 for 8-bit); within a (row-block,
 * k-block) the chunk c of every row is stored consecutively, chunks in (k-block,
 * c) order, row-blocks one after another -- a row-block is one contiguous run
 * along K.  Inside a chunk each 32-bit word holds one k16 step's codes in the
 * order the dequantizer emits TMEM columns {k, k+1}:
 *   4-bit word: nibble j = code (j < 4 ? 2j : 2(j-4)+1) of its 8-code group;
 *   8-bit word: byte b   = code 2(b&1) + (b>>1)        of its 4-code group. */
static int64_t native_rows_in(int64_t rows, int64_t rb) {
    int64_t left = rows - rb * 128;
    return left < 128 ? left : 128;
}

static int64_t native_chunk(int bits, int64_t rows, int64_t kblk, int64_t r, int64_t kb,
                            int64_t c) {
    int64_t cpr = bits == 4 ? 2 : 4, rb = r / 128;
    return rb * 128 * kblk * cpr + (kb * cpr + c) * native_rows_in(rows, rb) + r % 128;
}

static int64_t native_index(int bits, int64_t rows, int64_t cols, int64_t r, int64_t c) {
    int64_t kblk = (cols + 63) / 64, kb = c / 64, kk = c % 64;
    if (bits == 4) {
        int64_t ch = kk / 32, cc = kk % 32, w = cc / 8, q = cc % 8;
        int64_t j = (q % 2) ? 4 + q / 2 : q / 2;
        return native_chunk(4, rows, kblk, r, kb, ch) * 32 + w * 8 + j;
    }
    int64_t ch = kk / 16, cc = kk % 16, w = cc / 4, q = cc % 4;
    return native_chunk(8, rows, kblk, r, kb, ch) * 16 + w * 4 + 2 * (q % 2) + q / 2;
}

/* layout_index, packing.cpp:57-66 (+ the native kind). */
int64_t ro_layout_index(int kind, int tr, int tc, int bits, int64_t rows, int64_t cols,
                        int64_t r, int64_t c) {
    if (kind == RO_ROW_MAJOR) return r * cols + c;
    if (kind == RO_NATIVE) return native_index(bits, rows, cols, r, c);
    int64_t tpr = (cols + tc - 1) / tc;
    int64_t tile = (r / tr) * tpr + c / tc;
    return tile * tr * tc + (c % tc) * tr + r % tr;
}

/* layout_slots, packing.cpp:68-73 (+ native). */
int64_t ro_layout_slots(int kind, int tr, int tc, int bits, int64_t rows, int64_t cols) {
    (void)bits;
    if (kind == RO_ROW_MAJOR) return rows * cols;
    if (kind == RO_NATIVE) return rows * ((cols + 63) / 64 * 64);
    return ((rows + tr - 1) / tr * tr) * ((cols + tc - 1) / tc * tc);
}

int64_t ro_layout_bytes(int kind, int tr, int tc, int bits, int64_t rows, int64_t cols) {
    return ro_packed_size(ro_layout_slots(kind, tr, tc, bits, rows, cols), bits);
}

/* reshuffle, packing.cpp:75-92: scatter logical codes, zero padding, pack. */
void ro_encode_layout(const int8_t* logical, int64_t rows, int64_t cols, int bits, int kind,
                      int tr, int tc, uint8_t* out) {
    int64_t slots = ro_layout_slots(kind, tr, tc, bits, rows, cols);
    int8_t* placed = (int8_t*)calloc((size_t)(slots > 0 ? slots : 1), 1);
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c)
            placed[ro_layout_index(kind, tr, tc, bits, rows, cols, r, c)] = logical[r * cols + c];
    ro_pack(placed, slots, bits, out);
    free(placed);
}

/* logical_codes / code_at, quant.cpp:33-47,173-180. */
void ro_decode_layout(const uint8_t* data, int64_t rows, int64_t cols, int bits, int kind,
                      int tr, int tc, int8_t* logical) {
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            int64_t idx = ro_layout_index(kind, tr, tc, bits, rows, cols, r, c);
            int8_t v;
            if (bits == 8) {
                v = (int8_t)((int)data[idx] - 128);
            } else {
                uint8_t b = data[idx >> 1];
                v = (int8_t)((int)((idx & 1) ? (b >> 4) : (b & 0x0F)) - 8);
            }
            logical[r * cols + c] = v;
        }
}


/* Native scale order: per 128-row row-block, [group][row] with the block's
 * row count padded to 8; padded rows get 0. */
int64_t ro_native_scale_count(int64_t rows, int64_t gpr) { return gpr * ((rows + 7) / 8 * 8); }

void ro_native_scales(const uint16_t* s16, int64_t rows, int64_t gpr, uint16_t* out) {
    memset(out, 0, (size_t)ro_native_scale_count(rows, gpr) * 2);
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t j = 0; j < gpr; ++j) {
            int64_t rb = r / 128, r8 = (native_rows_in(rows, rb) + 7) / 8 * 8;
            out[rb * 128 * gpr + j * r8 + r % 128] = s16[r * gpr + j];
        }
}

/* dequantize_tensor, quant.cpp:143-171: float(code) * scale (one f32 multiply). */
void ro_dequantize(const int8_t* logical, const float* scales, int64_t rows, int64_t cols,
                   int64_t g, float* out) {
    int64_t gpr = (cols + g - 1) / g;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c)
            out[r * cols + c] = (float)logical[r * cols + c] * scales[r * gpr + c / g];
}

/* ---- GEMMs (proj/core/src/gemm.cpp) --------------------------------------------- */

/* gemm_fused, gemm.cpp:46-92: per output, per group: f32 block subtotal over
 * k ascending, then acc += S * block.  Reads the kernel_interleaved bytes
 * through the constant-stride slot formula (gemm.cpp:64-66). */
void ro_gemm_fused(const float* a, int64_t m, int64_t k, const uint8_t* data, int bits,
                   int tr, int tc, int64_t n, int64_t g, const float* scales, float* out) {
    int64_t gpr = (k + g - 1) / g;
    int64_t tpr = (k + tc - 1) / tc;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            const float* arow = a + i * k;
            int64_t base = (j / tr) * tpr * tr * tc + j % tr;
            float acc = 0.0f;
            for (int64_t q = 0; q < gpr; ++q) {
                int64_t k0 = q * g, k1 = (k0 + g < k) ? k0 + g : k;
                float block = 0.0f;
                for (int64_t kk = k0; kk < k1; ++kk) {
                    int64_t slot = base + kk * tr;
                    int code;
                    if (bits == 4) {
                        uint8_t b = data[slot >> 1];
                        code = (int)((slot & 1) ? (b >> 4) : (b & 0x0F)) - 8;
                    } else {
                        code = (int)data[slot] - 128;
                    }
                    block += arow[kk] * (float)code;
                }
                acc += scales[j * gpr + q] * block;
            }
            out[i * n + j] = acc;
        }
}

/* dense_blocked_gemm, gemm.cpp:23-42. */
static void dense_blocked(const float* a, int64_t m, int64_t k, const float* w, int64_t n,
                          int64_t blk, float* out) {
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            const float* arow = a + i * k;
            const float* wrow = w + j * k;
            float acc = 0.0f;
            for (int64_t k0 = 0; k0 < k; k0 += blk) {
                int64_t k1 = (k0 + blk < k) ? k0 + blk : k;
                float block = 0.0f;
                for (int64_t kk = k0; kk < k1; ++kk) block += arow[kk] * wrow[kk];
                acc += block;
            }
            out[i * n + j] = acc;
        }
}

/* gemm_dequant, gemm.cpp:94-98 = dequantize_tensor + dense_blocked(g). */
void ro_gemm_dequant(const float* a, int64_t m, int64_t k, const int8_t* logical, int64_t n,
                     int64_t g, const float* scales, float* out) {
    float* wf = (float*)malloc((size_t)(n * k > 0 ? n * k : 1) * sizeof(float));
    ro_dequantize(logical, scales, n, k, g, wf);
    dense_blocked(a, m, k, wf, n, g, out);
    free(wf);
}

/* gemm_float, gemm.cpp:111-119. */
void ro_gemm_float(const float* a, int64_t m, int64_t k, const float* w, int64_t n,
                   int64_t block, float* out) {
    dense_blocked(a, m, k, w, n, block, out);
}

/* gemm_oracle, gemm.cpp:121-149: exact products in f64, k-ascending f64 sum,
 * one final rounding to f32. */
void ro_gemm_oracle_f64(const float* a, int64_t m, int64_t k, const int8_t* logical, int64_t n,
                        int64_t g, const float* scales, double* out) {
    int64_t gpr = (k + g - 1) / g;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int64_t kk = 0; kk < k; ++kk) {
                double wv = (double)logical[j * k + kk] * (double)scales[j * gpr + kk / g];
                acc += (double)a[i * k + kk] * wv;
            }
            out[i * n + j] = acc;
        }
}

void ro_gemm_oracle(const float* a, int64_t m, int64_t k, const int8_t* logical, int64_t n,
                    int64_t g, const float* scales, float* out) {
    int64_t gpr = (k + g - 1) / g;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int64_t kk = 0; kk < k; ++kk) {
                double wv = (double)logical[j * k + kk] * (double)scales[j * gpr + kk / g];
                acc += (double)a[i * k + kk] * wv;
            }
            out[i * n + j] = (float)acc;
        }
}

/* ---- PRNG (proj/core/include/rtnq/rng.hpp:24-66) -------------------------------- */

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void ro_xoshiro_fill_unit(uint64_t seed, uint64_t stream, float* out, int64_t n, float mult) {
    uint64_t sm = seed ^ (stream * 0x9E3779B97F4A7C15ull), s[4];
    for (int i = 0; i < 4; ++i) { /* splitmix64, rng.hpp:24-35 */
        uint64_t z = (sm += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        s[i] = z ^ (z >> 31);
    }
    for (int64_t i = 0; i < n; ++i) { /* xoshiro256**, rng.hpp:44-55 */
        uint64_t res = rotl64(s[1] * 5, 7) * 9, t = s[1] << 17;
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t;
        s[3] = rotl64(s[3], 45);
        float u = (float)(uint32_t)(res >> 40) * (1.0f / 8388608.0f) - 1.0f; /* rng.hpp:57-61 */
        out[i] = mult * u; /* toy.cpp:161-164 multiplies amp * next_unit() */
    }
}
