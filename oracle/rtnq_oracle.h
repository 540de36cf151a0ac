/*
 * rtnq_oracle.h -- CPU restatement of the reference rtnq hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2505_15909_b200/,
 * include/) may link, load or call this code.  It is the checker used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks every function here
 * against (a) the reference's own known-answer tests (proj/tests/test_*.cpp)
 * and (b) golden vectors produced by the reference library itself, compiled
 * from /root/reference by oracle/Makefile into oracle/_ref/ and dumped by
 * tests/golden/make_golden.py.
 *
 * All citations are relative to /root/reference/.
 */
#ifndef RTNQ_ORACLE_H
#define RTNQ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Layout kinds (proj/core/include/rtnq/types.hpp:69-83 for 0 and 1; 2 is the
 * B200 GEMM-native layout defined by this repository). */
enum { RO_ROW_MAJOR = 0, RO_KERNEL = 1, RO_NATIVE = 2 };

enum { RO_OK = 0, RO_INVALID = 1, RO_SHAPE = 2, RO_CORRUPT = 3 };

uint16_t ro_f32_to_f16(float value);
float ro_f16_to_f32(uint16_t bits);

float ro_scale_divisor(int bits);
int ro_qmin(int bits);
int ro_qmax(int bits);

/* Returns RO_OK and *out, or RO_INVALID for an empty group / non-finite value. */
int ro_compute_scale(const float* v, int64_t n, int bits, float* out);
int8_t ro_quantize_one(float v, float scale, int bits);

/* groups_per_row with the reference's validation; <0 on error (-RO_INVALID, -RO_SHAPE). */
int64_t ro_groups_per_row(int64_t g, int ragged, int64_t cols);

/* Logical int8 codes (rows*cols, row-major) and f32 scales (rows*gpr). */
int ro_quantize_tensor(const float* w, int64_t rows, int64_t cols, int bits, int64_t g,
                       int ragged, int8_t* codes, float* scales);

int64_t ro_packed_size(int64_t len, int bits);
int ro_pack(const int8_t* codes, int64_t n, int bits, uint8_t* out);
void ro_unpack(const uint8_t* bytes, int64_t n, int bits, int8_t* out);

/* Storage slot of logical (r, c).  tr/tc only matter for RO_KERNEL; bits only
 * for RO_NATIVE (its k-block is 64 codes for 4-bit, 32 for 8-bit). */
int64_t ro_layout_index(int kind, int tr, int tc, int bits, int64_t rows, int64_t cols,
                        int64_t r, int64_t c);
int64_t ro_layout_slots(int kind, int tr, int tc, int bits, int64_t rows, int64_t cols);

/* Packed bytes of a rows x cols code matrix in `kind` (padding slots hold 0). */
int64_t ro_layout_bytes(int kind, int tr, int tc, int bits, int64_t rows, int64_t cols);
void ro_encode_layout(const int8_t* logical, int64_t rows, int64_t cols, int bits, int kind,
                      int tr, int tc, uint8_t* out);
void ro_decode_layout(const uint8_t* data, int64_t rows, int64_t cols, int bits, int kind,
                      int tr, int tc, int8_t* logical);

/* Native-order f16 scales: [group][strip16][gid 0..7][half 0..1]. */
int64_t ro_native_scale_count(int64_t rows, int64_t gpr);
void ro_native_scales(const uint16_t* scales_f16, int64_t rows, int64_t gpr, uint16_t* out);

/* codes * scale, f32, row-major rows x cols. */
void ro_dequantize(const int8_t* logical, const float* scales, int64_t rows, int64_t cols,
                   int64_t g, float* out);

/* The reference GEMMs.  a: m x k f32 row-major; out: m x n f32 row-major. */
void ro_gemm_fused(const float* a, int64_t m, int64_t k, const uint8_t* data, int bits,
                   int tr, int tc, int64_t n, int64_t g, const float* scales, float* out);
void ro_gemm_dequant(const float* a, int64_t m, int64_t k, const int8_t* logical, int64_t n,
                     int64_t g, const float* scales, float* out);
void ro_gemm_oracle(const float* a, int64_t m, int64_t k, const int8_t* logical, int64_t n,
                    int64_t g, const float* scales, float* out);
void ro_gemm_float(const float* a, int64_t m, int64_t k, const float* w, int64_t n,
                   int64_t block, float* out);
/* f64 oracle variant returning the unrounded double accumulators (for tolerance work). */
void ro_gemm_oracle_f64(const float* a, int64_t m, int64_t k, const int8_t* logical, int64_t n,
                        int64_t g, const float* scales, double* out);

/* Reference PRNG (proj/core/include/rtnq/rng.hpp:24-66). */
void ro_xoshiro_fill_unit(uint64_t seed, uint64_t stream, float* out, int64_t n, float mult);

#ifdef __cplusplus
}
#endif
#endif
