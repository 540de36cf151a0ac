/*
 * rtnq_capi.h -- the C-ABI boundary of the B200 rtnq library (librtnq_b200.so).
 *
 * The reference (/root/reference/proj) is a C++20 library with no FFI; its
 * public surface is the rtnq:: functions in proj/core/include/rtnq/*.hpp.  Each
 * entry point below is the plain-pointer, status-returning form of one of
 * those functions (cited), so that
 *   - include/rtnq/*.hpp (the drop-in C++ headers, implemented in
 *     paper_2505_15909_b200/csrc/dropin/) rebuilds reference consumers
 *     unchanged on top of it, and
 *   - Python (ctypes), or any other FFI, can bind it directly.
 *
 * Conventions
 *   - Every function returns an rtnq_status (0 = OK).  The message of the last
 *     failure on the calling thread is rtnq_last_error().  Status codes map
 *     1:1 onto the reference exception classes (proj/core/include/rtnq/error.hpp).
 *   - rtnq_dev_* functions take DEVICE pointers owned by the caller and a
 *     cudaStream_t passed as void*; they are asynchronous and never allocate
 *     (scratch comes from a caller-provided workspace sized by the matching
 *     *_workspace_bytes query).  Data-dependent errors (non-finite inputs) are
 *     reported through an optional device int32 flag; rtnq_dev_check_flag()
 *     synchronizes the stream and converts it into a status.
 *   - rtnq_* functions without the dev_ prefix take HOST buffers and are
 *     synchronous: they copy to the GPU, run the same kernels, copy back and
 *     validate exactly like the reference (same checks, same error classes).
 *     They exist for drop-in parity; the performance path is rtnq_dev_*.
 *   - There is no CPU compute fallback.  Without a usable CUDA device every
 *     compute entry point returns RTNQ_E_CUDA.
 */
#ifndef RTNQ_CAPI_H
#define RTNQ_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RTNQ_CAPI_VERSION 1

typedef int rtnq_status;
enum {
    RTNQ_OK = 0,
    RTNQ_E_INVALID_INPUT = 1, /* rtnq::InvalidInputError (error.hpp:19-23) */
    RTNQ_E_SHAPE = 2,         /* rtnq::ShapeError        (error.hpp:25-29) */
    RTNQ_E_CORRUPT = 3,       /* rtnq::CorruptDataError  (error.hpp:31-35) */
    RTNQ_E_PLAN = 4,          /* rtnq::PlanError         (error.hpp:37-53) */
    RTNQ_E_IO = 5,            /* rtnq::IoError           (error.hpp:55-59) */
    RTNQ_E_CUDA = 6,          /* no device / launch failure (no reference analogue) */
    RTNQ_E_INTERNAL = 7,
    RTNQ_E_UNSUPPORTED = 8    /* shape/dtype combination the chosen kernel cannot run */
};

/* Element types of activations, weights, scales and outputs. */
enum { RTNQ_F32 = 0, RTNQ_F16 = 1, RTNQ_BF16 = 2 };

/* Code layouts.  ROW_MAJOR and KERNEL_INTERLEAVED are the reference's
 * LayoutTag kinds (types.hpp:62-83); NATIVE_SM100 is the tensor-core operand
 * order of this library. */
enum { RTNQ_ROW_MAJOR = 0, RTNQ_KERNEL_INTERLEAVED = 1, RTNQ_NATIVE_SM100 = 2,
       RTNQ_NATIVE_I8 = 3, /* 128x128 pre-swizzled tiles: the int8-MMA operand of W8 per-channel */
       RTNQ_NATIVE_I4 = 4  /* 128-row x 128-code nibble tiles: the int8-MMA operand of W4 group-128 */ };

/* Scale orders: REF = [row][group] as in QuantTensor::scales (quant.hpp:33);
 * NATIVE = per 128-row row-block, [group][row padded to 8], so a
 * unit's scales are one contiguous 16-byte-aligned run. */
enum { RTNQ_SCALES_REF = 0, RTNQ_SCALES_NATIVE = 1 };

/* GEMM paths.  FUSED/DEQUANT_FIRST mirror rtnq::GemmPath (gemm.hpp:12); AUTO
 * is gemm_auto's rule (gemm.cpp:100-109); ORACLE is gemm_oracle. */
enum { RTNQ_PATH_FUSED = 0, RTNQ_PATH_DEQUANT_FIRST = 1, RTNQ_PATH_AUTO = 2,
       RTNQ_PATH_ORACLE = 3 };

typedef struct {
    int32_t kind;      /* RTNQ_ROW_MAJOR | RTNQ_KERNEL_INTERLEAVED | RTNQ_NATIVE_SM100 | RTNQ_NATIVE_I8 | RTNQ_NATIVE_I4 */
    int32_t tile_rows; /* KERNEL_INTERLEAVED only (LayoutTag::tile_rows, default 16) */
    int32_t tile_cols; /* KERNEL_INTERLEAVED only (LayoutTag::tile_cols, default 4) */
} rtnq_layout;

/* ---- library ------------------------------------------------------------------- */
int rtnq_version(void);
const char* rtnq_last_error(void);
/* Number of SMs of the current device (148 on B200); RTNQ_E_CUDA without a GPU. */
rtnq_status rtnq_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ---- geometry (pure host arithmetic; no GPU needed) ------------------------------- */
/* GroupSpec::groups_per_row (types.hpp:30-38); returns -status on error. */
int64_t rtnq_groups_per_row(int64_t g, int ragged, int64_t cols);
/* layout_slots (packing.hpp:43-45 / packing.cpp:68-73), plus the native kind. */
int64_t rtnq_layout_slots(rtnq_layout layout, int bits, int64_t rows, int64_t cols);
/* packed_size(layout_slots(...)) (packing.hpp:24-26): bytes of a code buffer. */
int64_t rtnq_layout_bytes(rtnq_layout layout, int bits, int64_t rows, int64_t cols);
/* layout_index (packing.hpp:39-41 / packing.cpp:57-66); -status if out of bounds. */
int64_t rtnq_layout_index(rtnq_layout layout, int bits, int64_t rows, int64_t cols, int64_t r,
                          int64_t c);
/* Elements of a native-order scale array for rows x gpr scales. */
int64_t rtnq_native_scale_count(int64_t rows, int64_t groups_per_row);

/* ---- device API (performance path) ------------------------------------------------ */

/* Fused RTN quantize-and-pack (replaces compute_scale + quantize_tensor + pack +
 * reshuffle: quant.cpp:49-68,100-141, packing.cpp:6-32,75-92).  Reads w
 * (rows x cols, row-major, dtype w_dtype) once and writes any non-NULL subset
 * of: row-major packed codes (== QuantTensor::data), kernel_interleaved(16,4)
 * packed codes (== reshuffle(q, LayoutTag::kernel()).data), native codes,
 * f32 scales (== QuantTensor::scales), f16 scales in reference order
 * (== f32_to_f16 of each), f16 scales in native order.  Bit-exact with the
 * reference.  Non-finite weights set *err_flag |= 1 (InvalidInputError). */
size_t rtnq_dev_quantize_workspace_bytes(int64_t rows, int64_t cols, int bits, int64_t g,
                                         int ragged);
rtnq_status rtnq_dev_quantize_pack(const void* w, int w_dtype, int64_t rows, int64_t cols,
                                   int bits, int64_t g, int ragged, uint8_t* codes_row_major,
                                   uint8_t* codes_kernel16x4, uint8_t* codes_native,
                                   float* scales_f32, uint16_t* scales_f16,
                                   uint16_t* scales_f16_native, int32_t* err_flag,
                                   void* workspace, size_t workspace_bytes, void* stream);

/* rtnq_dev_quantize_pack with the layout of `codes_native` chosen by native_kind:
 * RTNQ_NATIVE_SM100 (== rtnq_dev_quantize_pack), RTNQ_NATIVE_I4 (W4 group 128) or
 * RTNQ_NATIVE_I8 (W8 per-channel).  For the two int8-MMA layouts, when no
 * kernel_interleaved output is requested and cols % 128 == 0 (I4) / cols % 16 == 0 (I8),
 * ONE kernel reads the weights once and writes the native tiles (padding included), the
 * optional row-major bytes and the scales; otherwise the row-major bytes are quantized first
 * (caller's codes_row_major or the workspace) and relaid out. */
size_t rtnq_dev_quantize_workspace_bytes_ex(int64_t rows, int64_t cols, int bits, int64_t g,
                                            int ragged, int native_kind);
rtnq_status rtnq_dev_quantize_pack_ex(const void* w, int w_dtype, int64_t rows, int64_t cols,
                                      int bits, int64_t g, int ragged, int native_kind,
                                      uint8_t* codes_row_major, uint8_t* codes_kernel16x4,
                                      uint8_t* codes_native, float* scales_f32,
                                      uint16_t* scales_f16, uint16_t* scales_f16_native,
                                      int32_t* err_flag, void* workspace, size_t workspace_bytes,
                                      void* stream);

/* Layout conversion of packed codes (reshuffle, packing.cpp:75-92, generalized
 * to any pair of kinds; used to load row-major RTNCKPT1 codes into the native
 * layout).  Pure permutation plus zero padding. */
rtnq_status rtnq_dev_relayout(const uint8_t* src, rtnq_layout from, uint8_t* dst, rtnq_layout to,
                              int bits, int64_t rows, int64_t cols, void* stream);

/* Reference-order scales (f32 or f16) -> native-order f16 scales. */
rtnq_status rtnq_dev_native_scales(const void* scales, int scales_dtype, int64_t rows,
                                   int64_t groups_per_row, uint16_t* out, void* stream);

/* dequantize_tensor (quant.cpp:143-171): out[r][c] = float(code) * scale,
 * rounded once to out_dtype.  Bit-exact for RTNQ_F32. */
rtnq_status rtnq_dev_dequantize(const uint8_t* codes, rtnq_layout layout, int bits, int64_t rows,
                                int64_t cols, int64_t g, const void* scales, int scales_dtype,
                                int scales_order, void* out, int out_dtype, void* stream);

/* The quantized linear: out (m x n) = a (m x k) * W^T, W = codes * scales
 * (gemm.hpp:18-49).  Kernel selection:
 *   FUSED, NATIVE_SM100 codes, a in BF16/F16, scales F16 native order:
 *       sm_100a tensor-core W4A16/W8A16 kernel (tcgen05.mma with the weights
 *       dequantized into TMEM, TMA pipeline, stream-K with a deterministic
 *       fixup).  Needs g % 16 == 0 or g >= k, k % 8 == 0 and
 *       16-byte aligned a / codes / scales.
 *   FUSED, any layout, a in F32, scales F32 reference order:
 *       reference-exact CUDA-core kernel, bit-identical to gemm_fused
 *       (gemm.cpp:46-92).
 *   DEQUANT_FIRST, a in F32: dequantize + blocked f32 GEMM, bit-identical to
 *       gemm_dequant (gemm.cpp:94-98).
 *   ORACLE: f64 accumulation, bit-identical to gemm_oracle (gemm.cpp:121-149).
 *   AUTO: m >= threshold ? DEQUANT_FIRST : FUSED (gemm.cpp:100-109);
 *       *chosen (nullable) receives the path taken.
 * err_flag (nullable): set to 1 if any activation is non-finite (checked by a
 * separate pass; InvalidInputError in the reference, gemm.cpp:17-18). */
size_t rtnq_dev_linear_workspace_bytes(int64_t m, int64_t n, int64_t k, int bits, int64_t g,
                                       int path, rtnq_layout layout);
rtnq_status rtnq_dev_linear(const void* a, int a_dtype, int64_t m, int64_t k,
                            const uint8_t* codes, rtnq_layout layout, int bits, int64_t n,
                            int64_t g, int ragged, const void* scales, int scales_dtype,
                            int scales_order, void* out, int out_dtype, int path,
                            int64_t threshold, int* chosen, int32_t* err_flag, void* workspace,
                            size_t workspace_bytes, void* stream);

/* rtnq_dev_linear with launch flags.  RTNQ_FLAG_PDL launches the tensor-core
 * kernel with programmatic dependent launch: its weight prefetch starts before
 * the previous kernel in the stream finishes (only activations wait), so the
 * caller asserts that the previous kernel does not write this weight's codes or
 * scales -- true for every linear of a decode step. */
#define RTNQ_FLAG_PDL 1u
rtnq_status rtnq_dev_linear_ex(const void* a, int a_dtype, int64_t m, int64_t k,
                               const uint8_t* codes, rtnq_layout layout, int bits, int64_t n,
                               int64_t g, int ragged, const void* scales, int scales_dtype,
                               int scales_order, void* out, int out_dtype, int path,
                               int64_t threshold, int* chosen, int32_t* err_flag,
                               void* workspace, size_t workspace_bytes, void* stream,
                               unsigned flags);

/* gemm_float (gemm.cpp:111-119): dense f32 weights, blocked accumulation. */
rtnq_status rtnq_dev_gemm_float(const float* a, int64_t m, int64_t k, const float* w, int64_t n,
                                int64_t block, float* out, void* stream);

/* ---- decode layer (the callers around the linear; SURVEY §3C toy.cpp:91-117, with
 * Llama-3.1 GQA/RoPE/KV cache).  bf16 device tensors, f32 math, async on `stream`. */
/* x (m x h) += delta (nullable), then out = rmsnorm(x) * weight (toy.cpp:19-30). */
rtnq_status rtnq_dev_add_rmsnorm(void* x, const void* delta, const void* weight, void* out,
                                 int64_t m, int64_t h, float eps, void* stream);
/* act (m x f) = silu(gate_up[:, :f]) * gate_up[:, f:] (toy.cpp:108-112). */
rtnq_status rtnq_dev_silu_mul(const void* gate_up, void* act, int64_t m, int64_t f, void* stream);
/* The int8 kernels' activation planes (a = 2^s (P0 + P1/2^7 + P2/2^14)):
 * planes [3][m][k] int8 and exponents [m] int32, device buffers.  rtnq_dev_act_planes computes
 * them from a bf16/f16 activation; the _planes variants of add+RMSNorm and SiLU*up emit them
 * for their bf16 output rows in the same kernel; rtnq_dev_linear_planes then runs the W4
 * (RTNQ_NATIVE_I4) or W8 (RTNQ_NATIVE_I8) linear on them without recomputing. */
rtnq_status rtnq_dev_act_planes(const void* a, int a_dtype, int64_t m, int64_t k, int8_t* planes,
                                int32_t* texp, void* stream);
rtnq_status rtnq_dev_add_rmsnorm_planes(void* x, const void* delta, const void* weight, void* out,
                                        int64_t m, int64_t h, float eps, int8_t* planes, int32_t* texp,
                                        void* stream);
rtnq_status rtnq_dev_silu_mul_planes(const void* gate_up, void* act, int64_t m, int64_t f,
                                     int8_t* planes, int32_t* texp, void* stream);
rtnq_status rtnq_dev_linear_planes(const int8_t* planes, const int32_t* texp, int64_t m, int64_t k,
                                   const uint8_t* codes, rtnq_layout layout, int bits, int64_t n,
                                   int64_t g, int ragged, const void* scales, int sdtype, int sorder,
                                   void* out, int odtype, void* ws, size_t ws_bytes, void* stream,
                                   unsigned flags);
/* One decode step of GQA attention: qkv rows [hq*d | hkv*d | hkv*d]; the rotated key and
 * the value are appended to the caches ([batch][max_len][hkv][d]) at `pos`, then each
 * query head attends over positions [0, pos].  head_dim 128, hq/hkv <= 32.
 * With <= 8 query heads per KV head the kernel is launched as a programmatic dependent of the
 * previous kernel on the stream and reads the cached rows [0, pos) BEFORE waiting for it (they
 * stream in under that kernel's tail): those rows must not be written by the kernel launched
 * immediately before this call (a decode stack writes them one step earlier).  RTNQ_ATTN_PDL=0
 * launches it stream-ordered. */
rtnq_status rtnq_dev_decode_attention(const void* qkv, void* k_cache, void* v_cache, void* out,
                                      int64_t batch, int64_t hq, int64_t hkv, int64_t head_dim,
                                      int64_t max_len, int64_t pos, float rope_theta,
                                      void* stream);
/* The same with the split-context merge scratch (self-resetting counters + partials) from a
 * caller workspace of rtnq_dev_decode_attention_workspace_bytes(batch, hq, hkv, max_len) bytes,
 * zero-initialized once and reused per stream; rtnq_dev_decode_attention uses a per-device
 * buffer instead (one stream at a time). */
size_t rtnq_dev_decode_attention_workspace_bytes(int64_t batch, int64_t hq, int64_t hkv, int64_t max_len);
rtnq_status rtnq_dev_decode_attention_ws(const void* qkv, void* k_cache, void* v_cache, void* out,
                                         int64_t batch, int64_t hq, int64_t hkv, int64_t head_dim,
                                         int64_t max_len, int64_t pos, float rope_theta, void* ws,
                                         size_t ws_bytes, void* stream);
/* The same, also writing the activation planes ([3][batch][hq * head_dim] int8, [batch] exponents)
 * of `out` for the int8 o-projection (rtnq_dev_linear_planes): the last CTA of each token computes
 * them from the token's output row, so the o-projection needs no planes kernel. */
rtnq_status rtnq_dev_decode_attention_planes(const void* qkv, void* k_cache, void* v_cache, void* out,
                                             int64_t batch, int64_t hq, int64_t hkv, int64_t head_dim,
                                             int64_t max_len, int64_t pos, float rope_theta, int8_t* planes,
                                             int32_t* texp, void* ws, size_t ws_bytes, void* stream);
/* Synchronizes `stream`, reads and clears *err_flag (device), returns
 * RTNQ_E_INVALID_INPUT if it was set. */
rtnq_status rtnq_dev_check_flag(int32_t* err_flag, void* stream);

/* ---- tensor-parallel partial sums over peer memory ------------------
 * Replaces the allreduce the reference's tensor-parallel split would need after a
 * row-split linear (no reference counterpart: the reference is single-device; the
 * sharding follows the Llama TP layout of SURVEY §8e).
 *
 * Every rank owns one symmetric buffer of rtnq_peer_buffer_bytes(cap) bytes
 * (rtnq_peer_alloc: zero-filled, its own allocation; cap = elements per slot, a
 * multiple of 8, >= tokens x hidden) and maps every peer's buffer: same process (one process
 * driving several devices, rtnq_peer_enable) or other processes (CUDA IPC:
 * rtnq_ipc_get_handle -> exchange -> rtnq_ipc_open).  peer_bufs[q] is rank q's
 * buffer as seen from this rank's device.
 *
 * A round: every rank runs rtnq_dev_linear_peer (its row-split partial goes
 * straight from the GEMM epilogue into its slot of every rank's buffer, bf16, then
 * a release flag), then one consumer on its own buffer: rtnq_dev_add_rmsnorm_peer
 * (x += sum of the partials, then RMSNorm, as rtnq_dev_add_rmsnorm with
 * delta = allreduce(partial)) or rtnq_dev_peer_reduce.  The sum runs over ranks
 * 0..world-1 in order in f32 with one bf16 rounding, so every rank gets the same
 * bits.  Consumers wait on the device; a rank's next producer must follow its
 * consumer in stream order. */
#define RTNQ_IPC_HANDLE_BYTES 64
size_t rtnq_peer_buffer_bytes(int64_t cap);
/* a zero-filled symmetric buffer of its own cudaMalloc allocation on the current device (an IPC
 * handle maps whole allocations, so the buffer must not be carved out of a pool) */
rtnq_status rtnq_peer_alloc(int64_t cap, void** dev_ptr);
rtnq_status rtnq_peer_free(void* dev_ptr);
rtnq_status rtnq_ipc_get_handle(void* dev_ptr, void* handle);
rtnq_status rtnq_ipc_open(const void* handle, void** dev_ptr);
rtnq_status rtnq_ipc_close(void* dev_ptr);
/* let `device` access `peer`'s memory (one process, several devices; no-op when equal) */
rtnq_status rtnq_peer_enable(int device, int peer);
/* rtnq_dev_linear_planes / rtnq_dev_linear with the output pushed to the peers:
 * either `a` (bf16 m x k) or `planes` + `texp`; m <= 64, m * n <= cap. */
rtnq_status rtnq_dev_linear_peer(const void* a, const int8_t* planes, const int32_t* texp, int64_t m,
                                 int64_t k, const uint8_t* codes, rtnq_layout layout, int bits, int64_t n,
                                 int64_t g, int ragged, const void* scales, int sdtype, int sorder,
                                 void* const* peer_bufs, int world, int rank, int64_t cap,
                                 int32_t* err_flag, void* ws, size_t ws_bytes, void* stream,
                                 unsigned flags);
/* x (m x h) += sum of the round's partials (this rank's buffer), out = rmsnorm(x) * weight,
 * optional planes of out (as rtnq_dev_add_rmsnorm_planes). */
rtnq_status rtnq_dev_add_rmsnorm_peer(void* x, void* peer_buf, int world, int64_t cap,
                                      const void* weight, void* out, int64_t m, int64_t h, float eps,
                                      int8_t* planes, int32_t* texp, void* stream);
/* out[0..n) = (accumulate ? out + : ) sum of the round's partials. */
rtnq_status rtnq_dev_peer_reduce(void* peer_buf, int world, int64_t cap, void* out, int64_t n,
                                 int accumulate, void* stream);

/* ---- host API (drop-in parity path; synchronous; host buffers) -------------------- */

/* compute_scale (quant.hpp:48-50). */
rtnq_status rtnq_compute_scale(const float* values, int64_t n, int bits, float* scale_out);
/* quantize_group (quant.hpp:52-57).  scale_in == NULL computes the scale
 * (the float* overload); otherwise *scale_in is used as given. */
rtnq_status rtnq_quantize_group(const float* values, int64_t n, int bits, const float* scale_in,
                                float* scale_out, int8_t* codes_out);
/* dequantize_group (quant.hpp:59-62); CorruptData on out-of-range codes. */
rtnq_status rtnq_dequantize_group(const int8_t* codes, int64_t n, float scale, int bits,
                                  float* out);
/* quantize_tensor (quant.hpp:64-67): row-major packed data + f32 scales. */
rtnq_status rtnq_quantize_tensor(const float* w, int64_t rows, int64_t cols, int bits, int64_t g,
                                 int ragged, uint8_t* data_out, float* scales_out);
/* pack (packing.hpp:28): codes -> offset-binary bytes; InvalidInput if out of range. */
rtnq_status rtnq_pack(const int8_t* codes, int64_t n, int bits, uint8_t* out);
/* unpack (packing.hpp:30-32); CorruptData if nbytes != packed_size(n, bits). */
rtnq_status rtnq_unpack(const uint8_t* bytes, int64_t nbytes, int64_t n, int bits, int8_t* out);
/* logical_codes (quant.hpp:73-74): codes of any layout in row-major order. */
rtnq_status rtnq_logical_codes(const uint8_t* data, int64_t nbytes, rtnq_layout layout, int bits,
                               int64_t rows, int64_t cols, int8_t* out);
/* reshuffle (packing.hpp:47-49) between any two layouts. */
rtnq_status rtnq_reshuffle(const uint8_t* data, int64_t nbytes, rtnq_layout from, rtnq_layout to,
                           int bits, int64_t rows, int64_t cols, uint8_t* out);
/* dequantize_tensor (quant.hpp:69-71). */
rtnq_status rtnq_dequantize_tensor(const uint8_t* data, int64_t nbytes, rtnq_layout layout,
                                   int bits, int64_t rows, int64_t cols, int64_t g, int ragged,
                                   const float* scales, float* out);
/* gemm_fused / gemm_dequant / gemm_auto / gemm_oracle (gemm.hpp:31-44). */
rtnq_status rtnq_gemm(int path, const float* a, int64_t m, int64_t k, const uint8_t* data,
                      int64_t nbytes, rtnq_layout layout, int bits, int64_t n, int64_t g,
                      int ragged, const float* scales, int64_t threshold, int* chosen,
                      float* out);
/* f32_to_f16 / f16_to_f32 (f16.hpp:13-16, f16.cpp:8-63) over arrays: RNE narrowing
 * (quiet NaN kept), exact widening.  Pure host functions (no device needed). */
rtnq_status rtnq_f32_to_f16(const float* in, int64_t n, uint16_t* out);
rtnq_status rtnq_f16_to_f32(const uint16_t* in, int64_t n, float* out);
/* gemm_float (gemm.hpp:46-49). */
rtnq_status rtnq_gemm_float(const float* a, int64_t m, int64_t k, const float* w, int64_t n,
                            int64_t block, float* out);

/* ---- selective precision (plan.hpp:84-110; host-only logic) ----------------------- */
/* parse_plan + render_plan + resolve_plan.  table (nullable, layers*4 bytes)
 * receives 4 or 8 per (layer, module) slot (slot = layer*4 + module_id-1).
 * canonical (nullable) receives render_plan(parse_plan(text)).  On a parse
 * error returns RTNQ_E_PLAN with *error_offset = byte offset (-1 if none). */
rtnq_status rtnq_plan_resolve(const char* text, int64_t layers, uint8_t* table,
                              char* canonical, int64_t canonical_cap, int64_t* error_offset);
/* effective_bits (plan.hpp:105-110) of a table over per-module shapes
 * rows[4] x cols[4] with group g. */
rtnq_status rtnq_effective_bits(const uint8_t* table, int64_t layers, const int64_t* rows4,
                                const int64_t* cols4, int64_t g, int include_scales,
                                double* out);

#ifdef __cplusplus
}
#endif
#endif /* RTNQ_CAPI_H */
