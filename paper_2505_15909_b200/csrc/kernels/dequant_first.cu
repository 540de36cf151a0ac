// dequant_first.cu -- the dequant-first linear on the tensor cores (the reference's
// gemm_dequant, gemm.cpp:94-98, and the m >= threshold branch of gemm_auto, :100-109).
//
// For large batches the fused weight-only kernels re-stream the weights once per 64-token
// chunk, while a dequantized weight matrix feeds a plain tensor-core GEMM at full rate.  The
// weights are dequantized exactly (W = S * code in f32, quant.cpp:143-171) and split into two
// 16-bit terms, W = hi + lo with hi = round16(W), lo = round16(W - hi): 16 + 16 significant bits
// cover the f16 scale (11) times the code (<= 8), so hi + lo is W to about 2^-17.  Then
//   out = a . hi^T + a . lo^T
// in one hand-written tcgen05 kernel (dense_tc.cu: both terms into one f32 TMEM accumulator,
// the output type written by its epilogue).  Activations are exact in their 16-bit type, so
// the result matches the f32 reference path within the 1e-5 parity bar.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>


#include "../common.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {
namespace {

template <typename T>
__device__ __forceinline__ T to16(float v);
template <>
__device__ __forceinline__ __nv_bfloat16 to16<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ __half to16<__half>(float v) { return __float2half_rn(v); }
template <typename T>
__device__ __forceinline__ float from16(T v);
template <>
__device__ __forceinline__ float from16<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
__device__ __forceinline__ float from16<__half>(__half v) { return __half2float(v); }

// One thread per weight, row-major hi/lo output; the code comes from any layout.
template <typename T>
__global__ void dequant_split_kernel(const uint8_t* __restrict__ codes, Layout L, int bits, int64_t rows,
                                     int64_t cols, int64_t g, int64_t gpr, const uint16_t* __restrict__ scales,
                                     int sorder, T* __restrict__ hi, T* __restrict__ lo, int64_t ld) {
    const int64_t n = rows * cols;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / cols, c = i % cols;
        const int code = code_at_slot(codes, bits, layout_slot(L, bits, rows, cols, r, c), L.kind);
        const int64_t j = c / g;
        const int64_t si = sorder == RTNQ_SCALES_NATIVE ? native_scale_index(rows, gpr, r, j) : r * gpr + j;
        const float w = __fmul_rn(float(code), __half2float(__ushort_as_half(scales[si])));
        const T h = to16<T>(w);
        hi[r * ld + c] = h;
        lo[r * ld + c] = to16<T>(w - from16<T>(h));
    }
}

// The int8-MMA layouts tile by tile (one thread per 16-byte chunk of a tile row, no per-weight
// layout arithmetic): RTNQ_NATIVE_I4 (8 KiB tiles, chunk q of row r at ((q ^ (r / 2 % 4)) * 16),
// byte p = code(p) << 4 | code(64 + p), 4-bit two's complement) and RTNQ_NATIVE_I8 (16 KiB
// 128B-swizzled s8 tiles, chunk c at ((c ^ r % 8) * 16)); rows [n][ld], codes past cols skipped.
template <typename T, int BITS>
__global__ void dequant_split_native_kernel(const uint8_t* __restrict__ codes, int64_t rows, int64_t cols,
                                            int64_t g, int64_t gpr, const uint16_t* __restrict__ scales,
                                            T* __restrict__ hi, T* __restrict__ lo, int64_t ld) {
    constexpr int CPR = BITS == 4 ? 4 : 8;             // 16-byte chunks per 128-code tile row
    constexpr int TILE = BITS == 4 ? 8192 : 16384;
    const int64_t kt = (cols + 127) / 128, total = rows * kt * CPR;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int q = int(i % CPR);
        const uint32_t rt = uint32_t(i / CPR);  // rows * tiles per row < 2^32 (checked by the launcher)
        const int64_t t = rt % uint32_t(kt), r = rt / uint32_t(kt), rr = r & 127;
        const int64_t tile = (r >> 7) * kt + t;
        const int sw = BITS == 4 ? int((rr >> 1) & 3) : int(rr & 7);
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(codes + tile * TILE + rr * (TILE / 128) + ((q ^ sw) << 4)));
        const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
        // (k of byte e, run 0 / run 1): W4 k = 128 t + 16 q + e and + 64; W8 k = 128 t + 16 q + e
#pragma unroll
        for (int run = 0; run < (BITS == 4 ? 2 : 1); ++run) {
            const int64_t k0 = 128 * t + 16 * q + 64 * run;
            if (k0 >= cols) continue;
            alignas(16) T h[16], l[16];
            // one scale per run: these layouts have g = 128 or one group per row, so a 16-aligned
            // run of 16 codes never crosses a group
            const float s = __half2float(__ushort_as_half(scales[native_scale_index(rows, gpr, r, k0 / g)]));
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int code = BITS == 4 ? (run == 0 ? int(int8_t(b[e])) >> 4 : int(int8_t(b[e] << 4)) >> 4)
                                           : int(int8_t(b[e]));
                const float w = __fmul_rn(float(code), s);
                h[e] = to16<T>(w);
                l[e] = to16<T>(w - from16<T>(h[e]));
            }
            T* ho = hi + r * ld + k0;
            T* lo_ = lo + r * ld + k0;
            if (k0 + 16 <= cols && (ld & 7) == 0) {
                reinterpret_cast<uint4*>(ho)[0] = reinterpret_cast<const uint4*>(h)[0];
                reinterpret_cast<uint4*>(ho)[1] = reinterpret_cast<const uint4*>(h)[1];
                reinterpret_cast<uint4*>(lo_)[0] = reinterpret_cast<const uint4*>(l)[0];
                reinterpret_cast<uint4*>(lo_)[1] = reinterpret_cast<const uint4*>(l)[1];
            } else {
                for (int e = 0; e < 16 && k0 + e < cols; ++e) ho[e] = h[e], lo_[e] = l[e];
            }
        }
    }
}

// Eight consecutive columns per thread (cols % 8 == 0): one 64-bit division per 8 weights,
// 16-byte stores of hi and lo.
template <typename T>
__global__ void dequant_split8_kernel(const uint8_t* __restrict__ codes, Layout L, int bits, int64_t rows,
                                      int64_t cols, int64_t g, int64_t gpr, const uint16_t* __restrict__ scales,
                                      int sorder, T* __restrict__ hi, T* __restrict__ lo) {
    const int64_t n8 = rows * cols / 8, c8 = cols / 8;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / c8, c0 = (i - r * c8) * 8;
        alignas(16) T h[8], l[8];
        int64_t jprev = -1;
        float s = 0.0f;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int64_t c = c0 + e, j = c / g;
            if (j != jprev) {
                const int64_t si = sorder == RTNQ_SCALES_NATIVE ? native_scale_index(rows, gpr, r, j) : r * gpr + j;
                s = __half2float(__ushort_as_half(scales[si]));
                jprev = j;
            }
            const int code = code_at_slot(codes, bits, layout_slot(L, bits, rows, cols, r, c), L.kind);
            const float w = __fmul_rn(float(code), s);
            h[e] = to16<T>(w);
            l[e] = to16<T>(w - from16<T>(h[e]));
        }
        *reinterpret_cast<uint4*>(hi + i * 8) = *reinterpret_cast<const uint4*>(h);
        *reinterpret_cast<uint4*>(lo + i * 8) = *reinterpret_cast<const uint4*>(l);
    }
}

}  // namespace

// [hi | lo] with rows padded to 8 elements (the TMA row stride), plus a padded copy of the
// activations when k % 8 != 0
static int64_t pad8(int64_t k) { return (k + 7) / 8 * 8; }
static size_t round256(size_t b) { return (b + 255) / 256 * 256; }

size_t dequant_first_workspace_bytes(int64_t m, int64_t n, int64_t k, int odtype) {
    (void)odtype;  // the output type is written by the GEMM's epilogue
    const size_t w = round256(size_t(n) * size_t(pad8(k)) * 2);
    const size_t a = round256(size_t(m) * size_t(pad8(k)) * 2);  // used if k % 8 or a is unaligned
    return 2 * w + a;
}

const char* launch_dequant_first(const void* a, int a_dtype, int64_t m, int64_t n, int64_t k,
                                 const uint8_t* codes, Layout L, int bits, int64_t g, int64_t gpr,
                                 const uint16_t* scales, int sorder, void* out, int odtype, void* ws,
                                 cudaStream_t st) {
    if (a_dtype != RTNQ_BF16 && a_dtype != RTNQ_F16) return "dequant-first tensor path needs bf16/f16 activations";
    const int64_t kp = pad8(k);
    const size_t wbytes = round256(size_t(n) * size_t(kp) * 2);
    char* wsb = static_cast<char*>(ws);
    void* hi = wsb;
    void* lo = wsb + wbytes;
    const void* ap = a;
    const bool copy_a = k % 8 || (reinterpret_cast<uintptr_t>(a) & 15);  // the TMA needs 16-byte rows and base
    if (copy_a) {
        void* acopy = wsb + 2 * wbytes;
        if (cudaMemsetAsync(acopy, 0, size_t(m) * size_t(kp) * 2, st) != cudaSuccess ||
            cudaMemcpy2DAsync(acopy, size_t(kp) * 2, a, size_t(k) * 2, size_t(k) * 2, size_t(m),
                              cudaMemcpyDeviceToDevice, st) != cudaSuccess)
            return "dequant-first: activation copy failed";
        ap = acopy;
    }
    const int64_t nk = n * k;
    const bool native_i = sorder == RTNQ_SCALES_NATIVE &&
                          ((L.kind == RTNQ_NATIVE_I4 && bits == 4) || (L.kind == RTNQ_NATIVE_I8 && bits == 8)) &&
                          g % 16 == 0;
    if (native_i) {
        if (k % 8 && cudaMemsetAsync(hi, 0, 2 * wbytes, st) != cudaSuccess) return "dequant-first: memset failed";
        const int64_t chunks = n * ((k + 127) / 128) * (bits == 4 ? 4 : 8);
        if (n * ((k + 127) / 128) >= (int64_t(1) << 32)) return "dequant-first: weight too large";
        const unsigned bl = unsigned(chunks / 256 + 1 < 148 * 16 ? chunks / 256 + 1 : 148 * 16);
        if (a_dtype == RTNQ_BF16 && bits == 4)
            dequant_split_native_kernel<__nv_bfloat16, 4><<<bl, 256, 0, st>>>(
                codes, n, k, g, gpr, scales, static_cast<__nv_bfloat16*>(hi), static_cast<__nv_bfloat16*>(lo), kp);
        else if (a_dtype == RTNQ_BF16)
            dequant_split_native_kernel<__nv_bfloat16, 8><<<bl, 256, 0, st>>>(
                codes, n, k, g, gpr, scales, static_cast<__nv_bfloat16*>(hi), static_cast<__nv_bfloat16*>(lo), kp);
        else if (bits == 4)
            dequant_split_native_kernel<__half, 4><<<bl, 256, 0, st>>>(codes, n, k, g, gpr, scales,
                                                                      static_cast<__half*>(hi), static_cast<__half*>(lo), kp);
        else
            dequant_split_native_kernel<__half, 8><<<bl, 256, 0, st>>>(codes, n, k, g, gpr, scales,
                                                                      static_cast<__half*>(hi), static_cast<__half*>(lo), kp);
    } else if (k % 8 == 0) {
        const unsigned b8 = unsigned(nk / 8 / 256 + 1 < 148 * 16 ? nk / 8 / 256 + 1 : 148 * 16);
        if (a_dtype == RTNQ_BF16)
            dequant_split8_kernel<__nv_bfloat16><<<b8, 256, 0, st>>>(codes, L, bits, n, k, g, gpr, scales, sorder,
                                                                    static_cast<__nv_bfloat16*>(hi),
                                                                    static_cast<__nv_bfloat16*>(lo));
        else
            dequant_split8_kernel<__half><<<b8, 256, 0, st>>>(codes, L, bits, n, k, g, gpr, scales, sorder,
                                                             static_cast<__half*>(hi), static_cast<__half*>(lo));
    } else {
        // padded rows: the pad columns are zero (they meet the activations' zero pad)
        if (cudaMemsetAsync(hi, 0, 2 * wbytes, st) != cudaSuccess) return "dequant-first: memset failed";
        const unsigned blocks = unsigned(nk / 256 + 1 < 148 * 16 ? nk / 256 + 1 : 148 * 16);
        if (a_dtype == RTNQ_BF16)
            dequant_split_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(codes, L, bits, n, k, g, gpr, scales, sorder,
                                                                       static_cast<__nv_bfloat16*>(hi),
                                                                       static_cast<__nv_bfloat16*>(lo), kp);
        else
            dequant_split_kernel<__half><<<blocks, 256, 0, st>>>(codes, L, bits, n, k, g, gpr, scales, sorder,
                                                                static_cast<__half*>(hi), static_cast<__half*>(lo),
                                                                kp);
    }
    if (cudaGetLastError() != cudaSuccess) return "dequant kernel launch failed";
    // row-major out[m][n] = a[m][k] . (hi + lo)[n][k]^T, one tcgen05 kernel
    return launch_dense_hilo(ap, copy_a ? kp : k, hi, lo, kp, a_dtype, m, n, kp, out, odtype, st);
}

}  // namespace rtnq_b200
