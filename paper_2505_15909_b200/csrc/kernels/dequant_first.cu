// dequant_first.cu -- the dequant-first linear on the tensor cores (the reference's
// gemm_dequant, gemm.cpp:94-98, and the m >= threshold branch of gemm_auto, :100-109).
//
// For large batches the fused weight-only kernels re-stream the weights once per 64-token
// chunk, while a dequantized weight matrix feeds a plain tensor-core GEMM at full rate.  The
// weights are dequantized exactly (W = S * code in f32, quant.cpp:143-171) and split into two
// 16-bit terms, W = hi + lo with hi = round16(W), lo = round16(W - hi): 16 + 16 significant bits
// cover the f16 scale (11) times the code (<= 8), so hi + lo is W to about 2^-17.  Then
//   out = a . hi^T + a . lo^T
// as two cuBLAS GEMMs (16-bit inputs, f32 accumulate and f32 C) -- a plain library GEMM, the
// one place this library calls cuBLAS.  Activations are exact in their 16-bit type, so the
// result matches the f32 reference path within the 1e-5 parity bar.
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <mutex>
#include <unordered_map>

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
                                     int sorder, T* __restrict__ hi, T* __restrict__ lo) {
    const int64_t n = rows * cols;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / cols, c = i % cols;
        const int code = code_at_slot(codes, bits, layout_slot(L, bits, rows, cols, r, c), L.kind);
        const int64_t j = c / g;
        const int64_t si = sorder == RTNQ_SCALES_NATIVE ? native_scale_index(rows, gpr, r, j) : r * gpr + j;
        const float w = __fmul_rn(float(code), __half2float(__ushort_as_half(scales[si])));
        const T h = to16<T>(w);
        hi[i] = h;
        lo[i] = to16<T>(w - from16<T>(h));
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

__global__ void cast_out_kernel(const float* __restrict__ c, void* __restrict__ out, int odtype, int64_t n) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        store_elem(out, odtype, i, c[i]);
}

cublasHandle_t handle_for_device() {
    static std::mutex mu;
    static std::unordered_map<int, cublasHandle_t> handles;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = handles.find(dev);
    if (it != handles.end()) return it->second;
    cublasHandle_t h = nullptr;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    cublasSetMathMode(h, CUBLAS_DEFAULT_MATH);  // no TF32 down-conversion of the f32 C
    handles[dev] = h;
    return h;
}

}  // namespace

size_t dequant_first_workspace_bytes(int64_t m, int64_t n, int64_t k, int odtype) {
    const size_t w = size_t(n) * size_t(k) * 2;  // one 16-bit term
    const size_t c = odtype == RTNQ_F32 ? 0 : size_t(m) * size_t(n) * 4;
    return 2 * ((w + 255) / 256 * 256) + c;
}

const char* launch_dequant_first(const void* a, int a_dtype, int64_t m, int64_t n, int64_t k,
                                 const uint8_t* codes, Layout L, int bits, int64_t g, int64_t gpr,
                                 const uint16_t* scales, int sorder, void* out, int odtype, void* ws,
                                 cudaStream_t st) {
    if (a_dtype != RTNQ_BF16 && a_dtype != RTNQ_F16) return "dequant-first tensor path needs bf16/f16 activations";
    cublasHandle_t h = handle_for_device();
    if (!h) return "cublasCreate failed";
    const size_t wbytes = (size_t(n) * size_t(k) * 2 + 255) / 256 * 256;
    char* wsb = static_cast<char*>(ws);
    void* hi = wsb;
    void* lo = wsb + wbytes;
    float* c = odtype == RTNQ_F32 ? static_cast<float*>(out) : reinterpret_cast<float*>(wsb + 2 * wbytes);
    const int64_t nk = n * k;
    const unsigned blocks = unsigned(nk / 256 + 1 < 148 * 16 ? nk / 256 + 1 : 148 * 16);
    if (k % 8 == 0) {
        const unsigned b8 = unsigned(nk / 8 / 256 + 1 < 148 * 16 ? nk / 8 / 256 + 1 : 148 * 16);
        if (a_dtype == RTNQ_BF16)
            dequant_split8_kernel<__nv_bfloat16><<<b8, 256, 0, st>>>(codes, L, bits, n, k, g, gpr, scales, sorder,
                                                                    static_cast<__nv_bfloat16*>(hi),
                                                                    static_cast<__nv_bfloat16*>(lo));
        else
            dequant_split8_kernel<__half><<<b8, 256, 0, st>>>(codes, L, bits, n, k, g, gpr, scales, sorder,
                                                             static_cast<__half*>(hi), static_cast<__half*>(lo));
    } else if (a_dtype == RTNQ_BF16)
        dequant_split_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(codes, L, bits, n, k, g, gpr, scales, sorder,
                                                                   static_cast<__nv_bfloat16*>(hi),
                                                                   static_cast<__nv_bfloat16*>(lo));
    else
        dequant_split_kernel<__half><<<blocks, 256, 0, st>>>(codes, L, bits, n, k, g, gpr, scales, sorder,
                                                            static_cast<__half*>(hi), static_cast<__half*>(lo));
    if (cudaGetLastError() != cudaSuccess) return "dequant kernel launch failed";
    if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) return "cublasSetStream failed";
    // row-major out[m][n] = a[m][k] . W[n][k]^T  ==  column-major C(n x m) = W^T(op T) . a
    const cudaDataType_t t = a_dtype == RTNQ_BF16 ? CUDA_R_16BF : CUDA_R_16F;
    const float one = 1.0f, zero = 0.0f;
    for (int term = 0; term < 2; ++term) {
        const cublasStatus_t s = cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, int(n), int(m), int(k), &one,
                                              term ? lo : hi, t, int(k), a, t, int(k), term ? &one : &zero, c,
                                              CUDA_R_32F, int(n), CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
        if (s != CUBLAS_STATUS_SUCCESS) return "cublasGemmEx failed";
    }
    if (odtype != RTNQ_F32) {
        const int64_t mn = m * n;
        cast_out_kernel<<<unsigned(mn / 256 + 1 < 148 * 8 ? mn / 256 + 1 : 148 * 8), 256, 0, st>>>(c, out, odtype, mn);
        if (cudaGetLastError() != cudaSuccess) return "cast kernel launch failed";
    }
    return nullptr;
}

}  // namespace rtnq_b200
