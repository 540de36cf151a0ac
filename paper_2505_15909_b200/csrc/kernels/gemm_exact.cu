// gemm_exact.cu -- CUDA-core GEMMs with the reference's exact accumulation
// order, so the drop-in rtnq::gemm_* calls are bit-identical to the reference:
//   gemm_fused   (gemm.cpp:46-92)   per group: f32 block += a*code (k ascending),
//                                   then acc += S * block;
//   dense blocked (gemm.cpp:23-42)  per block of `blk`: block += a*w, acc += block
//                                   (gemm_dequant and gemm_float);
//   gemm_oracle  (gemm.cpp:121-149) f64 products and sum, one f32 rounding.
// Every product and sum is an explicit _rn intrinsic: no FMA contraction, like
// the reference's default x86-64 build.  These are the parity path for f32
// activations; the performance path is the tensor-core kernel in wgemm_sm100.cu.
#include "../common.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {

// One thread per output element; threads of a warp share the activation row
// (broadcast loads) and walk adjacent weight rows.
__global__ void gemm_fused_exact_kernel(const float* __restrict__ a, int64_t m, int64_t k,
                                        const uint8_t* __restrict__ codes, Layout L, int bits,
                                        int64_t n, int64_t g, int64_t gpr,
                                        const float* __restrict__ scales,
                                        float* __restrict__ out) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= m * n) return;
    const int64_t i = e / n, j = e % n;
    const float* arow = a + i * k;
    const float* srow = scales + j * gpr;
    // kernel_interleaved: constant slot stride for a fixed row (gemm.cpp:64-66)
    const bool inter = L.kind == RTNQ_KERNEL_INTERLEAVED;
    const int64_t tpr = inter ? (k + L.tc - 1) / L.tc : 0;
    const int64_t base = inter ? (j / L.tr) * tpr * L.tr * L.tc + j % L.tr : 0;
    float acc = 0.0f;
    for (int64_t q = 0; q < gpr; ++q) {
        const int64_t k0 = q * g, k1 = min(k0 + g, k);
        float block = 0.0f;
        for (int64_t kk = k0; kk < k1; ++kk) {
            const int64_t slot = inter ? base + kk * L.tr : layout_slot(L, bits, n, k, j, kk);
            block = __fadd_rn(block, __fmul_rn(arow[kk], float(code_at_slot(codes, bits, slot, L.kind))));
        }
        acc = __fadd_rn(acc, __fmul_rn(srow[q], block));
    }
    out[e] = acc;
}

__global__ void dense_blocked_kernel(const float* __restrict__ a, int64_t m, int64_t k,
                                     const float* __restrict__ w, int64_t n, int64_t blk,
                                     float* __restrict__ out) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= m * n) return;
    const int64_t i = e / n, j = e % n;
    const float* arow = a + i * k;
    const float* wrow = w + j * k;
    float acc = 0.0f;
    for (int64_t k0 = 0; k0 < k; k0 += blk) {
        const int64_t k1 = min(k0 + blk, k);
        float block = 0.0f;
        for (int64_t kk = k0; kk < k1; ++kk)
            block = __fadd_rn(block, __fmul_rn(arow[kk], wrow[kk]));
        acc = __fadd_rn(acc, block);
    }
    out[e] = acc;
}

__global__ void gemm_oracle_kernel(const float* __restrict__ a, int64_t m, int64_t k,
                                   const uint8_t* __restrict__ codes, Layout L, int bits,
                                   int64_t n, int64_t g, int64_t gpr,
                                   const float* __restrict__ scales, float* __restrict__ out) {
    const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= m * n) return;
    const int64_t i = e / n, j = e % n;
    double acc = 0.0;
    for (int64_t kk = 0; kk < k; ++kk) {
        const int code = code_at_slot(codes, bits, layout_slot(L, bits, n, k, j, kk), L.kind);
        const double wv = __dmul_rn(double(code), double(scales[j * gpr + kk / g]));
        acc = __dadd_rn(acc, __dmul_rn(double(a[i * k + kk]), wv));
    }
    out[e] = float(acc);
}

void launch_gemm_fused_exact(const float* a, int64_t m, int64_t k, const uint8_t* codes,
                             Layout L, int bits, int64_t n, int64_t g, int64_t gpr,
                             const float* scales, float* out, cudaStream_t st) {
    if (m * n == 0) return;
    gemm_fused_exact_kernel<<<unsigned((m * n + 127) / 128), 128, 0, st>>>(
        a, m, k, codes, L, bits, n, g, gpr, scales, out);
}

void launch_dense_blocked(const float* a, int64_t m, int64_t k, const float* w, int64_t n,
                          int64_t blk, float* out, cudaStream_t st) {
    if (m * n == 0) return;
    dense_blocked_kernel<<<unsigned((m * n + 127) / 128), 128, 0, st>>>(a, m, k, w, n, blk, out);
}

void launch_gemm_oracle(const float* a, int64_t m, int64_t k, const uint8_t* codes, Layout L,
                        int bits, int64_t n, int64_t g, int64_t gpr, const float* scales,
                        float* out, cudaStream_t st) {
    if (m * n == 0) return;
    gemm_oracle_kernel<<<unsigned((m * n + 127) / 128), 128, 0, st>>>(a, m, k, codes, L, bits, n,
                                                                      g, gpr, scales, out);
}

}  // namespace rtnq_b200
