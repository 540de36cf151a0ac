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
#include <cstdlib>

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

// The same arithmetic, parallel over groups instead of outputs, for the reference's own operand
// layout (kernel_interleaved 16 x tc, gemm.cpp:64-66): a warp owns one 16-row tile row-group and
// MT tokens; lane l computes the f32 block sums of groups l, l + 32 (k ascending, one lane per
// group, so every block sum is the reference's), parks them in shared memory, and then 16 * MT
// lanes fold them into the outputs in group order (acc += S * block).  Bit-identical to
// gemm_fused_exact_kernel; at k = 4096 one 8 / 16-byte load gives a k step of all 16 rows.
constexpr int kExactWarps = 4;
template <int BITS, int MT>
__global__ void __launch_bounds__(32 * kExactWarps) gemm_fused_exact_ki16_kernel(
    const float* __restrict__ a, int64_t m, int64_t k, const uint8_t* __restrict__ codes, int tc, int64_t n,
    int64_t g, int gpr, const float* __restrict__ scales, float* __restrict__ out) {
    extern __shared__ float sb[];  // [warp][group][16 rows][MT]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t jt = int64_t(blockIdx.x) * kExactWarps + warp;  // 16-row group
    const int64_t t0 = int64_t(blockIdx.y) * MT;
    if (jt * 16 >= n) return;
    float* wsb = sb + size_t(warp) * gpr * 16 * MT;
    const int64_t tpr = (k + tc - 1) / tc;
    const int64_t base = jt * tpr * 16 * tc;  // slot of (row jt * 16, k = 0); + k * 16 + r
    const float* arow[MT];
#pragma unroll
    for (int t = 0; t < MT; ++t) arow[t] = a + min(t0 + t, m - 1) * k;
    for (int q = lane; q < gpr; q += 32) {
        const int64_t k0 = q * g, k1 = min(k0 + g, k);
        float blk[16][MT];
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int t = 0; t < MT; ++t) blk[r][t] = 0.0f;
        int64_t kk = k0;
        // four k steps per round: 16-byte activation loads, codes of 4 steps at once (the
        // products still accumulate in k order)
        if ((k & 3) == 0 && (k0 & 3) == 0) {
            for (; kk + 4 <= k1; kk += 4) {
                float4 av4[MT];
#pragma unroll
                for (int t = 0; t < MT; ++t) av4[t] = __ldg(reinterpret_cast<const float4*>(arow[t] + kk));
                uint32_t cw[4][BITS == 4 ? 2 : 4];
#pragma unroll
                for (int st = 0; st < 4; ++st) {
                    if constexpr (BITS == 4) {
                        const uint2 w = *reinterpret_cast<const uint2*>(codes + ((base + (kk + st) * 16) >> 1));
                        cw[st][0] = w.x, cw[st][1] = w.y;
                    } else {
                        const uint4 w = *reinterpret_cast<const uint4*>(codes + base + (kk + st) * 16);
                        cw[st][0] = w.x, cw[st][1] = w.y;
                        if constexpr (BITS == 8) cw[st][2] = w.z, cw[st][3] = w.w;
                    }
                }
#pragma unroll
                for (int st = 0; st < 4; ++st) {
#pragma unroll
                    for (int r = 0; r < 16; ++r) {
                        const int c = BITS == 4 ? int((cw[st][r >> 3] >> (4 * (r & 7))) & 15u) - 8
                                                : int((cw[st][r >> 2] >> (8 * (r & 3))) & 255u) - 128;
                        const float cf = float(c);
#pragma unroll
                        for (int t = 0; t < MT; ++t) {
                            const float x = st == 0 ? av4[t].x : st == 1 ? av4[t].y : st == 2 ? av4[t].z : av4[t].w;
                            blk[r][t] = __fadd_rn(blk[r][t], __fmul_rn(x, cf));
                        }
                    }
                }
            }
        }
        for (; kk < k1; ++kk) {
            int c[16];
            if constexpr (BITS == 4) {
                const uint2 w = *reinterpret_cast<const uint2*>(codes + ((base + kk * 16) >> 1));
#pragma unroll
                for (int r = 0; r < 16; ++r) c[r] = int(((r < 8 ? w.x : w.y) >> (4 * (r & 7))) & 15u) - 8;
            } else {
                const uint4 w = *reinterpret_cast<const uint4*>(codes + base + kk * 16);
                const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int r = 0; r < 16; ++r) c[r] = int((ww[r >> 2] >> (8 * (r & 3))) & 255u) - 128;
            }
            float av[MT];
#pragma unroll
            for (int t = 0; t < MT; ++t) av[t] = __ldg(arow[t] + kk);
#pragma unroll
            for (int r = 0; r < 16; ++r)
#pragma unroll
                for (int t = 0; t < MT; ++t) blk[r][t] = __fadd_rn(blk[r][t], __fmul_rn(av[t], float(c[r])));
        }
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int t = 0; t < MT; ++t) wsb[(q * 16 + r) * MT + t] = blk[r][t];
    }
    __syncwarp();
    for (int o = lane; o < 16 * MT; o += 32) {  // output (row r, token t), groups in order
        const int r = o / MT, t = o % MT;
        const int64_t j = jt * 16 + r, ti = t0 + t;
        if (j >= n || ti >= m) continue;
        const float* srow = scales + j * gpr;
        float acc = 0.0f;
        for (int q = 0; q < gpr; ++q) acc = __fadd_rn(acc, __fmul_rn(srow[q], wsb[(q * 16 + r) * MT + t]));
        out[ti * n + j] = acc;
    }
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

template <int BITS, int MT>
static void launch_ki16(const float* a, int64_t m, int64_t k, const uint8_t* codes, int tc, int64_t n, int64_t g,
                        int gpr, const float* scales, float* out, cudaStream_t st) {
    const size_t smem = size_t(kExactWarps) * gpr * 16 * MT * sizeof(float);
    static bool configured = false;  // the largest request: 4 warps x 128 groups x 16 x MT floats
    if (!configured) {
        cudaFuncSetAttribute(gemm_fused_exact_ki16_kernel<BITS, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(kExactWarps * 128 * 16 * MT * sizeof(float)));
        configured = true;
    }
    const dim3 grid(unsigned((n + 16 * kExactWarps - 1) / (16 * kExactWarps)), unsigned((m + MT - 1) / MT));
    gemm_fused_exact_ki16_kernel<BITS, MT><<<grid, 32 * kExactWarps, smem, st>>>(a, m, k, codes, tc, n, g, gpr,
                                                                                scales, out);
}

void launch_gemm_fused_exact(const float* a, int64_t m, int64_t k, const uint8_t* codes,
                             Layout L, int bits, int64_t n, int64_t g, int64_t gpr,
                             const float* scales, float* out, cudaStream_t st) {
    if (m * n == 0) return;
    // the reference's kernel layout (16 x tc tiles), up to 128 groups per row, m < 2^16 chunks
    if (L.kind == RTNQ_KERNEL_INTERLEAVED && L.tr == 16 && gpr <= 128 && (m + 3) / 4 < 65536 &&
        !std::getenv("RTNQ_EXACT_SIMPLE")) {
        const int gp = int(gpr);
        if (m == 1) {
            bits == 4 ? launch_ki16<4, 1>(a, m, k, codes, L.tc, n, g, gp, scales, out, st)
                      : launch_ki16<8, 1>(a, m, k, codes, L.tc, n, g, gp, scales, out, st);
        } else if (m == 2) {
            bits == 4 ? launch_ki16<4, 2>(a, m, k, codes, L.tc, n, g, gp, scales, out, st)
                      : launch_ki16<8, 2>(a, m, k, codes, L.tc, n, g, gp, scales, out, st);
        } else {
            bits == 4 ? launch_ki16<4, 4>(a, m, k, codes, L.tc, n, g, gp, scales, out, st)
                      : launch_ki16<8, 4>(a, m, k, codes, L.tc, n, g, gp, scales, out, st);
        }
        return;
    }
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
