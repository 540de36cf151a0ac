// quant_fused.cu -- one-pass RTN quantize-and-pack (the hot quantize kernel).
//
// One CTA of 256 threads owns a 16-row x 128-column tile: it reads the weights
// once (128-bit loads), reduces group absmax with warp shuffles, computes the
// reference scale and codes (common.cuh), stages the codes in shared memory and
// writes every requested layout with coalesced 32/64-bit stores:
//   row-major packed (== QuantTensor::data, quant.cpp:139 / packing.cpp:6-32),
//   kernel_interleaved(16,4) (== reshuffle(q, kernel()).data, packing.cpp:75-92),
//   native sm100 operand order,
// plus f32 / f16 / native-f16 scales.  A 16 x 128 tile maps to exactly one
// contiguous 1 KiB (4-bit) / 2 KiB (8-bit) span of the 16x4 layout and to 2 / 4
// whole 512-byte native k-blocks, so no output byte is shared between CTAs.
// Domain: cols % 128 == 0 and g a power of two <= 128 (every BASELINE config
// except per-channel 8-bit, which takes the generic path in quant.cu).
#include <float.h>

#include "../common.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {

namespace {
constexpr int kTileR = 16, kTileC = 128, kThreads = 256;

template <int DT>
__device__ __forceinline__ void load8(const void* w, int64_t idx, float (&v)[8]) {
    if constexpr (DT == RTNQ_F32) {
        const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(w) + idx);
        const float4 x = __ldg(p), y = __ldg(p + 1);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
    } else {
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(
            static_cast<const uint16_t*>(w) + idx));
        const uint32_t u[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if constexpr (DT == RTNQ_BF16) {
                v[2 * i] = __uint_as_float(u[i] << 16);
                v[2 * i + 1] = __uint_as_float(u[i] & 0xFFFF0000u);
            } else {
                const __half2 h = *reinterpret_cast<const __half2*>(&u[i]);
                const float2 f = __half22float2(h);
                v[2 * i] = f.x;
                v[2 * i + 1] = f.y;
            }
        }
    }
}
}  // namespace

template <int DT, int BITS>
__global__ void __launch_bounds__(kThreads)
quant_fused_kernel(const void* __restrict__ w, int64_t rows, int64_t cols, int64_t g,
                   uint8_t* __restrict__ rm, uint8_t* __restrict__ k164,
                   uint8_t* __restrict__ nat, float* __restrict__ s32,
                   uint16_t* __restrict__ s16, uint16_t* __restrict__ s16n,
                   int32_t* __restrict__ err) {
    __shared__ int8_t sc[kTileR][kTileC];
    const int t = threadIdx.x;
    const int lr = t >> 4, lc = (t & 15) * 8;  // local row, first local column
    const int64_t strip = blockIdx.y, cb = blockIdx.x;
    const int64_t r = strip * kTileR + lr, c0 = cb * kTileC + lc;
    const int64_t gpr = cols / g;
    const bool live = r < rows;

    float v[8];
    if (live) load8<DT>(w, r * cols + c0, v);
    else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = 0.0f;
    }

    // ---- group absmax + finiteness (quant.cpp:50-57) ----
    float a[8];
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = fabsf(v[i]);
        bad |= !(a[i] <= FLT_MAX);
    }
    float gmax[8];  // absmax of the group holding element i
    if (g >= 8) {
        float m = a[0];
#pragma unroll
        for (int i = 1; i < 8; ++i) m = fmaxf(m, a[i]);
        const int lanes = int(g >> 3);  // 1..16 lanes share a group (same half-warp row)
        for (int o = 1; o < lanes; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
#pragma unroll
        for (int i = 0; i < 8; ++i) gmax[i] = m;
    } else {
        const int gi = int(g);
        for (int b = 0; b < 8; b += gi) {
            float m = a[b];
            for (int i = 1; i < gi; ++i) m = fmaxf(m, a[b + i]);
            for (int i = 0; i < gi; ++i) gmax[b + i] = m;
        }
    }
    if (__any_sync(0xffffffffu, bad && live) && (t & 31) == 0 && err) atomicOr(err, 1);

    // ---- scales + codes ----
    float sv[8];  // one f64 division per distinct group held by this thread
    if (g >= 8) {
        const float s = scale_from_absmax(gmax[0], BITS);
#pragma unroll
        for (int i = 0; i < 8; ++i) sv[i] = s;
    } else {
        for (int b = 0; b < 8; b += int(g)) {
            const float s = scale_from_absmax(gmax[b], BITS);
            for (int i = 0; i < int(g); ++i) sv[b + i] = s;
        }
    }
    int8_t code[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float s = sv[i];
        code[i] = live ? int8_t(quantize_one(v[i], s, BITS)) : int8_t(0);
        const int64_t c = c0 + i;
        if (live && (c % g) == 0) {  // first element of a group publishes its scale
            const int64_t j = c / g;
            if (s32) s32[r * gpr + j] = s;
            const uint16_t h = __half_as_ushort(__float2half_rn(s));
            if (s16) s16[r * gpr + j] = h;
            if (s16n) s16n[native_scale_index(rows, gpr, r, j)] = h;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) sc[lr][lc + i] = code[i];

    // ---- row-major packed, straight from registers ----
    if (rm && live) {
        if constexpr (BITS == 4) {
            uint32_t p = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) p |= uint32_t(code[i] + 8) << (4 * i);
            *reinterpret_cast<uint32_t*>(rm + ((r * cols + c0) >> 1)) = p;
        } else {
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                lo |= uint32_t(uint8_t(code[i] + 128)) << (8 * i);
                hi |= uint32_t(uint8_t(code[i + 4] + 128)) << (8 * i);
            }
            *reinterpret_cast<uint2*>(rm + r * cols + c0) = make_uint2(lo, hi);
        }
    }
    __syncthreads();

    // ---- kernel_interleaved(16,4): one contiguous span per tile ----
    if (k164) {
        const int64_t tpr = cols / 4;
        if constexpr (BITS == 4) {
            uint8_t* dst = k164 + (strip * tpr + cb * 32) * 32;  // 32 tiles x 32 B
            const int B = 4 * t;                                 // first byte of this thread
            const int tile = B >> 5, wb = B & 31, cc = tile * 4 + (wb >> 3);
            uint32_t p = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int rr = 2 * ((wb & 7) + i);
                p |= (uint32_t(sc[rr][cc] + 8) | (uint32_t(sc[rr + 1][cc] + 8) << 4)) << (8 * i);
            }
            *reinterpret_cast<uint32_t*>(dst + B) = p;
        } else {
            uint8_t* dst = k164 + (strip * tpr + cb * 32) * 64;  // 32 tiles x 64 B
            const int B = 8 * t;
            const int tile = B >> 6, slot0 = B & 63;
            const int cc = tile * 4 + (slot0 >> 4), rr0 = slot0 & 15;
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                lo |= uint32_t(uint8_t(sc[rr0 + i][cc] + 128)) << (8 * i);
                hi |= uint32_t(uint8_t(sc[rr0 + 4 + i][cc] + 128)) << (8 * i);
            }
            *reinterpret_cast<uint2*>(dst + B) = make_uint2(lo, hi);
        }
    }

    // ---- native: whole 512-byte k-blocks ----
    if (nat) {
        const int64_t ns = (rows + 15) / 16;
        if constexpr (BITS == 4) {
            const int q = t >> 7, o = 4 * (t & 127), lane = o >> 4, j = (o & 15) >> 2;
            const int gid = lane >> 2, tig = lane & 3;
            uint32_t p = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int rr = gid + 8 * ((e >> 1) & 1);
                const int cc = q * 64 + j * 16 + 2 * tig + 8 * (e >> 2) + (e & 1);
                p |= uint32_t(sc[rr][cc] + 8) << (4 * ((e & 1) * 4 + (e >> 1)));
            }
            const int64_t kb = cb * 2 + q;
            *reinterpret_cast<uint32_t*>(nat + native_chunk(ns, cols / 64, strip, kb) * 512 + o) = p;
        } else {
            const int q = t >> 6, o = 8 * (t & 63), lane = o >> 4, j = (o & 15) >> 3;
            const int gid = lane >> 2, tig = lane & 3;
            uint32_t w2[2] = {0, 0};
#pragma unroll
            for (int pb = 0; pb < 8; ++pb) {
                const int e = (pb >> 2) * 4 + (pb & 1) * 2 + ((pb >> 1) & 1);
                const int rr = gid + 8 * ((e >> 1) & 1);
                const int cc = q * 32 + j * 16 + 2 * tig + 8 * (e >> 2) + (e & 1);
                w2[pb >> 2] |= uint32_t(uint8_t(sc[rr][cc] + 128)) << (8 * (pb & 3));
            }
            const int64_t kb = cb * 4 + q;
            *reinterpret_cast<uint2*>(nat + native_chunk(ns, cols / 32, strip, kb) * 512 + o) =
                make_uint2(w2[0], w2[1]);
        }
    }
}

bool quant_fused_supported(int64_t rows, int64_t cols, int bits, int64_t g) {
    (void)bits;
    return rows > 0 && cols > 0 && cols % kTileC == 0 && g >= 1 && g <= kTileC &&
           (g & (g - 1)) == 0 && (rows + 15) / 16 <= 65535;
}

void launch_quant_fused(const void* w, int dtype, int64_t rows, int64_t cols, int bits,
                        int64_t g, uint8_t* rm, uint8_t* k164, uint8_t* nat, float* s32,
                        uint16_t* s16, uint16_t* s16n, int32_t* err, cudaStream_t st) {
    const dim3 grid(unsigned(cols / kTileC), unsigned((rows + 15) / 16));
#define RTNQ_QF(DT, B) \
    quant_fused_kernel<DT, B><<<grid, kThreads, 0, st>>>(w, rows, cols, g, rm, k164, nat, s32, s16, s16n, err)
    if (bits == 4) {
        if (dtype == RTNQ_F32) RTNQ_QF(RTNQ_F32, 4);
        else if (dtype == RTNQ_F16) RTNQ_QF(RTNQ_F16, 4);
        else RTNQ_QF(RTNQ_BF16, 4);
    } else {
        if (dtype == RTNQ_F32) RTNQ_QF(RTNQ_F32, 8);
        else if (dtype == RTNQ_F16) RTNQ_QF(RTNQ_F16, 8);
        else RTNQ_QF(RTNQ_BF16, 8);
    }
#undef RTNQ_QF
}

}  // namespace rtnq_b200
