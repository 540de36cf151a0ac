// int8_mma.cuh -- shared pieces of the tcgen05 kind::i8 weight-only GEMMs (wgemm_i8.cu: W8
// per-channel, wgemm_i4.cu: W4 group-128): PTX wrappers (mbarrier, TMA, tcgen05), the
// work cursor, and the activation-planes kernel that turns bf16/f16 activations into three
// exact int8 planes.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "../common.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {
namespace imma {

constexpr int kRows = 128;  // UMMA M = one row-block

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
// The suspend-time hint keeps a waiting warp parked until the phase completes (or ~1 ms)
// instead of re-polling every few hundred cycles: spinning warps take issue slots from the
// working warps of the same SM sub-partition (ncu: ~17% of the W4 kernel's instructions).
#ifndef RTNQ_MBAR_HINT_NS
#define RTNQ_MBAR_HINT_NS 1000000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n"
        "@!P bra W_%=;\n}\n" ::"r"(su32(b)),
        "r"(ph), "n"(RTNQ_MBAR_HINT_NS)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(su32(b))
        : "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, int c0, int c1, int c2,
                                      uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3, %4}], [%5];" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(b))
        : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void commit(uint64_t* b) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b))
        : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void ld8(uint32_t taddr, uint32_t* d) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7])
                 : "r"(taddr)
                 : "memory");
}
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t* d) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
          "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]),
          "=r"(d[14]), "=r"(d[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void store_out(void* out, int dt, int64_t i, float v) {
    if (dt == RTNQ_F32) static_cast<float*>(out)[i] = v;
    else if (dt == RTNQ_BF16) static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
    else static_cast<__half*>(out)[i] = __float2half_rn(v);
}
// K-major, 128-byte swizzle: 8-row atoms of 128 B (SBO = 1024), layout type 2.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}
// The unit sequence of a CTA: runs of <= 2 k-blocks inside one row-block and one 128-code
// block, tracked incrementally (no division on the issue path).
template <int SPAN>  // k-blocks per stage (2 per 16 KiB tile)
struct Cursor {
    int u, u1, b, kb, KBLK;
    __device__ Cursor(int u0, int u1_, int KBLK_) : u(u0), u1(u1_), KBLK(KBLK_) {
        b = u0 / KBLK_;
        kb = u0 - b * KBLK_;
    }
    __device__ bool more() const { return u < u1; }
    __device__ int chunk() const {
        const int left_seg = KBLK - kb, left = u1 - u, cap = SPAN - (kb & (SPAN - 1));
        const int n = left_seg < left ? left_seg : left;
        return n < cap ? n : cap;
    }
    __device__ bool seg_end(int n) const { return kb + n == KBLK || u + n == u1; }
    __device__ void advance(int n) {
        u += n;
        kb += n;
        if (kb == KBLK) kb = 0, ++b;
    }
};
__device__ __forceinline__ void mma_i8_elect(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc,
                                             uint32_t acc) {
    asm volatile(
        "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}
// Warp-uniform MMA issue: the whole (converged) warp executes the asm, one elected lane issues
// every MMA of the block.  Measured (scratch/tmem_bw.cu): ~13 cycles per M128 x N16 x K32 MMA,
// and N = 48 at the tensor-core floor (24 cycles), against ~100 cycles per MMA when one lane
// inside a divergent branch issues them (the compiler wraps each tcgen05.mma in an elect loop
// with a register -> uniform-register move).  The same elected lane must issue the commits.
//
// 4 k-steps of K = 32 into one accumulator: A from TMEM at a, a + 8, a + 16, a + 24 (32-bit
// columns of 4 s8), B descriptors bd, bd + 2, bd + 4, bd + 6 (32-byte steps); acc = 0
// overwrites D with the first product.
__device__ __forceinline__ void mma4_i8_ts_warp(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred e, p0, p1;\n.reg .b32 a1, a2, a3;\n.reg .b64 b1, b2, b3;\n"
        "setp.ne.b32 p0, %4, 0;\nsetp.eq.b32 p1, 0, 0;\n"
        "add.u32 a1, %1, 8;\nadd.u32 a2, %1, 16;\nadd.u32 a3, %1, 24;\n"
        "add.u64 b1, %2, 2;\nadd.u64 b2, %2, 4;\nadd.u64 b3, %2, 6;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p0;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %3, p1;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a2], b2, %3, p1;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a3], b3, %3, p1;\n}\n" ::"r"(d),
        "r"(a), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}
// 2 k-steps of K = 32, A and B from shared memory (descriptors ad, ad + 2 and bd, bd + 2).
__device__ __forceinline__ void mma2_i8_ss_warp(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred e, p0, p1;\n.reg .b64 a1, b1;\n"
        "setp.ne.b32 p0, %4, 0;\nsetp.eq.b32 p1, 0, 0;\n"
        "add.u64 a1, %1, 2;\nadd.u64 b1, %2, 2;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p0;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, %3, p1;\n}\n" ::"r"(d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ bool elect_leader() {
    uint32_t e;
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}\n" : "=r"(e));
    return e != 0;
}
__device__ __forceinline__ void commit_elect(uint64_t* b) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(b))
        : "memory");
}
__device__ __forceinline__ void elect_arrive(uint64_t* b) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" ::"r"(
            su32(b))
        : "memory");
}
__device__ __forceinline__ void elect_bulk(void* dst, const void* src, uint64_t* b, uint32_t bytes) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n"
        "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(
            su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(b))
        : "memory");
}
__device__ __forceinline__ void elect_prefetch(const void* src, uint32_t bytes) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e cp.async.bulk.prefetch.L2.global [%0], %1;\n}\n" ::"l"(src), "r"(bytes)
        : "memory");
}
__device__ __forceinline__ void elect_tma3d(void* dst, const CUtensorMap* m, int c0, int c1, int c2,
                                            uint64_t* b, uint32_t bytes) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%6], %5;\n"
        "@e cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3, %4}], [%6];\n}\n" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(bytes), "r"(su32(b))
        : "memory");
}

// expect_tx once for all boxes of a stage, then the box loads (no further arrivals)
__device__ __forceinline__ void elect_expect(uint64_t* b, uint32_t bytes) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(su32(b)), "r"(bytes)
        : "memory");
}
__device__ __forceinline__ void elect_tma3d_tx(void* dst, const CUtensorMap* m, int c0, int c1, int c2,
                                               uint64_t* b) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3, %4}], [%5];\n}\n" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(b))
        : "memory");
}

__device__ __forceinline__ int cta_of(int64_t u, int64_t U, int G) {
    return int(((u + 1) * G - 1) / U);
}

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---- activation planes ------------------------------------------------------------------
// One CTA per token (PDL secondary of whatever produced the activations):
//   s = exponent(max|a|) - 6 so |a| / 2^s < 64; three exact int8 planes.
// 16-byte loads of 8 activations; up to kVPT vectors per thread stay in registers between
// the max and the split (one pass over memory for K <= 512 * 8 * kVPT), longer rows reload.
#ifndef RTNQ_PLANES_SLICE_V
#define RTNQ_PLANES_SLICE_V 512
#endif
constexpr int kPlaneThreads = 256, kSliceV = RTNQ_PLANES_SLICE_V;  // 16-byte vectors per CTA slice

// While the activations are split, pull the head of every GEMM CTA's weight range into L2
// (cp.async.bulk.prefetch.L2): the GEMM that follows then finds its first stages on chip
// instead of paying a DRAM round trip after launch.  The unit -> byte map is the layout's:
// NATIVE_I8 (kind 8): a 16 KiB tile per 2 units, NATIVE_I4 (kind 4): an 8 KiB tile per unit.
struct WeightPrefetch {
    const uint8_t* base = nullptr;  // nullptr: none
    int64_t bytes = 0;              // the whole codes array (clamp)
    int kind = 0, U = 0, G = 0, csize = 1, KBLK = 0;
    uint32_t head = 0;              // bytes per CTA
};
__device__ __forceinline__ void prefetch_weight_heads(const WeightPrefetch& w) {
    if (!w.base) return;
    const int nthr = blockDim.x * gridDim.x * gridDim.y;
    const int gt = (blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
    for (int c = gt; c < w.G; c += nthr) {
        int u0;
        if (w.csize > 1) {
            const int b = c / w.csize, r = c % w.csize;
            u0 = b * w.KBLK + r * w.KBLK / w.csize;
        } else {
            u0 = int(int64_t(c) * w.U / w.G);
        }
        const int64_t off = w.kind == 8
            ? (int64_t(u0 / w.KBLK) * ((w.KBLK + 1) >> 1) + ((u0 % w.KBLK) >> 1)) * 16384
            : int64_t(u0) * 8192;
        if (off >= w.bytes) continue;
        const uint32_t n = uint32_t(w.bytes - off < int64_t(w.head) ? w.bytes - off : int64_t(w.head));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(w.base + off), "r"(n & ~15u) : "memory");
    }
}
// grid (M, ceil(K / 8 / kSliceV)): every CTA of a token re-reduces the token's max over the
// whole row (L2-resident, loads all in flight), then splits its own slice into planes.
template <int AT, bool VEC>
__global__ void __launch_bounds__(kPlaneThreads) act_planes_kernel(const void* __restrict__ a, int K, int M,
                                                                   int8_t* __restrict__ planes,
                                                                   int32_t* __restrict__ texp, unsigned long long* stamps,
                                                                   const WeightPrefetch pf, int early,
                                                                   int32_t* __restrict__ err) {
    __shared__ float wmax[kPlaneThreads / 32];
    const bool first = blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0;
    if (stamps && first) stamps[0] = gtime();
    prefetch_weight_heads(pf);  // weights are read-only: no need to wait for the predecessor
    // early: the GEMM that consumes these planes may launch before the predecessor finishes, so
    // its weight stream overlaps the predecessor's tail.  Safe: everything it writes depends on
    // the planes, which it reads only after its own griddepcontrol.wait (this grid complete).
    if (early) asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (!early) asm volatile("griddepcontrol.launch_dependents;");
    if (stamps && first) stamps[1] = gtime();
    const int t = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint16_t* rowp = static_cast<const uint16_t*>(a) + int64_t(t) * K;
    const int nv = K / 8, v0 = blockIdx.y * kSliceV;
    auto load4 = [&](int v) -> uint4 {
        if constexpr (VEC) return __ldg(reinterpret_cast<const uint4*>(rowp) + v);
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = uint32_t(rowp[v * 8 + 2 * i]) | (uint32_t(rowp[v * 8 + 2 * i + 1]) << 16);
        return make_uint4(w[0], w[1], w[2], w[3]);
    };
    auto cvt = [](uint32_t h) -> float {
        if constexpr (AT == RTNQ_BF16) return __uint_as_float(h << 16);
        else return __half2float(__ushort_as_half(static_cast<unsigned short>(h)));
    };
    // non-finite inputs (InvalidInputError in the reference, gemm.cpp:13-19): an all-ones
    // exponent field in either half of a word, folded into the max pass
    constexpr uint32_t kExpMask = AT == RTNQ_BF16 ? 0x7F807F80u : 0x7C007C00u;
    uint32_t nonfinite = 0;
    auto vmax = [&](const uint4& q, float m) {
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            m = fmaxf(m, fmaxf(fabsf(cvt(w[i] & 0xffffu)), fabsf(cvt(w[i] >> 16))));
            const uint32_t e = w[i] & kExpMask;
            nonfinite |= ((e & 0xffffu) == (kExpMask & 0xffffu)) | ((e >> 16) == (kExpMask >> 16));
        }
        return m;
    };
    // this CTA's slice stays in registers; the rest of the row is only max-reduced
    uint4 keep[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int v = v0 + tid + j * kPlaneThreads;
        keep[j] = v < nv ? load4(v) : make_uint4(0, 0, 0, 0);
    }
    float mx = fmaxf(vmax(keep[0], 0.0f), vmax(keep[1], 0.0f));
    for (int v = tid; v < nv; v += 4 * kPlaneThreads) {
        uint4 q[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int vv = v + j * kPlaneThreads;
            q[j] = (vv < nv && (vv < v0 || vv >= v0 + kSliceV)) ? load4(vv) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) mx = vmax(q[j], mx);
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) wmax[warp] = mx;
    if (err && blockIdx.y == 0 && __any_sync(0xffffffffu, nonfinite) && lane == 0) atomicOr(err, 1);
    __syncthreads();
    float amax = 0.0f;
#pragma unroll
    for (int i = 0; i < kPlaneThreads / 32; ++i) amax = fmaxf(amax, wmax[i]);
    int e = 0;
    if (amax > 0.0f) frexpf(amax, &e);  // amax in [2^(e-1), 2^e)
    const int s = max(e - 6, -126);      // |a| / 2^s < 64; 2^s stays a normal float
    if (tid == 0 && blockIdx.y == 0) texp[t] = s;
    const float inv = __int_as_float((127 - s) << 23);  // 2^-s, exact scaling
    // round to nearest even and the integer bits in one add: for |y| < 2^22,
    // bits(y + 1.5 * 2^23) - bits(1.5 * 2^23) = rint(y)
    auto rnd = [](float y, float& r) {
        const float b = y + 12582912.0f;
        r = b - 12582912.0f;
        return uint32_t(__float_as_int(b) - 0x4B400000);
    };
    auto split = [&](const uint4& q, int v) {
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        uint32_t pk[3][2] = {{0, 0}, {0, 0}, {0, 0}};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float y = cvt(i & 1 ? w[i >> 1] >> 16 : w[i >> 1] & 0xffffu) * inv;  // exact
            float r0, r1, r2;
            const uint32_t q0 = rnd(y, r0);
            const float y1 = (y - r0) * 128.0f;  // exact
            const uint32_t q1 = rnd(y1, r1);
            const uint32_t q2 = rnd((y1 - r1) * 128.0f, r2);
            pk[0][i >> 2] |= (q0 & 0xffu) << (8 * (i & 3));
            pk[1][i >> 2] |= (q1 & 0xffu) << (8 * (i & 3));
            pk[2][i >> 2] |= (q2 & 0xffu) << (8 * (i & 3));
        }
#pragma unroll
        for (int pl = 0; pl < 3; ++pl)
            *reinterpret_cast<uint2*>(planes + (int64_t(pl) * M + t) * K + int64_t(v) * 8) =
                make_uint2(pk[pl][0], pk[pl][1]);
    };
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int v = v0 + tid + j * kPlaneThreads;
        if (v < nv) split(keep[j], v);
    }
    if (stamps && first) stamps[2] = gtime();
}

// The whole bf16 row `rowp` (K values, K % 8 == 0, 16-byte aligned, written by this CTA before
// a __syncthreads) -> planes of token t and its exponent: the planes kernel's arithmetic for
// the kernels that produce activations (add+RMSNorm, SiLU*up) and emit the planes themselves.
__device__ __forceinline__ void row_to_planes(const uint16_t* __restrict__ rowp, int K, int t, int M,
                                              int8_t* __restrict__ planes, int32_t* __restrict__ texp) {
    __shared__ float wmax_r[32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
    const int nv = K / 8;
    auto cvt = [](uint32_t h) -> float { return __uint_as_float(h << 16); };
    float mx = 0.0f;
    for (int v = tid; v < nv; v += blockDim.x) {
        const uint4 q = *reinterpret_cast<const uint4*>(rowp + v * 8);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) mx = fmaxf(mx, fmaxf(fabsf(cvt(w[i] & 0xffffu)), fabsf(cvt(w[i] >> 16))));
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) wmax_r[warp] = mx;
    __syncthreads();
    float amax = 0.0f;
    for (int i = 0; i < nw; ++i) amax = fmaxf(amax, wmax_r[i]);
    int e = 0;
    if (amax > 0.0f) frexpf(amax, &e);
    const int s = max(e - 6, -126);
    if (tid == 0) texp[t] = s;
    const float inv = __int_as_float((127 - s) << 23);
    for (int v = tid; v < nv; v += blockDim.x) {
        const uint4 q = *reinterpret_cast<const uint4*>(rowp + v * 8);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        uint32_t pk[3][2] = {{0, 0}, {0, 0}, {0, 0}};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float y = cvt(i & 1 ? w[i >> 1] >> 16 : w[i >> 1] & 0xffffu) * inv;
            const float b0 = y + 12582912.0f, r0 = b0 - 12582912.0f;
            const float y1 = (y - r0) * 128.0f;
            const float b1 = y1 + 12582912.0f, r1 = b1 - 12582912.0f;
            const float b2 = (y1 - r1) * 128.0f + 12582912.0f;
            pk[0][i >> 2] |= (uint32_t(__float_as_int(b0) - 0x4B400000) & 0xffu) << (8 * (i & 3));
            pk[1][i >> 2] |= (uint32_t(__float_as_int(b1) - 0x4B400000) & 0xffu) << (8 * (i & 3));
            pk[2][i >> 2] |= (uint32_t(__float_as_int(b2) - 0x4B400000) & 0xffu) << (8 * (i & 3));
        }
#pragma unroll
        for (int pl = 0; pl < 3; ++pl)
            *reinterpret_cast<uint2*>(planes + (int64_t(pl) * M + t) * K + int64_t(v) * 8) =
                make_uint2(pk[pl][0], pk[pl][1]);
    }
}

// ---- tensor-parallel partial sums over peer memory ------------------------------
// Every rank owns one symmetric buffer (same layout, opened by every peer through CUDA IPC):
//   header (256 B): int epoch (local), int flags[8] (flags[q]: last round rank q delivered here),
//                   int done (producer CTAs finished), int consumed (consumer CTAs done)
//   slots: [2 parities][8 ranks][cap] bf16 -- rank q's partial of round e lands in slot [e & 1][q]
// A row-split linear of round e = epoch + 1 writes its output rows straight into its slot of
// EVERY rank's buffer (P2P stores over NVLink; its own buffer too), then its last CTA raises
// flags[rank] = e on every rank (release, system scope).  The consumer (add+RMSNorm, or a
// reduce kernel) waits for all flags >= e, sums the slots in rank order -- the same sum on every
// rank -- and bumps its local epoch.  Two parities: a rank writes round e + 1 only after its own
// consumer of round e, which waited for everyone's round e, so no slot is overwritten while read.
using rtnq_b200::kPeerHeader;
using rtnq_b200::kPeerMax;
using rtnq_b200::PeerOut;
__device__ __forceinline__ int* peer_epoch(char* b) { return reinterpret_cast<int*>(b); }
__device__ __forceinline__ int* peer_flags(char* b) { return reinterpret_cast<int*>(b) + 1; }
__device__ __forceinline__ int* peer_done(char* b) { return reinterpret_cast<int*>(b) + 1 + kPeerMax; }
__device__ __forceinline__ int* peer_consumed(char* b) { return reinterpret_cast<int*>(b) + 2 + kPeerMax; }
__device__ __forceinline__ __nv_bfloat16* peer_slot(char* b, int64_t cap, int parity, int q) {
    return reinterpret_cast<__nv_bfloat16*>(b + kPeerHeader) + (int64_t(parity) * kPeerMax + q) * cap;
}
// the round a producer writes: the local epoch + 1 (its consumer of the previous round bumped
// it).  Read only after the caller's dependency on the previous grid is resolved (the GEMM
// epilogue reads it after its griddepcontrol.wait / planes barrier; a griddepcontrol.wait placed
// here, even on a branch never taken, measured +2.3 us per W8 launch)
// (bufs is a kernel parameter: indexed with compile-time indices only -- a runtime index takes
// the parameter's address, which measured +2.5 us per launch of the W8 kernel even when the
// peer path is never taken)
__device__ __forceinline__ char* peer_buf(const PeerOut& po, int q) {
    char* b = nullptr;
#pragma unroll
    for (int i = 0; i < kPeerMax; ++i)
        if (i == q) b = po.bufs[i];
    return b;
}
__device__ __forceinline__ int peer_round(const PeerOut& po) {
    return *reinterpret_cast<volatile int*>(peer_epoch(peer_buf(po, po.rank))) + 1;
}
// element i of this rank's partial -> every rank's slot [e & 1][rank]
__device__ __forceinline__ void peer_store(const PeerOut& po, int e, int64_t i, float v) {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
#pragma unroll
    for (int q = 0; q < kPeerMax; ++q)
        if (q < po.world) peer_slot(po.bufs[q], po.cap, e & 1, po.rank)[i] = h;
}
// kernel end, thread 0 of each CTA after a CTA-wide barrier: the last of G CTAs flags round e
// on every rank (the CTA's stores were ordered before the barrier; the fence makes them visible
// system-wide before the counter, the flags after it)
__device__ __forceinline__ void peer_complete(const PeerOut& po, int e, int G) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    char* own = peer_buf(po, po.rank);
    if (atomicAdd(peer_done(own), 1) == G - 1) {
        *peer_done(own) = 0;
        asm volatile("fence.acq_rel.sys;" ::: "memory");
#pragma unroll
        for (int q = 0; q < kPeerMax; ++q)
            if (q < po.world)
                asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(peer_flags(po.bufs[q]) + po.rank), "r"(e)
                             : "memory");
    }
}
// 16 bytes of a slot (L2, not L1: the same slot address was read two rounds ago)
__device__ __forceinline__ uint4 peer_ld16(const __nv_bfloat16* p) { return __ldcg(reinterpret_cast<const uint4*>(p)); }
// consumer: wait until every rank delivered round e into this rank's buffer `b`
__device__ __forceinline__ void peer_wait(char* b, int world, int e) {
    for (int q = 0; q < world; ++q) {
        int got;
        for (;;) {
            asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(got) : "l"(peer_flags(b) + q) : "memory");
            if (got >= e) break;
            __nanosleep(64);
        }
    }
}
// consumer CTA done reading round e: the last of G bumps the local epoch (the next producer of
// this rank runs after this grid, stream-ordered)
__device__ __forceinline__ void peer_consumed_by(char* b, int G) {
    if (atomicAdd(peer_consumed(b), 1) == G - 1) {
        *peer_consumed(b) = 0;
        atomicAdd(peer_epoch(b), 1);
    }
}

// ---- activation planes computed inside the GEMM (no separate planes kernel) -----------------
// A stand-alone planes kernel costs each int8 linear ~5 us at batch 16 in a back-to-back chain
// (launch + two grid dependencies) for ~1 us of work.  Instead, the GEMM CTAs compute the
// planes of the launch's tokens themselves (CTA c: tokens c, c + G, ...) with their epilogue /
// expansion warps, which are idle until the first weights land, and publish them through a
// self-resetting workspace counter; one warp per CTA acquires it before the first planes TMA.
// fewer tokens: the stand-alone planes kernel (W4 gate_up at batch 8 / 9 / 10: 17.1 vs 19.0 us;
// batch 12 / 16: 21.8 vs 23.7 us in the GEMM; env RTNQ_OWN_PLANES_MIN_M overrides for W4)
constexpr int kOwnPlanesMinM = 11;
struct OwnPlanes {
    const void* a = nullptr;  // activations [Mtot][K], bf16 / f16; nullptr: planes precomputed
    int a_dtype = 0;
    int* done = nullptr;      // tokens published by this launch (workspace, starts at 0)
    int* consumed = nullptr;  // CTAs that have acquired them; the last one resets both
    int32_t* err = nullptr;   // |= 1 on a non-finite activation (InvalidInputError)
};

// One token row -> its planes and exponent (act_planes_kernel's arithmetic), by `nthr` threads
// (tid in [0, nthr)) synchronized with the named barrier `bar`; `red` is nthr / 32 floats of smem.
template <int AT>
__device__ __forceinline__ void token_planes(const uint16_t* __restrict__ rowp, int K, int t, int M,
                                             int8_t* __restrict__ planes, int32_t* __restrict__ texp,
                                             int32_t* err, int tid, int nthr, int bar, float* red,
                                             long long* dtl = nullptr, long long dt0 = 0, int sv0 = 0,
                                             int sv1 = -1) {
    if (dtl && tid == 0) dtl[0] = clock64() - dt0;
    auto cvt = [](uint32_t h) -> float {
        if constexpr (AT == RTNQ_BF16) return __uint_as_float(h << 16);
        else return __half2float(__ushort_as_half(static_cast<unsigned short>(h)));
    };
    constexpr uint32_t kExpMask = AT == RTNQ_BF16 ? 0x7F807F80u : 0x7C007C00u;
    const int nv = K / 8;
    // the first kHold vectors of this thread stay in registers between the two passes (K <= 8 *
    // kHold * nthr: one load of the row); longer rows reload the rest.  Few: these registers count
    // against the whole GEMM kernel that runs this producer in its epilogue / expansion warps
#ifndef RTNQ_PLANES_HOLD
#define RTNQ_PLANES_HOLD 2
#endif
    constexpr int kHold = RTNQ_PLANES_HOLD;
    uint4 held[kHold > 0 ? kHold : 1];
#pragma unroll
    for (int h = 0; h < kHold; ++h) {
        const int v = tid + h * nthr;
        if (v < nv) held[h] = __ldcg(reinterpret_cast<const uint4*>(rowp) + v);
    }
    float mx = 0.0f;
    uint32_t nonfinite = 0;
    auto scan = [&](const uint4& q) {
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            mx = fmaxf(mx, fmaxf(fabsf(cvt(w[i] & 0xffffu)), fabsf(cvt(w[i] >> 16))));
            const uint32_t e = w[i] & kExpMask;
            nonfinite |= ((e & 0xffffu) == (kExpMask & 0xffffu)) | ((e >> 16) == (kExpMask >> 16));
        }
    };
#pragma unroll
    for (int h = 0; h < kHold; ++h)
        if (tid + h * nthr < nv) scan(held[h]);
    if (dtl && tid == 0) dtl[1] = clock64() - dt0;
    for (int v = tid + kHold * nthr; v < nv; v += nthr) scan(__ldcg(reinterpret_cast<const uint4*>(rowp) + v));
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (err && __any_sync(0xffffffffu, nonfinite) && (tid & 31) == 0) atomicOr(err, 1);
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nthr) : "memory");
    float amax = 0.0f;
    for (int i = 0; i < nthr / 32; ++i) amax = fmaxf(amax, red[i]);
    int e = 0;
    if (amax > 0.0f) frexpf(amax, &e);
    const int s = max(e - 6, -126);
    if (tid == 0 && sv0 == 0) texp[t] = s;
    const float inv = __int_as_float((127 - s) << 23);
    if (dtl && tid == 0) dtl[2] = clock64() - dt0;
    auto split = [&](const uint4& q, int v) {
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        uint32_t pk[3][2] = {{0, 0}, {0, 0}, {0, 0}};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float y = cvt(i & 1 ? w[i >> 1] >> 16 : w[i >> 1] & 0xffffu) * inv;
            const float b0 = y + 12582912.0f, r0 = b0 - 12582912.0f;
            const float y1 = (y - r0) * 128.0f;
            const float b1 = y1 + 12582912.0f, r1 = b1 - 12582912.0f;
            const float b2 = (y1 - r1) * 128.0f + 12582912.0f;
            pk[0][i >> 2] |= (uint32_t(__float_as_int(b0) - 0x4B400000) & 0xffu) << (8 * (i & 3));
            pk[1][i >> 2] |= (uint32_t(__float_as_int(b1) - 0x4B400000) & 0xffu) << (8 * (i & 3));
            pk[2][i >> 2] |= (uint32_t(__float_as_int(b2) - 0x4B400000) & 0xffu) << (8 * (i & 3));
        }
#pragma unroll
        for (int pl = 0; pl < 3; ++pl)
            *reinterpret_cast<uint2*>(planes + (int64_t(pl) * M + t) * K + int64_t(v) * 8) =
                make_uint2(pk[pl][0], pk[pl][1]);
    };
    if (sv0 == 0 && (sv1 < 0 || sv1 >= nv)) {  // the whole row
#pragma unroll
        for (int h = 0; h < kHold; ++h)
            if (tid + h * nthr < nv) split(held[h], tid + h * nthr);
        for (int v = tid + kHold * nthr; v < nv; v += nthr) split(__ldcg(reinterpret_cast<const uint4*>(rowp) + v), v);
    } else {  // this CTA's slice [sv0, sv1) of the row's vectors (the exponent needs the whole row)
        for (int v = sv0 + tid; v < sv1; v += nthr) split(__ldcg(reinterpret_cast<const uint4*>(rowp) + v), v);
    }
    if (dtl && tid == 0) dtl[3] = clock64() - dt0;
    // every thread's planes stores are done before the caller publishes the token
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nthr) : "memory");
    if (dtl && tid == 0) dtl[4] = clock64() - dt0;
}

// Units of the launch's planes work: a token row is cut into S slices so that more of the G CTAs
// take part (each slice CTA reduces the whole row's max -- L2-resident -- and splits only its
// slice), with at least RTNQ_PLANES_MIN_SLICE_V 8-element vectors per slice: W4 down (K = 14336)
// at batch 16 / 32 / 64 gets 1.4 / 1.1 / 0.6 us faster, K = 4096 rows stay whole (r2_w4_limiter.md §9).
#ifndef RTNQ_PLANES_MIN_SLICE_V
#define RTNQ_PLANES_MIN_SLICE_V 256
#endif
__device__ __forceinline__ int own_planes_slices(int M, int G, int K) {
    int S = G / (M > 0 ? M : 1);
    S = S < 1 ? 1 : S;
    const int cap = (K / 8 + RTNQ_PLANES_MIN_SLICE_V - 1) / RTNQ_PLANES_MIN_SLICE_V;
    return S > cap ? cap : S;
}

// Producers: CTA c of G computes units u = c, c + G, ... < M * S (token u % M, slice u / M),
// after the activations' producer grid has completed (griddepcontrol.wait), and publishes each.
__device__ __forceinline__ void own_planes_produce(const OwnPlanes& op, int K, int m0, int M, int Mtot, int c,
                                                   int G, int8_t* planes, int32_t* texp, int tid, int nthr,
                                                   int bar, float* red, long long* dtl = nullptr,
                                                   long long dt0 = 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int S = own_planes_slices(M, G, K), nv = K / 8;
    for (int u = c; u < M * S; u += G) {
        const int t = u % M, sl = u / M;
        const int sv0 = int(int64_t(sl) * nv / S), sv1 = S == 1 ? -1 : int(int64_t(sl + 1) * nv / S);
        const uint16_t* rowp = static_cast<const uint16_t*>(op.a) + int64_t(m0 + t) * K;
        if (op.a_dtype == RTNQ_BF16)
            token_planes<RTNQ_BF16>(rowp, K, m0 + t, Mtot, planes, texp, op.err, tid, nthr, bar, red, dtl, dt0, sv0,
                                    sv1);
        else
            token_planes<RTNQ_F16>(rowp, K, m0 + t, Mtot, planes, texp, op.err, tid, nthr, bar, red, nullptr, 0, sv0,
                                   sv1);
        if (tid == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");  // the consumers read them by TMA
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(op.done) : "memory");
            if (dtl) dtl[5] = clock64() - dt0;
        }
    }
}

// Consumer (one whole warp per CTA): returns once all M tokens of this launch are published.  The
// last of the G CTAs to get here resets both counters; the next launch on this workspace only
// touches them after its own griddepcontrol.wait, i.e. after this grid has completed.
__device__ __forceinline__ void own_planes_acquire(const OwnPlanes& op, int M, int G, int K) {
    const int units = M * own_planes_slices(M, G, K);
    // the previous launch on this workspace must be complete before its counters are read: with
    // PDL (and free SMs) this grid's CTAs can start while it still runs
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if ((threadIdx.x & 31) == 0) {
        int got;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(got) : "l"(op.done) : "memory");
            if (got >= units) break;
            __nanosleep(32);
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (atomicAdd(op.consumed, 1) == G - 1) {
            atomicExch(op.done, 0);
            atomicExch(op.consumed, 0);
        }
    }
    __syncwarp();
}

template <int AT, bool VEC>
inline cudaError_t launch_planes(const void* a, int K, int M, int8_t* planes, int32_t* texp, unsigned long long* stamps,
                                 const WeightPrefetch& pf, int32_t* err,
                                 cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(M), unsigned((K / 8 + kSliceV - 1) / kSliceV));
    cfg.blockDim = dim3(kPlaneThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    static const int early = [] {
        const char* e = std::getenv("RTNQ_PDL_EARLY");
        return e ? std::atoi(e) : 1;
    }();
    return cudaLaunchKernelEx(&cfg, act_planes_kernel<AT, VEC>, a, K, M, planes, texp, stamps, pf, early, err);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);
inline EncodeFn encoder() {
    static EncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<EncodeFn>(f);
    }();
    return fn;
}

inline int sms() {
    static int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

}  // namespace imma
}  // namespace rtnq_b200
