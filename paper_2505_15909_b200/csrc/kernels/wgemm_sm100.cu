// wgemm_sm100.cu -- W4A16 / W8A16 weight-only GEMM for decode batches (m <= 64).
//
// out[m][n] = sum_k a[m][k] * code[n][k] * S[n][k/g]   (gemm.hpp:18-27)
//
// Design:
//  * Weights are the M operand of mma.m16n8k16 (16 output channels per tile),
//    tokens the N operand, so a batch of 1..8 tokens costs one n8 tile.
//  * Codes are stored in the native layout (common.cuh): for a CTA row-block of
//    256 channels x one k-block (64 4-bit / 32 8-bit codes) the 8 KiB of codes are
//    contiguous, so ONE cp.async.bulk (TMA, UBLKCP) moves each pipeline stage;
//    group scales (native order) and the activation rows ride on the same
//    mbarrier.  A dedicated producer warp keeps STAGES stages in flight.
//  * Each lane's 16-byte slice of a stage is its own A fragments: one LDS.128,
//    then LOP3/PRMT magic-number dequantization to bf16x2/f16x2 codes (exact
//    integers), mma into a per-group f32 block accumulator, and one FFMA per
//    element per group: acc += S * block -- the reference's accumulation
//    structure (gemm.cpp:69-87), with the scale applied in f32 (exact codes, no
//    f16 code*scale rounding).
//  * Stream-K: the (row-block, k-block) units are split evenly over the grid;
//    row-blocks shared by several CTAs are combined by the last CTA to arrive,
//    always summing the partials in CTA order (deterministic, no float atomics).
//  * PDL: weight prefetch for the first STAGES stages is issued before
//    griddepcontrol.wait; only the activation copies wait for the producer grid.
#include <cuda_runtime.h>

#include <cstdlib>

#include "../common.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {
namespace wg {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
// m16 strips per consumer warp: 2 for decode batches <= 16 tokens (256-channel
// row-blocks halve activation re-reads), 1 above (keeps the f32 block + group
// accumulators of 4..8 n8 tiles in registers: 9 warps leave 168 regs/thread).
__host__ __device__ constexpr int mt_for(int nt8) { return nt8 <= 2 ? 2 : 1; }
// Two co-resident CTAs per SM (two producer warps, twice the bytes in flight)
// while the accumulators fit in 96 registers; one CTA for 64-token batches.
__host__ __device__ constexpr int ctas_per_sm(int nt8) { return nt8 >= 8 ? 1 : 2; }

struct Params {
    const void* a;
    const uint8_t* codes;
    const uint16_t* scales;
    void* out;
    float* partials;
    int* counters;
    int64_t N, K;
    int M;            // tokens in this launch (<= 64)
    int NS;           // 16-row strips (ceil(N / 16))
    int NB;           // row-blocks (ceil(NS / STRIPS))
    int KBLK;         // k-blocks (K / KB)
    int U;            // units = NB * KBLK
    int G;            // CTAs
    int out_dtype;
    int scale_groups;   // scale groups per stage: 1 (g >= KB) or KB / g
    int steps_per_group;  // k16 steps per group when g < KB, else 0
    int kb_group_mask;  // g >= KB and g < K: g/KB - 1 (flush when (kb+1) & mask == 0); -1: never
    int kb_per_group_shift;  // log2(g / KB) when g >= KB and g < K
};

// ---- PTX wrappers ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void grid_dep_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void grid_dep_launch() {
    asm volatile("griddepcontrol.launch_dependents;" :::);
}
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;  // (a & b) | c
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t lop3_and_xor(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;  // (a & b) ^ c
    asm("lop3.b32 %0, %1, %2, %3, 0x6A;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
template <int AT>
__device__ __forceinline__ uint32_t sub2(uint32_t a, uint32_t b) {
    uint32_t d;
    if constexpr (AT == RTNQ_BF16) asm("sub.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    else asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t fma2_f16(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// ---- register dequantizers: one k16 step of one lane -> 4 A registers ------------------
// 4-bit word: nibble j holds A element (j<4 ? 2j : 2(j-4)+1) (native layout), so
// register i = {nibble i, nibble i+4} = {a_2i, a_2i+1}.
template <int AT>
__device__ __forceinline__ void dequant4(uint32_t q, uint32_t (&r)[4]) {
    if constexpr (AT == RTNQ_BF16) {
        // bf16 128.0 = 0x4300: (nibble | 0x4300) == 128 + u; minus 136 -> u - 8.
        const uint32_t magic = 0x43004300u, sub = 0x43084308u, mask = 0x000F000Fu;
        r[0] = sub2<AT>(lop3_and_or(q, mask, magic), sub);
        r[1] = sub2<AT>(lop3_and_or(q >> 4, mask, magic), sub);
        r[2] = sub2<AT>(lop3_and_or(q >> 8, mask, magic), sub);
        r[3] = sub2<AT>(lop3_and_or(q >> 12, mask, magic), sub);
    } else {
        // f16 1024.0 = 0x6400; high nibbles land as 1024 + 16u -> *1/16 - 72.
        const uint32_t magic = 0x64006400u, sub = 0x64086408u;
        const uint32_t mul = 0x2C002C00u, add = 0xD480D480u;
        const uint32_t q8 = q >> 8;
        r[0] = sub2<AT>(lop3_and_or(q, 0x000F000Fu, magic), sub);
        r[1] = fma2_f16(lop3_and_or(q, 0x00F000F0u, magic), mul, add);
        r[2] = sub2<AT>(lop3_and_or(q8, 0x000F000Fu, magic), sub);
        r[3] = fma2_f16(lop3_and_or(q8, 0x00F000F0u, magic), mul, add);
    }
}

// 8-bit words: w0 = bytes [a0 a2 a1 a3], w1 = [a4 a6 a5 a7] (offset-binary u = c+128).
template <int AT>
__device__ __forceinline__ void dequant8(uint32_t w0, uint32_t w1, uint32_t (&r)[4]) {
    if constexpr (AT == RTNQ_BF16) {
        // x = 128 + (u & 127); y = 128 if u >= 128 else 256; x - y == u - 128 exactly.
        const uint32_t m7 = 0x007F007Fu, m8 = 0x00800080u, mg = 0x43004300u, mh = 0x43804380u;
        r[0] = sub2<AT>(lop3_and_or(w0, m7, mg), lop3_and_xor(w0, m8, mh));
        r[1] = sub2<AT>(lop3_and_or(w0 >> 8, m7, mg), lop3_and_xor(w0 >> 8, m8, mh));
        r[2] = sub2<AT>(lop3_and_or(w1, m7, mg), lop3_and_xor(w1, m8, mh));
        r[3] = sub2<AT>(lop3_and_or(w1 >> 8, m7, mg), lop3_and_xor(w1 >> 8, m8, mh));
    } else {
        const uint32_t hi = 0x64646464u, sub = 0x64806480u;  // 1024 + u - 1152
        r[0] = sub2<AT>(prmt(w0, hi, 0x4240u), sub);
        r[1] = sub2<AT>(prmt(w0, hi, 0x4341u), sub);
        r[2] = sub2<AT>(prmt(w1, hi, 0x4240u), sub);
        r[3] = sub2<AT>(prmt(w1, hi, 0x4341u), sub);
    }
}

template <int AT>
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
    if constexpr (AT == RTNQ_BF16)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    else
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
                 : "=r"(r0), "=r"(r1)
                 : "r"(addr));
}

__device__ __forceinline__ void store_out(void* out, int dt, int64_t i, float v) {
    if (dt == RTNQ_F32) static_cast<float*>(out)[i] = v;
    else if (dt == RTNQ_BF16) static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
    else static_cast<__half*>(out)[i] = __float2half_rn(v);
}

// ---- compile-time geometry ---------------------------------------------------------------
template <int BITS, int NT8, int STAGES>
struct Geo {
    static constexpr int MT = mt_for(NT8);                   // strips per warp
    static constexpr int STRIPS = MT * kConsumerWarps;       // strips per row-block
    static constexpr int ROWS = 16 * STRIPS;                 // channels per row-block
    static constexpr int CODE_BYTES = STRIPS * 512;          // one k-block of a row-block
    static constexpr int KB = BITS == 4 ? 64 : 32;           // codes per k-block
    static constexpr int STEPS = KB / 16;                    // k16 steps per stage
    static constexpr int MPAD = NT8 * 8;                     // padded tokens
    static constexpr int ASTRIDE = KB * 2 + 16;              // bytes per smem activation row
    static constexpr int SCALE_BYTES = STEPS * STRIPS * 32;  // up to KB/16 groups per stage
    static constexpr int ACT_BYTES = MPAD * ASTRIDE;
    static constexpr int STAGE_BYTES = (CODE_BYTES + SCALE_BYTES + ACT_BYTES + 127) / 128 * 128;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 2 * STAGES * 8 + 16;
};

// CTA that owns unit u under the even split of U units over G CTAs.
__device__ __forceinline__ int cta_of(int64_t u, int64_t U, int G) {
    return int(((u + 1) * G - 1) / U);
}

template <int BITS, int AT, int NT8, int STAGES>
__global__ void __launch_bounds__(kThreads, ctas_per_sm(NT8)) wgemm_kernel(const Params p) {
    using GG = Geo<BITS, NT8, STAGES>;
    constexpr int KB = GG::KB, STEPS = GG::STEPS, MT = GG::MT, STRIPS = GG::STRIPS;
    constexpr int CODE_BYTES = GG::CODE_BYTES, ROWS = GG::ROWS;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * GG::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    volatile int* flag = reinterpret_cast<volatile int*>(empty + STAGES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int u0 = int(int64_t(c) * p.U / p.G), u1 = int(int64_t(c + 1) * p.U / p.G);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1 + 32);  // producer expect_tx + 32 lanes' cp.async arrivals
            mbar_init(&empty[s], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    grid_dep_launch();

    if (warp == kConsumerWarps) {
        // ===================== producer warp (all 32 lanes issue copies) =====================
        const int n_units = u1 - u0;
        const int prologue = n_units < STAGES ? n_units : STAGES;
        const uint32_t act_bytes = uint32_t(KB * 2);
        const int64_t a_row = p.K * 2;
        // Codes + scales: one TMA bulk copy each (a bulk-copy instruction costs ~70
        // cycles of producer issue, so a stage uses as few as possible).
        auto weights = [&](int b, int kb, int s) {
            if (lane != 0) return;
            const int strips = min(STRIPS, p.NS - b * STRIPS);
            uint8_t* st = smem + s * GG::STAGE_BYTES;
            mbar_expect_tx(&full[s], uint32_t(strips * 512 + p.scale_groups * strips * 32));
            bulk_g2s(st, p.codes + (int64_t(kb) * p.NS + b * STRIPS) * 512, uint32_t(strips * 512),
                     &full[s]);
            for (int q = 0; q < p.scale_groups; ++q) {
                const int64_t grp = p.steps_per_group ? int64_t(kb) * p.scale_groups + q
                                    : (p.kb_group_mask < 0 ? 0 : kb >> p.kb_per_group_shift);
                bulk_g2s(st + CODE_BYTES + q * STRIPS * 32,
                         p.scales + (grp * p.NS + b * STRIPS) * 16, uint32_t(strips * 32),
                         &full[s]);
            }
        };
        // Activations: 16-byte cp.async (LDGSTS) per lane -- M rows x KB*2 bytes is
        // too fragmented for bulk copies.  Each lane then arms the stage's mbarrier
        // to fire when its copies land (cp.async.mbarrier.arrive.noinc).
        auto acts = [&](int kb, int s) {
            const uint32_t dst = smem_u32(smem + s * GG::STAGE_BYTES + CODE_BYTES + GG::SCALE_BYTES);
            const uint8_t* src = static_cast<const uint8_t*>(p.a) + int64_t(kb) * (KB * 2);
            constexpr int CHUNKS = KB * 2 / 16;  // 16-byte chunks per row
            for (int i = lane; i < p.M * CHUNKS; i += 32) {
                const int r = i / CHUNKS, ch = i % CHUNKS;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 dst + r * GG::ASTRIDE + ch * 16),
                             "l"(src + r * a_row + ch * 16)
                             : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                             smem_u32(&full[s]))
                         : "memory");
        };
        {
            int b = u0 / p.KBLK, kb = u0 - b * p.KBLK;
            for (int it = 0; it < prologue; ++it) {
                weights(b, kb, it);
                if (++kb == p.KBLK) kb = 0, ++b;
            }
        }
        grid_dep_wait();  // activations are produced by the previous kernel
        int b = u0 / p.KBLK, kb = u0 - b * p.KBLK;
        for (int it = 0; it < prologue; ++it) {
            acts(kb, it);
            if (++kb == p.KBLK) kb = 0, ++b;
        }
        int s = prologue % STAGES;
        uint32_t phase = prologue == STAGES ? 0u : 1u;  // parity of the empty phase to await
        for (int it = prologue; it < n_units; ++it) {
            mbar_wait(&empty[s], phase);
            weights(b, kb, s);
            acts(kb, s);
            if (++kb == p.KBLK) kb = 0, ++b;
            if (++s == STAGES) s = 0, phase ^= 1u;
        }
        return;
    }

    // ===================== consumer warps =====================
    const int gid = lane >> 2, tig = lane & 3;
    float acc[MT][NT8][4], blk[MT][NT8][4];

    auto zero = [](float (&x)[MT][NT8][4]) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
                for (int i = 0; i < 4; ++i) x[mt][nt][i] = 0.0f;
    };

    // Row-block epilogue: direct store, or partial + deterministic last-arriver combine.
    auto epilogue = [&](int b, bool sole_owner) {
        const int strips = min(STRIPS, p.NS - b * STRIPS);
        auto write = [&](float (&v)[MT][NT8][4]) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const int strip = MT * warp + mt;
                if (strip >= strips) continue;
#pragma unroll
                for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int64_t n = int64_t(b) * ROWS + strip * 16 + gid + 8 * (i >> 1);
                        const int m = nt * 8 + 2 * tig + (i & 1);
                        if (n < p.N && m < p.M)
                            store_out(p.out, p.out_dtype, int64_t(m) * p.N + n, v[mt][nt][i]);
                    }
            }
        };
        if (sole_owner) {
            write(acc);
            return;
        }
        constexpr int PER = MT * NT8 * 4;
        const int tid = threadIdx.x;  // 0..255
        const int slot = 2 * c + (b == u0 / p.KBLK ? 0 : 1);
        float4* mine = reinterpret_cast<float4*>(p.partials + (int64_t(slot) * 256 + tid) * PER);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt)
                mine[mt * NT8 + nt] = make_float4(acc[mt][nt][0], acc[mt][nt][1], acc[mt][nt][2],
                                                  acc[mt][nt][3]);
        __threadfence();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const int c_first = cta_of(int64_t(b) * p.KBLK, p.U, p.G);
        const int c_last = cta_of(int64_t(b + 1) * p.KBLK - 1, p.U, p.G);
        if (tid == 0) {
            const int prev = atomicAdd(p.counters + b, 1);
            const int last = prev == c_last - c_first;
            if (last) p.counters[b] = 0;  // self-reset for the next launch
            *flag = last;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (!*flag) return;
        __threadfence();
        float sum[MT][NT8][4];
        zero(sum);
        for (int cc = c_first; cc <= c_last; ++cc) {  // fixed order: deterministic
            const int cu0 = int(int64_t(cc) * p.U / p.G);
            const int cs = 2 * cc + (b == cu0 / p.KBLK ? 0 : 1);
            const float4* src =
                reinterpret_cast<const float4*>(p.partials + (int64_t(cs) * 256 + tid) * PER);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT8; ++nt) {
                    const float4 x = __ldcg(src + mt * NT8 + nt);
                    sum[mt][nt][0] += x.x;
                    sum[mt][nt][1] += x.y;
                    sum[mt][nt][2] += x.z;
                    sum[mt][nt][3] += x.w;
                }
        }
        write(sum);
    };

    // acc += S * blk for scale slot q of stage `st`, then clear blk
    auto flush = [&](const uint8_t* st, int q) {
        const uint32_t* sw = reinterpret_cast<const uint32_t*>(st + CODE_BYTES + q * STRIPS * 32);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const uint32_t h2 = sw[(MT * warp + mt) * 8 + gid];
            const float2 sc = __half22float2(*reinterpret_cast<const __half2*>(&h2));
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt) {
                acc[mt][nt][0] = fmaf(sc.x, blk[mt][nt][0], acc[mt][nt][0]);
                acc[mt][nt][1] = fmaf(sc.x, blk[mt][nt][1], acc[mt][nt][1]);
                acc[mt][nt][2] = fmaf(sc.y, blk[mt][nt][2], acc[mt][nt][2]);
                acc[mt][nt][3] = fmaf(sc.y, blk[mt][nt][3], acc[mt][nt][3]);
                blk[mt][nt][0] = blk[mt][nt][1] = blk[mt][nt][2] = blk[mt][nt][3] = 0.0f;
            }
        }
    };

    // One stage: MT strips x STEPS k16 steps x NT8 token tiles.
    auto compute = [&](const uint8_t* st, uint32_t st_act, int live_strips) {
        uint32_t wv[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const uint4 q =
                *reinterpret_cast<const uint4*>(st + ((MT * warp + mt) * 32 + lane) * 16);
            wv[mt][0] = q.x;
            wv[mt][1] = q.y;
            wv[mt][2] = q.z;
            wv[mt][3] = q.w;
        }
        const uint32_t a_base = st_act + (lane & 7) * GG::ASTRIDE + (lane >> 3) * 16;
#pragma unroll
        for (int j2 = 0; j2 < STEPS; j2 += 2) {
            uint32_t bf[NT8][4];
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt)
                ldsm_x4(a_base + nt * 8 * GG::ASTRIDE + j2 * 32, bf[nt][0], bf[nt][1], bf[nt][2],
                        bf[nt][3]);
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
                const int j = j2 + jj;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    if (MT > 1 && MT * warp + mt >= live_strips) continue;
                    uint32_t af[4];
                    if constexpr (BITS == 4) dequant4<AT>(wv[mt][j], af);
                    else dequant8<AT>(wv[mt][2 * j], wv[mt][2 * j + 1], af);
#pragma unroll
                    for (int nt = 0; nt < NT8; ++nt)
                        mma16816<AT>(blk[mt][nt], af, bf[nt][2 * jj], bf[nt][2 * jj + 1]);
                }
                if (p.steps_per_group && ((j + 1) % p.steps_per_group) == 0)
                    flush(st, j / p.steps_per_group);
            }
        }
    };

    const uint32_t smem_base = smem_u32(smem);
    int b = u0 / p.KBLK, kb = u0 - b * p.KBLK;
    int seg_kb0 = kb;
    int live = min(STRIPS, p.NS - b * STRIPS);
    int s = 0;
    uint32_t phase = 0;
    zero(acc);
    zero(blk);
    for (int u = u0; u < u1; ++u) {
        mbar_wait(&full[s], phase);
        const uint8_t* st = smem + s * GG::STAGE_BYTES;
        if (MT * warp < live)
            compute(st, smem_base + s * GG::STAGE_BYTES + CODE_BYTES + GG::SCALE_BYTES, live);
        const bool seg_end = (u + 1 == u1) || (kb + 1 == p.KBLK);
        if (!p.steps_per_group && (seg_end || ((kb + 1) & p.kb_group_mask) == 0)) flush(st, 0);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == STAGES) s = 0, phase ^= 1u;
        if (seg_end) {
            epilogue(b, seg_kb0 == 0 && kb + 1 == p.KBLK);
            zero(acc);
            if (++kb == p.KBLK) kb = 0, ++b;
            seg_kb0 = kb;
            live = min(STRIPS, p.NS - b * STRIPS);
        } else {
            ++kb;
        }
    }
}

// ---- host side ------------------------------------------------------------------------

int sm_count() {
    static int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

int nt8_for(int64_t m) { return m <= 8 ? 1 : m <= 16 ? 2 : m <= 32 ? 4 : 8; }

int ctas_for(int64_t U, int nt8) {  // a full wave (env override for tests/tuning)
    int G = ctas_per_sm(nt8) * sm_count();
    if (const char* e = std::getenv("RTNQ_WGEMM_CTAS")) G = std::atoi(e);
    if (G < 1) G = 1;
    return int(U < G ? U : G);
}

template <int BITS, int AT, int NT8, int STAGES>
cudaError_t launch_t(const Params& p, cudaStream_t st, bool pdl) {
    constexpr int smem = Geo<BITS, NT8, STAGES>::SMEM;
    auto kern = wgemm_kernel<BITS, AT, NT8, STAGES>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(p.G));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

template <int BITS, int AT>
cudaError_t launch_bits(const Params& p, int nt8, cudaStream_t st, bool pdl) {
    switch (nt8) {
        case 1: return launch_t<BITS, AT, 1, 8>(p, st, pdl);
        case 2: return launch_t<BITS, AT, 2, 8>(p, st, pdl);
        case 4: return launch_t<BITS, AT, 4, 6>(p, st, pdl);
        default: return launch_t<BITS, AT, 8, 5>(p, st, pdl);
    }
}

}  // namespace wg

const char* wgemm_unsupported(int64_t m, int64_t n, int64_t k, int bits, int64_t g, int a_dtype) {
    (void)m;
    (void)n;
    if (a_dtype != RTNQ_BF16 && a_dtype != RTNQ_F16) return "activations must be bf16 or f16";
    const int64_t kb = native_kblock(bits);
    if (k % kb != 0) return "k must be a multiple of 64 (4-bit) / 32 (8-bit) for the tensor-core path";
    if (!(g >= k || g % 16 == 0)) return "group size must be a multiple of 16 (or span the row)";
    if (g < kb && kb % g != 0) return "unsupported group size";
    return nullptr;
}

// Workspace: [counters: fixed 64 KiB][stream-K partial slots].  The counters sit
// at a fixed offset so that, whatever shapes share one workspace, partial data
// never lands on a counter (they self-reset to zero and must start at zero).
constexpr size_t kCounterBytes = 64 * 1024;  // 16384 row-blocks (>= 2M channels)

size_t wgemm_workspace_bytes(int64_t m, int64_t n, int64_t k, int bits, int64_t g) {
    (void)g;
    const int64_t kb = native_kblock(bits);
    const int nt8 = wg::nt8_for(m < 64 ? m : 64), mt = wg::mt_for(nt8);
    const int64_t strips = 8 * mt;
    const int64_t NS = (n + 15) / 16, NB = (NS + strips - 1) / strips;
    const int64_t U = NB * (k / kb > 0 ? k / kb : 1);
    const int G = wg::ctas_for(U, nt8);
    return kCounterBytes + size_t(G) * 2 * 256 * (mt * nt8 * 4) * sizeof(float);
}

cudaError_t launch_wgemm(const WgemmArgs& A, cudaStream_t st) {
    const int64_t kb = native_kblock(A.bits);
    wg::Params p{};
    p.codes = A.codes;
    p.scales = A.scales;
    p.N = A.n;
    p.K = A.k;
    p.NS = int((A.n + 15) / 16);
    p.KBLK = int(A.k / kb);
    if (A.g >= A.k) {  // one group spanning the row (per-channel)
        p.scale_groups = 1;
        p.steps_per_group = 0;
        p.kb_group_mask = -1;
        p.kb_per_group_shift = 0;
    } else if (A.g >= kb) {
        p.scale_groups = 1;
        p.steps_per_group = 0;
        p.kb_group_mask = int(A.g / kb) - 1;
        p.kb_per_group_shift = __builtin_ctzll(uint64_t(A.g / kb));
    } else {
        p.scale_groups = int(kb / A.g);
        p.steps_per_group = int(A.g / 16);
        p.kb_group_mask = 0;
        p.kb_per_group_shift = 0;
    }
    p.out_dtype = A.out_dtype;
    p.counters = static_cast<int*>(A.workspace);
    p.partials = reinterpret_cast<float*>(static_cast<char*>(A.workspace) + kCounterBytes);
    if ((p.NS + 7) / 8 > int64_t(kCounterBytes / 4)) return cudaErrorInvalidValue;
    const int esz = A.out_dtype == RTNQ_F32 ? 4 : 2;
    for (int64_t m0 = 0; m0 < A.m; m0 += 64) {  // decode batches: one pass per 64 tokens
        p.M = int(A.m - m0 < 64 ? A.m - m0 : 64);
        p.a = static_cast<const char*>(A.a) + m0 * A.k * 2;
        p.out = static_cast<char*>(A.out) + m0 * A.n * esz;
        const int nt8 = wg::nt8_for(p.M), strips = 8 * wg::mt_for(nt8);
        p.NB = (p.NS + strips - 1) / strips;
        if (int64_t(p.NB) * p.KBLK >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
        p.U = p.NB * p.KBLK;
        p.G = wg::ctas_for(p.U, nt8);
        // PDL only between chunks of this call or when the caller vouches that the
        // previous kernel in the stream does not write this layer's weights.
        const bool pdl = A.pdl || m0 > 0;
        cudaError_t e;
        if (A.bits == 4)
            e = A.a_dtype == RTNQ_BF16 ? wg::launch_bits<4, RTNQ_BF16>(p, nt8, st, pdl)
                                       : wg::launch_bits<4, RTNQ_F16>(p, nt8, st, pdl);
        else
            e = A.a_dtype == RTNQ_BF16 ? wg::launch_bits<8, RTNQ_BF16>(p, nt8, st, pdl)
                                       : wg::launch_bits<8, RTNQ_F16>(p, nt8, st, pdl);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace rtnq_b200
