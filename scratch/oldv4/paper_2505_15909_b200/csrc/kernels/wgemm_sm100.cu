// wgemm_sm100.cu -- W4A16 / W8A16 weight-only GEMM for decode batches.
//
// out[m][n] = sum_k a[m][k] * code[n][k] * S[n][k/g]   (gemm.hpp:18-27)
//
// Design:
//  * Weights are the M operand of mma.m16n8k16 (16 output channels per tile),
//    tokens the N operand: a batch of 1..8 tokens costs one n8 tile.
//  * Native layout (common.cuh): a 256-channel row-block is one contiguous run
//    along K, so each CTA streams contiguous memory; a pipeline stage is two
//    k-blocks (16 KiB of codes) moved by ONE cp.async.bulk (TMA, UBLKCP), plus one
//    bulk copy for the stage's f16 group scales.  Activations (a few hundred
//    bytes per token and stage, too fragmented for bulk copies) come in with
//    16-byte cp.async (LDGSTS) from the producer warp's 32 lanes, completing on
//    the same mbarrier (cp.async.mbarrier.arrive.noinc).
//  * Each lane's 16 bytes of a (strip, k-block) tile are its own A fragments: one
//    LDS.128, then LOP3/PRMT magic-number dequantization to exact bf16x2/f16x2
//    codes, mma into a per-group f32 block accumulator, and one FFMA per element
//    per group: acc += S * block -- the reference's accumulation structure
//    (gemm.cpp:69-87) with the scale applied in f32.
//  * Stream-K: the (row-block, k-block) units are split evenly over the grid;
//    row-blocks shared by several CTAs are combined by the last CTA to arrive,
//    summing the partials in CTA order (deterministic, no float atomics).
//  * Occupancy: 1..8-token and 9..16-token batches run 4 consumer warps x 4
//    strips with two CTAs per SM (two producers, ~128 KiB in flight per SM);
//    17..32-token batches run 8 consumer warps x 2 strips, one CTA per SM.
//  * PDL (opt-in): weight prefetch for the first stages is issued before
//    griddepcontrol.wait; only the activation copies wait for the producer grid.
#include <cuda_runtime.h>

#include <cstdlib>

#include "../common.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {
namespace wg {

constexpr int kStrips = kNativeBlockStrips;  // 16 strips = 256 channels per row-block
constexpr int kKPS = 2;                      // k-blocks per pipeline stage

struct Params {
    const void* a;
    const uint8_t* codes;
    const uint16_t* scales;
    void* out;
    float* partials;
    int* counters;
    int64_t N, K;
    int M;       // tokens in this launch (<= 32)
    int NS;      // 16-row strips (ceil(N / 16))
    int NB;      // row-blocks (ceil(NS / 16))
    int KBLK;    // k-blocks (K / KB)
    int GPR;     // scale groups per row
    int U;       // units = NB * KBLK
    int G;       // CTAs
    int out_dtype;
    int log2g;   // log2(group size); 30 when one group spans the row
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
template <int BITS, int NT8, int CW, int STAGES>
struct Geo {
    static constexpr int MT = kStrips / CW;                  // strips per consumer warp
    static constexpr int THREADS = (CW + 1) * 32;
    static constexpr int KB = BITS == 4 ? 64 : 32;           // codes per k-block
    static constexpr int STEPS = KB / 16;                    // k16 steps per k-block
    static constexpr int MPAD = NT8 * 8;                     // padded tokens
    static constexpr int ASTRIDE = kKPS * KB * 2 + 16;       // bytes per smem activation row
    static constexpr int CODE_BYTES = kKPS * kStrips * 512;  // 16 KiB
    static constexpr int SCALE_BYTES = kKPS * STEPS * kStrips * 32;  // up to KB/16 groups/k-block
    static constexpr int ACT_BYTES = MPAD * ASTRIDE;
    static constexpr int STAGE_BYTES = (CODE_BYTES + SCALE_BYTES + ACT_BYTES + 127) / 128 * 128;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 2 * STAGES * 8 + 16;
};

// CTA that owns unit u under the even split of U units over G CTAs.
__device__ __forceinline__ int cta_of(int64_t u, int64_t U, int G) {
    return int(((u + 1) * G - 1) / U);
}

// The stage sequence of CTA c: consecutive chunks of <= kKPS k-blocks that never
// cross a row-block (segment) boundary.  Producer and consumers walk it alike.
struct Walker {
    int u, u1, b, kb, KBLK;
    __device__ Walker(int u0_, int u1_, int KBLK_) : u(u0_), u1(u1_), KBLK(KBLK_) {
        b = u0_ / KBLK_;
        kb = u0_ - b * KBLK_;
    }
    __device__ bool more() const { return u < u1; }
    __device__ int chunk() const {  // k-blocks in the current stage
        const int left_seg = KBLK - kb, left = u1 - u;
        const int n = left_seg < left ? left_seg : left;
        return n < kKPS ? n : kKPS;
    }
    __device__ bool seg_end(int n) const { return kb + n == KBLK || u + n == u1; }
    __device__ void advance(int n) {
        u += n;
        kb += n;
        if (kb == KBLK) kb = 0, ++b;
    }
};

template <int BITS, int AT, int NT8, int CW, int STAGES>
__global__ void __launch_bounds__(Geo<BITS, NT8, CW, STAGES>::THREADS, CW == 4 ? 2 : 1)
wgemm_kernel(const Params p) {
    using GG = Geo<BITS, NT8, CW, STAGES>;
    constexpr int KB = GG::KB, STEPS = GG::STEPS, MT = GG::MT;
    constexpr int CODE_BYTES = GG::CODE_BYTES;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * GG::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    volatile int* flag = reinterpret_cast<volatile int*>(empty + STAGES);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int u0 = int(int64_t(c) * p.U / p.G), u1 = int(int64_t(c + 1) * p.U / p.G);
    const int gmask = (1 << p.log2g) - 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1 + 32);  // producer expect_tx + 32 lanes' cp.async arrivals
            mbar_init(&empty[s], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    grid_dep_launch();

    if (warp == CW) {
        // ===================== producer warp =====================
        const int64_t a_row = p.K * 2;
        auto weights = [&](const Walker& w, int n, int s) {
            if (lane != 0) return;
            const int strips = min(kStrips, p.NS - w.b * kStrips);
            const int g0 = (w.kb * KB) >> p.log2g, g1 = ((w.kb + n) * KB - 1) >> p.log2g;
            const uint32_t code_bytes = uint32_t(n * strips * 512);
            const uint32_t scale_bytes = uint32_t((g1 - g0 + 1) * strips * 32);
            uint8_t* st = smem + s * GG::STAGE_BYTES;
            mbar_expect_tx(&full[s], code_bytes + scale_bytes);
            bulk_g2s(st, p.codes + (int64_t(w.b) * kStrips * p.KBLK + int64_t(w.kb) * strips) * 512,
                     code_bytes, &full[s]);
            bulk_g2s(st + CODE_BYTES,
                     p.scales + (int64_t(w.b) * kStrips * p.GPR + int64_t(g0) * strips) * 16,
                     scale_bytes, &full[s]);
        };
        auto acts = [&](const Walker& w, int n, int s) {
            const uint32_t dst = smem_u32(smem + s * GG::STAGE_BYTES + CODE_BYTES + GG::SCALE_BYTES);
            const uint8_t* src = static_cast<const uint8_t*>(p.a) + int64_t(w.kb) * (KB * 2);
            const int chunks = n * (KB * 2 / 16);  // 16-byte chunks per row
            for (int i = lane; i < p.M * chunks; i += 32) {
                const int r = i / chunks, ch = i - r * chunks;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 dst + r * GG::ASTRIDE + ch * 16),
                             "l"(src + r * a_row + ch * 16)
                             : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                             smem_u32(&full[s]))
                         : "memory");
        };
        // Prologue: weights for the first STAGES stages before waiting on the
        // producer grid (PDL); activations after.
        Walker w(u0, u1, p.KBLK);
        int pro = 0;
        {
            Walker t = w;
            for (; pro < STAGES && t.more(); ++pro) {
                const int n = t.chunk();
                weights(t, n, pro);
                t.advance(n);
            }
        }
        grid_dep_wait();
        for (int i = 0; i < pro; ++i) {
            const int n = w.chunk();
            acts(w, n, i);
            w.advance(n);
        }
        int s = pro % STAGES;
        uint32_t phase = pro == STAGES ? 0u : 1u;
        while (w.more()) {
            const int n = w.chunk();
            mbar_wait(&empty[s], phase);
            weights(w, n, s);
            acts(w, n, s);
            w.advance(n);
            if (++s == STAGES) s = 0, phase ^= 1u;
        }
        return;
    }

    // ===================== consumer warps =====================
    const int gid = lane >> 2, tig = lane & 3;
    constexpr int NTHREADS = CW * 32;
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
        const int strips = min(kStrips, p.NS - b * kStrips);
        auto write = [&](float (&v)[MT][NT8][4]) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const int strip = MT * warp + mt;
                if (strip >= strips) continue;
#pragma unroll
                for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int64_t n = int64_t(b) * (kStrips * 16) + strip * 16 + gid + 8 * (i >> 1);
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
        const int tid = threadIdx.x;
        const int slot = 2 * c + (b == u0 / p.KBLK ? 0 : 1);
        float4* mine = reinterpret_cast<float4*>(p.partials + (int64_t(slot) * NTHREADS + tid) * PER);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt)
                mine[mt * NT8 + nt] = make_float4(acc[mt][nt][0], acc[mt][nt][1], acc[mt][nt][2],
                                                  acc[mt][nt][3]);
        // Publish: the CTA barrier orders every thread's partial stores before thread
        // 0's gpu-scope release (fences are cumulative); the last arriver's acquire
        // makes all contributors' partials visible before its CTA-wide reads.
        asm volatile("bar.sync 1, %0;" ::"n"(NTHREADS) : "memory");
        const int c_first = cta_of(int64_t(b) * p.KBLK, p.U, p.G);
        const int c_last = cta_of(int64_t(b + 1) * p.KBLK - 1, p.U, p.G);
        if (tid == 0) {
            int prev;
            asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;"
                         : "=r"(prev)
                         : "l"(p.counters + b)
                         : "memory");
            const int last = prev == c_last - c_first;
            if (last) p.counters[b] = 0;  // self-reset for the next launch
            *flag = last;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(NTHREADS) : "memory");
        if (!*flag) return;
        float sum[MT][NT8][4];
        zero(sum);
        // contributors after the first start inside row-block b: their slot for b
        // is their first-segment slot
        const int first_bit = int(int64_t(c_first) * p.U / p.G) / p.KBLK == b ? 0 : 1;
        constexpr int BATCH = MT * NT8 >= 8 ? 1 : 2;
        for (int c0 = c_first; c0 <= c_last; c0 += BATCH) {
            float4 x[BATCH][MT * NT8];
#pragma unroll
            for (int q = 0; q < BATCH; ++q) {
                const int cc = c0 + q;
                if (cc > c_last) break;
                const int cs = 2 * cc + (cc == c_first ? first_bit : 0);
                const float4* src =
                    reinterpret_cast<const float4*>(p.partials + (int64_t(cs) * NTHREADS + tid) * PER);
#pragma unroll
                for (int i = 0; i < MT * NT8; ++i) x[q][i] = __ldcg(src + i);
            }
#pragma unroll
            for (int q = 0; q < BATCH; ++q) {
                if (c0 + q > c_last) break;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                    for (int nt = 0; nt < NT8; ++nt) {
                        const float4 v = x[q][mt * NT8 + nt];
                        sum[mt][nt][0] += v.x;
                        sum[mt][nt][1] += v.y;
                        sum[mt][nt][2] += v.z;
                        sum[mt][nt][3] += v.w;
                    }
            }
        }
        write(sum);
    };

    // acc += S * blk with the scales of group slot q of the stage, then clear blk.
    auto flush = [&](const uint8_t* sc_base, int strips, int q) {
        const uint32_t* sw = reinterpret_cast<const uint32_t*>(sc_base + q * strips * 32);
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

    const uint32_t smem_base = smem_u32(smem);
    const uint32_t a_lane = (lane & 7) * GG::ASTRIDE + (lane >> 3) * 16;  // ldmatrix row address
    Walker w(u0, u1, p.KBLK);
    int seg_kb0 = w.kb;
    int s = 0;
    uint32_t phase = 0;
    zero(acc);
    zero(blk);
    while (w.more()) {
        const int n = w.chunk();
        const bool seg_end = w.seg_end(n);
        const int strips = min(kStrips, p.NS - w.b * kStrips);
        mbar_wait(&full[s], phase);
        const uint8_t* st = smem + s * GG::STAGE_BYTES;
        const uint8_t* sc = st + CODE_BYTES;
        const uint32_t st_act = smem_base + s * GG::STAGE_BYTES + CODE_BYTES + GG::SCALE_BYTES;
        const int g0 = (w.kb * KB) >> p.log2g;
        if (MT * warp < strips) {
#pragma unroll
            for (int kbl = 0; kbl < kKPS; ++kbl) {
                if (kbl >= n) break;
                const int kbg = w.kb + kbl;
                uint32_t wv[MT][4];  // this lane's 16 bytes of each of its strips
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    uint4 q = make_uint4(0, 0, 0, 0);
                    if (MT * warp + mt < strips)
                        q = *reinterpret_cast<const uint4*>(
                            st + ((kbl * strips + MT * warp + mt) * 32 + lane) * 16);
                    wv[mt][0] = q.x;
                    wv[mt][1] = q.y;
                    wv[mt][2] = q.z;
                    wv[mt][3] = q.w;
                }
#pragma unroll
                for (int j2 = 0; j2 < STEPS; j2 += 2) {
                    uint32_t bf[NT8][4];
#pragma unroll
                    for (int nt = 0; nt < NT8; ++nt)
                        ldsm_x4(st_act + a_lane + nt * 8 * GG::ASTRIDE + (kbl * KB + j2 * 16) * 2,
                                bf[nt][0], bf[nt][1], bf[nt][2], bf[nt][3]);
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const int j = j2 + jj;
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            uint32_t af[4];
                            if constexpr (BITS == 4) dequant4<AT>(wv[mt][j], af);
                            else dequant8<AT>(wv[mt][2 * j], wv[mt][2 * j + 1], af);
#pragma unroll
                            for (int nt = 0; nt < NT8; ++nt)
                                mma16816<AT>(blk[mt][nt], af, bf[nt][2 * jj], bf[nt][2 * jj + 1]);
                        }
                        // group boundary after this k16 step (groups of 16/32 codes)
                        const int knext = kbg * KB + (j + 1) * 16;
                        if (p.log2g < (BITS == 4 ? 6 : 5) && (knext & gmask) == 0)
                            flush(sc, strips, ((knext - 1) >> p.log2g) - g0);
                    }
                }
                // group boundary or segment end after this k-block (groups >= KB)
                if (p.log2g >= (BITS == 4 ? 6 : 5) &&
                    ((((kbg + 1) * KB) & gmask) == 0 || (seg_end && kbl == n - 1)))
                    flush(sc, strips, ((kbg * KB) >> p.log2g) - g0);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == STAGES) s = 0, phase ^= 1u;
        if (seg_end) {
            epilogue(w.b, seg_kb0 == 0 && w.kb + n == p.KBLK);
            zero(acc);
            w.advance(n);
            seg_kb0 = w.kb;
        } else {
            w.advance(n);
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

int nt8_for(int64_t m) { return m <= 8 ? 1 : m <= 16 ? 2 : 4; }
int cw_for(int nt8) { return nt8 <= 2 ? 4 : 8; }
int ctas_per_sm(int nt8) { return cw_for(nt8) == 4 ? 2 : 1; }

int ctas_for(int64_t U, int nt8) {  // a full wave (env override for tests/tuning)
    int G = ctas_per_sm(nt8) * sm_count();
    if (const char* e = std::getenv("RTNQ_WGEMM_CTAS")) G = std::atoi(e);
    if (G < 1) G = 1;
    return int(U < G ? U : G);
}

template <int BITS, int AT, int NT8, int CW, int STAGES>
cudaError_t launch_t(const Params& p, cudaStream_t st, bool pdl) {
    using GG = Geo<BITS, NT8, CW, STAGES>;
    auto kern = wgemm_kernel<BITS, AT, NT8, CW, STAGES>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             GG::SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(p.G));
    cfg.blockDim = dim3(GG::THREADS);
    cfg.dynamicSmemBytes = GG::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

// Stage counts keep two CTAs per SM under ~113 KiB of shared memory each (4
// consumer warps) or one CTA per SM under 227 KiB (8 consumer warps).
template <int BITS, int AT>
cudaError_t launch_bits(const Params& p, int nt8, cudaStream_t st, bool pdl) {
    switch (nt8) {
        case 1: return launch_t<BITS, AT, 1, 4, 4>(p, st, pdl);
        case 2: return launch_t<BITS, AT, 2, 4, 4>(p, st, pdl);
        default: return launch_t<BITS, AT, 4, 8, 7>(p, st, pdl);
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
    if (k >= (int64_t(1) << 30)) return "k too large";
    return nullptr;
}

// Workspace: [counters: fixed 64 KiB][stream-K partial slots].  The counters sit
// at a fixed offset so that, whatever shapes share one workspace, partial data
// never lands on a counter (they self-reset to zero and must start at zero).
constexpr size_t kCounterBytes = 64 * 1024;  // 16384 row-blocks (>= 4M channels)

size_t wgemm_workspace_bytes(int64_t m, int64_t n, int64_t k, int bits, int64_t g) {
    (void)g;
    const int64_t kb = native_kblock(bits);
    const int nt8 = wg::nt8_for(m < 32 ? m : 32);
    const int64_t NS = (n + 15) / 16, NB = (NS + wg::kStrips - 1) / wg::kStrips;
    const int64_t U = NB * (k / kb > 0 ? k / kb : 1);
    size_t part = 0;
    for (int t : {1, 2, 4}) {  // every variant a call may launch (token chunks of <= 32)
        if (t > nt8) break;
        const int G = wg::ctas_for(U, t);
        const size_t need = size_t(G) * 2 * (16 * 32 * t * 4) * sizeof(float);
        part = need > part ? need : part;
    }
    return kCounterBytes + part;
}

cudaError_t launch_wgemm(const WgemmArgs& A, cudaStream_t st) {
    const int64_t kb = native_kblock(A.bits);
    wg::Params p{};
    p.codes = A.codes;
    p.scales = A.scales;
    p.N = A.n;
    p.K = A.k;
    p.NS = int((A.n + 15) / 16);
    p.NB = (p.NS + wg::kStrips - 1) / wg::kStrips;
    p.KBLK = int(A.k / kb);
    p.GPR = int(A.g >= A.k ? 1 : (A.k + A.g - 1) / A.g);
    p.log2g = A.g >= A.k ? 30 : __builtin_ctzll(uint64_t(A.g));
    p.out_dtype = A.out_dtype;
    p.counters = static_cast<int*>(A.workspace);
    p.partials = reinterpret_cast<float*>(static_cast<char*>(A.workspace) + kCounterBytes);
    if (p.NB > int(kCounterBytes / 4) || int64_t(p.NB) * p.KBLK >= (int64_t(1) << 31))
        return cudaErrorInvalidValue;
    p.U = p.NB * p.KBLK;
    const int esz = A.out_dtype == RTNQ_F32 ? 4 : 2;
    for (int64_t m0 = 0; m0 < A.m; m0 += 32) {  // decode batches: one pass per 32 tokens
        p.M = int(A.m - m0 < 32 ? A.m - m0 : 32);
        p.a = static_cast<const char*>(A.a) + m0 * A.k * 2;
        p.out = static_cast<char*>(A.out) + m0 * A.n * esz;
        const int nt8 = wg::nt8_for(p.M);
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
