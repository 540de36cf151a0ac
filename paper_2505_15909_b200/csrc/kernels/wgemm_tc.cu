// wgemm_tc.cu -- W4A16 / W8A16 weight-only GEMM on the 5th-generation tensor cores.
//
// out[m][n] = sum_k a[m][k] * code[n][k] * S[n][k/g]   (gemm.hpp:18-27)
//
// One CTA computes a 128-row (output channel) x NT-token tile over a stream-K
// range of 64-code k-blocks.  Warp roles:
//   warp 4  producer: one cp.async.bulk (TMA) per stage for the codes of up to
//           KPS k-blocks (the native layout makes a row-block contiguous along K),
//           one for their f16 group scales, and 16-byte cp.async for the
//           activations, written directly in the UMMA K-major core-matrix order;
//           all complete on the stage's mbarrier.
//   warps 0-3 dequantizers: warp q owns TMEM lanes 32q..32q+31 = rows 32q+lane.
//           Each thread turns its row's codes into exact bf16/f16 integers with
//           LOP3/PRMT magic numbers and writes them with tcgen05.st straight into
//           a TMEM A-operand ring slot (32 columns = one k-block).  The same warps
//           are the epilogue: per quantization group they tcgen05.ld the f32
//           block accumulator and do acc += S[row][group] * block in registers --
//           the reference's block-then-scale structure (gemm.cpp:69-87) with
//           exact codes and the scale applied in f32.
//   warp 5  MMA issuer: one elected thread issues tcgen05.mma.cta_group::1.
//           kind::f16 with A in TMEM, B (activations) from shared memory and D in
//           TMEM (M=128, N=NT, K=16), and tcgen05.commit's to free A slots, smem
//           stages and publish finished group accumulators.
// Stream-K: the (row-block, k-block) units are split evenly over the grid;
// row-blocks shared by several CTAs are combined by the last CTA to arrive,
// summing partials in CTA order (deterministic; no float atomics).
// PDL (opt-in): weight prefetch for the first stages precedes griddepcontrol.wait.
#include <cuda_runtime.h>

#include <cstdlib>

#include "../common.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {
namespace tc {

constexpr int kRows = kNativeRows;  // 128: UMMA M
constexpr int kKB = kNativeKB;      // 64 codes per k-block
constexpr int kRA = 4;              // TMEM A-operand ring slots (k-blocks)
constexpr int kDequantWarps = 4;
constexpr int kThreads = (kDequantWarps + 2) * 32;

struct Params {
    const void* a;
    const uint8_t* codes;
    const uint16_t* scales;
    void* out;
    float* partials;
    int* counters;
    int64_t N, K;
    int M;      // tokens in this launch (<= NT)
    int NB;     // 128-row row-blocks
    int KBLK;   // 64-code k-blocks
    int GPR;    // scale groups per row
    int U;      // units = NB * KBLK
    int G;      // CTAs
    int out_dtype;
    int log2g;  // log2(group); 30 when one group spans the row
    int debug;  // RTNQ_WGEMM_DEBUG=2: producer copies nothing (compute-only profiling)
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
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
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

// ---- register dequantizers (exact integers as bf16x2 / f16x2 TMEM columns) -------------
// 4-bit word: nibble j holds code (j < 4 ? 2j : 2(j-4)+1) of 8 consecutive codes, so
// column i = {nibble i, nibble i+4} = codes {2i, 2i+1}.
template <int AT>
__device__ __forceinline__ void dequant4(uint32_t q, uint32_t* r) {
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

// 8-bit word: bytes [c0 c2 c1 c3] (offset-binary u = c + 128) -> columns {c0,c1}, {c2,c3}.
template <int AT>
__device__ __forceinline__ void dequant8(uint32_t w, uint32_t* r) {
    if constexpr (AT == RTNQ_BF16) {
        // x = 128 + (u & 127); y = 128 if u >= 128 else 256; x - y == u - 128 exactly.
        const uint32_t m7 = 0x007F007Fu, m8 = 0x00800080u, mg = 0x43004300u, mh = 0x43804380u;
        r[0] = sub2<AT>(lop3_and_or(w, m7, mg), lop3_and_xor(w, m8, mh));
        r[1] = sub2<AT>(lop3_and_or(w >> 8, m7, mg), lop3_and_xor(w >> 8, m8, mh));
    } else {
        const uint32_t hi = 0x64646464u, sub = 0x64806480u;  // 1024 + u - 1152
        r[0] = sub2<AT>(prmt(w, hi, 0x4240u), sub);
        r[1] = sub2<AT>(prmt(w, hi, 0x4341u), sub);
    }
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
        "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
        "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
        "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t d[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
          "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]),
          "=r"(d[14]), "=r"(d[15])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(d[i]);
}

__device__ __forceinline__ void store_out(void* out, int dt, int64_t i, float v) {
    if (dt == RTNQ_F32) static_cast<float*>(out)[i] = v;
    else if (dt == RTNQ_BF16) static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
    else static_cast<__half*>(out)[i] = __float2half_rn(v);
}

// ---- geometry ------------------------------------------------------------------------------
template <int BITS, int NT, int STAGES>
struct Geo {
    static constexpr int CPR = BITS == 4 ? 2 : 4;                  // 16-B chunks / row / k-block
    static constexpr int KPS = BITS == 4 ? 4 : 2;                  // k-blocks per stage
    static constexpr int CODE_BYTES = KPS * CPR * kRows * 16;      // 16 KiB
    static constexpr int MAX_GROUPS = KPS * kKB / 16;              // groups of >= 16 codes
    static constexpr int SCALE_BYTES = MAX_GROUPS * kRows * 2;
    static constexpr int ACT_KCH = KPS * kKB / 8;                  // 16-B k-chunks per token row
    static constexpr int ACT_BYTES = NT * ACT_KCH * 16;
    static constexpr int ACT_OFF = CODE_BYTES + SCALE_BYTES;
    static constexpr int STAGE_BYTES = (ACT_OFF + ACT_BYTES + 1023) / 1024 * 1024;
    static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
    static constexpr int SMEM = BAR_OFF + 1024 + 1024;  // barriers + alignment slack
    static constexpr int NDB_MAX = 8;                     // D buffers (2 per group in a k-block)
    static constexpr int TMEM_COLS = 256;                 // A ring 128 + D <= 128
};

__device__ __forceinline__ int cta_of(int64_t u, int64_t U, int G) {
    return int(((u + 1) * G - 1) / U);
}

// The stage sequence of a CTA: chunks of <= KPS k-blocks that never cross a
// row-block (segment) boundary.  Producer, MMA issuer and dequantizers walk it alike.
struct Walker {
    int u, u1, b, kb, KBLK, KPS;
    __device__ Walker(int u0_, int u1_, int KBLK_, int KPS_)
        : u(u0_), u1(u1_), KBLK(KBLK_), KPS(KPS_) {
        b = u0_ / KBLK_;
        kb = u0_ - b * KBLK_;
    }
    __device__ bool more() const { return u < u1; }
    __device__ int chunk() const {
        const int left_seg = KBLK - kb, left = u1 - u;
        const int n = left_seg < left ? left_seg : left;
        return n < KPS ? n : KPS;
    }
    __device__ bool seg_end(int n) const { return kb + n == KBLK || u + n == u1; }
    __device__ void advance(int n) {
        u += n;
        kb += n;
        if (kb == KBLK) kb = 0, ++b;
    }
};

template <int BITS, int AT, int NT, int STAGES, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) wgemm_tc_kernel(const Params p) {
    using GG = Geo<BITS, NT, STAGES>;
    constexpr int CPR = GG::CPR, KPS = GG::KPS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + GG::BAR_OFF);
    uint64_t* full = bars;                      // [STAGES] producer -> consumers
    uint64_t* empty = full + STAGES;            // [STAGES] consumers -> producer
    uint64_t* a_full = empty + STAGES;          // [kRA] dequant -> MMA
    uint64_t* a_empty = a_full + kRA;           // [kRA] MMA -> dequant
    uint64_t* d_full = a_empty + kRA;           // [NDB_MAX] MMA -> epilogue
    uint64_t* d_empty = d_full + GG::NDB_MAX;   // [NDB_MAX] epilogue -> MMA
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + GG::NDB_MAX);
    volatile int* flag = reinterpret_cast<volatile int*>(tmem_slot + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int u0 = int(int64_t(c) * p.U / p.G), u1 = int(int64_t(c + 1) * p.U / p.G);
    const int gmask = (1 << p.log2g) - 1;
    // D buffers: 2 per group that can end inside one k-block (groups of >= 16 codes)
    const int gpkb = p.log2g >= 6 ? 1 : (kKB >> p.log2g);
    const int ndb = 2 * gpkb;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1 + 32);           // expect_tx arrive + 32 lanes' cp.async
            mbar_init(&empty[s], kDequantWarps + 1);  // dequant warps + MMA commit
        }
        for (int i = 0; i < kRA; ++i) {
            mbar_init(&a_full[i], kDequantWarps);
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < GG::NDB_MAX; ++i) {
            mbar_init(&d_full[i], 1);
            mbar_init(&d_empty[i], kDequantWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kDequantWarps + 1) {  // MMA warp owns the TMEM allocation
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "n"(GG::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    grid_dep_launch();

    if (warp == kDequantWarps) {
        // ===================== producer =====================
        const int64_t a_row = p.K * 2;
        auto weights = [&](const Walker& w, int n, int s) {
            if (lane != 0) return;
            const int rows = min(kRows, int(p.N - int64_t(w.b) * kRows));
            const int rows8 = (rows + 7) / 8 * 8;
            const int g0 = (w.kb * kKB) >> p.log2g, g1 = ((w.kb + n) * kKB - 1) >> p.log2g;
            const uint32_t code_bytes = uint32_t(n * CPR * rows * 16);
            const uint32_t scale_bytes = uint32_t((g1 - g0 + 1) * rows8 * 2);
            uint8_t* st = smem + s * GG::STAGE_BYTES;
            if (p.debug & 2) {
                mbar_expect_tx(&full[s], 0);
                return;
            }
            mbar_expect_tx(&full[s], code_bytes + scale_bytes);
            bulk_g2s(st,
                     p.codes + (int64_t(w.b) * kRows * p.KBLK * CPR + int64_t(w.kb) * CPR * rows) * 16,
                     code_bytes, &full[s]);
            bulk_g2s(st + GG::CODE_BYTES,
                     p.scales + int64_t(w.b) * kRows * p.GPR + int64_t(g0) * rows8, scale_bytes,
                     &full[s]);
        };
        auto acts = [&](const Walker& w, int n, int s) {
            const uint32_t dst = smem_u32(smem + s * GG::STAGE_BYTES + GG::ACT_OFF);
            const uint8_t* src = static_cast<const uint8_t*>(p.a) + int64_t(w.kb) * (kKB * 2);
            const int kch = n * (kKB / 8);  // 16-byte chunks per token in this stage
            const int total = (p.debug & 2) ? 0 : p.M * kch;
            for (int i = lane; i < total; i += 32) {
                const int t = i / kch, ch = i - t * kch;
                // UMMA K-major core-matrix order: [token/8][k-chunk][token%8][16 B]
                const uint32_t d = dst + ((t >> 3) * GG::ACT_KCH + ch) * 128 + (t & 7) * 16;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
                             "l"(src + t * a_row + ch * 16)
                             : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                             smem_u32(&full[s]))
                         : "memory");
        };
        Walker w(u0, u1, p.KBLK, KPS);
        int pro = 0;
        {
            Walker t = w;
            for (; pro < STAGES && t.more(); ++pro) {
                const int n = t.chunk();
                weights(t, n, pro);
                t.advance(n);
            }
        }
        grid_dep_wait();  // activations come from the previous kernel
        for (int i = 0; i < pro; ++i) {
            const int n = w.chunk();
            acts(w, n, i);
            w.advance(n);
        }
        int s = pro % STAGES;
        uint32_t ph = pro == STAGES ? 0u : 1u;
        while (w.more()) {
            const int n = w.chunk();
            mbar_wait(&empty[s], ph);
            weights(w, n, s);
            acts(w, n, s);
            w.advance(n);
            if (++s == STAGES) s = 0, ph ^= 1u;
        }
    } else if (warp == kDequantWarps + 1) {
        // ===================== MMA issuer =====================
        constexpr uint32_t fmt = AT == RTNQ_BF16 ? 1u : 0u;
        constexpr uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) |
                                   (uint32_t(NT >> 3) << 17) | (uint32_t(kRows >> 4) << 24);
        const uint32_t d_col0 = kRA * 32;
        Walker w(u0, u1, p.KBLK, KPS);
        int s = 0, ra = 0;
        uint32_t ph = 0, pha = 0;
        int ord = 0;        // groups finished so far (D buffer = ord % ndb)
        bool fresh = true;  // next MMA starts a group
        while (w.more()) {
            const int n = w.chunk();
            const bool seg_end = w.seg_end(n);
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t act = smem_u32(smem + s * GG::STAGE_BYTES + GG::ACT_OFF);
            for (int kbl = 0; kbl < n; ++kbl) {
                const int kb = w.kb + kbl;
                mbar_wait(&a_full[ra], pha);
                tc_fence_after();
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int buf = ord % ndb;
                    if (fresh && ord >= ndb) {  // buffer reuse: wait for its epilogue
                        mbar_wait(&d_empty[buf], uint32_t((ord / ndb - 1) & 1));
                        tc_fence_after();
                    }
                    if (lane == 0) {
                        const uint32_t sa = act + (kbl * 4 + t) * 2 * 128;
                        const uint64_t bdesc = uint64_t((sa >> 4) & 0x3FFFu) |
                                               (uint64_t(128 >> 4) << 16) |
                                               (uint64_t((GG::ACT_KCH * 128) >> 4) << 32) |
                                               (1ull << 46);
                        const uint32_t d_addr = tmem + d_col0 + buf * NT;
                        const uint32_t a_addr = tmem + ra * 32 + t * 8;
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(
                                d_addr),
                            "r"(a_addr), "l"(bdesc), "r"(idesc), "r"(fresh ? 0 : 1)
                            : "memory");
                    }
                    __syncwarp();
                    fresh = false;
                    const int knext = kb * kKB + (t + 1) * 16;
                    if ((knext & gmask) == 0 || (seg_end && kbl == n - 1 && t == 3)) {
                        if (lane == 0) tc_commit(&d_full[buf]);
                        ++ord;
                        fresh = true;
                    }
                }
                if (lane == 0) tc_commit(&a_empty[ra]);
                if (++ra == kRA) ra = 0, pha ^= 1u;
            }
            if (lane == 0) tc_commit(&empty[s]);  // activations of this stage consumed
            __syncwarp();
            w.advance(n);
            if (++s == STAGES) s = 0, ph ^= 1u;
            if (seg_end) fresh = true;
        }
    } else {
        // ===================== dequantizers + epilogue =====================
        const int q = warp;                      // TMEM lane quadrant
        const int row = q * 32 + lane;           // row within the row-block
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        const uint32_t d_col0 = kRA * 32;
        float acc[NT];
#pragma unroll
        for (int i = 0; i < NT; ++i) acc[i] = 0.0f;
        // Groups whose accumulator is pending (finished in the previous k-block):
        // consumed one k-block later so the MMAs have landed.
        int pend_mask = 0, pend_ord0 = 0;  // bit t: a group ended after k16 step t
        float pend_s[4] = {0, 0, 0, 0};
        int ord = 0;

        auto drain = [&]() {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (!(pend_mask & (1 << t))) continue;
                const int o = pend_ord0 + __popc(pend_mask & ((1 << t) - 1)), buf = o % ndb;
                mbar_wait(&d_full[buf], uint32_t((o / ndb) & 1));
                tc_fence_after();
                const float sc = pend_s[t];
#pragma unroll
                for (int j = 0; j < NT; j += 16) {
                    float v[16];
                    tmem_ld16(tmem + lane_base + d_col0 + buf * NT + j, v);
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[j + e] = fmaf(sc, v[e], acc[j + e]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&d_empty[buf]);
            }
            pend_mask = 0;
        };

        auto epilogue = [&](int b, bool sole_owner) {
            const int rows = min(kRows, int(p.N - int64_t(b) * kRows));
            const int64_t n0 = int64_t(b) * kRows;
            auto write = [&](const float* v) {
                if (row < rows)
#pragma unroll
                    for (int m = 0; m < NT; ++m)
                        if (m < p.M) store_out(p.out, p.out_dtype, int64_t(m) * p.N + n0 + row, v[m]);
            };
            if (sole_owner) {
                write(acc);
                return;
            }
            const int slot = 2 * c + (b == u0 / p.KBLK ? 0 : 1);
            float4* mine = reinterpret_cast<float4*>(p.partials + (int64_t(slot) * kRows + row) * NT);
#pragma unroll
            for (int i = 0; i < NT / 4; ++i)
                mine[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int c_first = cta_of(int64_t(b) * p.KBLK, p.U, p.G);
            const int c_last = cta_of(int64_t(b + 1) * p.KBLK - 1, p.U, p.G);
            if (threadIdx.x == 0) {
                int prev;
                asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;"
                             : "=r"(prev)
                             : "l"(p.counters + b)
                             : "memory");
                const int last = prev == c_last - c_first;
                if (last) p.counters[b] = 0;  // self-reset for the next launch
                *flag = last;
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (!*flag) return;
            float sum[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) sum[i] = 0.0f;
            const int first_bit = int(int64_t(c_first) * p.U / p.G) / p.KBLK == b ? 0 : 1;
            for (int cc = c_first; cc <= c_last; ++cc) {  // fixed order: deterministic
                const int cs = 2 * cc + (cc == c_first ? first_bit : 0);
                const float4* src =
                    reinterpret_cast<const float4*>(p.partials + (int64_t(cs) * kRows + row) * NT);
#pragma unroll
                for (int i = 0; i < NT / 4; ++i) {
                    const float4 x = __ldcg(src + i);
                    sum[4 * i] += x.x;
                    sum[4 * i + 1] += x.y;
                    sum[4 * i + 2] += x.z;
                    sum[4 * i + 3] += x.w;
                }
            }
            write(sum);
        };

        Walker w(u0, u1, p.KBLK, KPS);
        int seg_kb0 = w.kb;
        int s = 0, ra = 0, rause = 0;
        uint32_t ph = 0, pha = 0;
        while (w.more()) {
            const int n = w.chunk();
            const bool seg_end = w.seg_end(n);
            const int rows = min(kRows, int(p.N - int64_t(w.b) * kRows));
            const int rows8 = (rows + 7) / 8 * 8;
            const int g0 = (w.kb * kKB) >> p.log2g;
            mbar_wait(&full[s], ph);
            const uint8_t* st = smem + s * GG::STAGE_BYTES;
            const __half* sc = reinterpret_cast<const __half*>(st + GG::CODE_BYTES);
            for (int kbl = 0; kbl < n; ++kbl) {
                const int kb = w.kb + kbl;
                if (rause >= kRA) mbar_wait(&a_empty[ra], pha ^ 1u);
                uint32_t col[32];
                if constexpr (BITS == 4) {
#pragma unroll
                    for (int ch = 0; ch < CPR; ++ch) {
                        const uint4 v = *reinterpret_cast<const uint4*>(
                            st + ((kbl * CPR + ch) * rows + row) * 16);
                        dequant4<AT>(v.x, col + ch * 16 + 0);
                        dequant4<AT>(v.y, col + ch * 16 + 4);
                        dequant4<AT>(v.z, col + ch * 16 + 8);
                        dequant4<AT>(v.w, col + ch * 16 + 12);
                    }
                } else {
#pragma unroll
                    for (int ch = 0; ch < CPR; ++ch) {
                        const uint4 v = *reinterpret_cast<const uint4*>(
                            st + ((kbl * CPR + ch) * rows + row) * 16);
                        dequant8<AT>(v.x, col + ch * 8 + 0);
                        dequant8<AT>(v.y, col + ch * 8 + 2);
                        dequant8<AT>(v.z, col + ch * 8 + 4);
                        dequant8<AT>(v.w, col + ch * 8 + 6);
                    }
                }
                tmem_st32(tmem + lane_base + ra * 32, col);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_full[ra]);
                if (++ra == kRA) ra = 0, pha ^= 1u;
                ++rause;
                // accumulators of the previous k-block's groups are ready by now
                drain();
                // groups finishing in this k-block (group ends, or the segment ends)
                pend_ord0 = ord;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int knext = kb * kKB + (t + 1) * 16;
                    if ((knext & gmask) == 0 || (seg_end && kbl == n - 1 && t == 3)) {
                        const int grp = (knext - 1) >> p.log2g;
                        pend_s[t] = __half2float(sc[(grp - g0) * rows8 + row]);
                        pend_mask |= 1 << t;
                        ++ord;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);  // codes + scales of this stage consumed
            if (++s == STAGES) s = 0, ph ^= 1u;
            if (seg_end) {
                drain();
                epilogue(w.b, seg_kb0 == 0 && w.kb + n == p.KBLK);
#pragma unroll
                for (int i = 0; i < NT; ++i) acc[i] = 0.0f;
                w.advance(n);
                seg_kb0 = w.kb;
            } else {
                w.advance(n);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kDequantWarps + 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(GG::TMEM_COLS));
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

// Token tile: the MMA N.  M=128 UMMA needs N % 16 == 0; the TMEM budget (A ring
// 128 columns + D buffers <= 128 columns) caps N by the D buffers a group size needs.
int nt_for(int64_t m, int64_t g) {
    const int ndb = g >= 64 ? 2 : 2 * int(64 / g);
    const int cap = 128 / ndb;  // 64 (g >= 64), 32 (g = 32), 16 (g = 16)
    int nt = m <= 16 ? 16 : m <= 32 ? 32 : 64;
    return nt < cap ? nt : cap;
}
int ctas_per_sm(int nt) { return nt <= 32 ? 2 : 1; }

int ctas_for(int64_t U, int nt) {
    int G = ctas_per_sm(nt) * sm_count();
    if (const char* e = std::getenv("RTNQ_WGEMM_CTAS")) G = std::atoi(e);
    if (G < 1) G = 1;
    return int(U < G ? U : G);
}

template <int BITS, int AT, int NT, int STAGES, int MINB>
cudaError_t launch_t(const Params& p, cudaStream_t st, bool pdl) {
    using GG = Geo<BITS, NT, STAGES>;
    auto kern = wgemm_tc_kernel<BITS, AT, NT, STAGES, MINB>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, GG::SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(p.G));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = GG::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

// Stages: two CTAs per SM must each stay under ~110 KiB of shared memory.
template <int BITS, int AT>
cudaError_t launch_bits(const Params& p, int nt, cudaStream_t st, bool pdl) {
    switch (nt) {
        case 16: return launch_t<BITS, AT, 16, BITS == 4 ? 3 : 4, 2>(p, st, pdl);
        case 32: return launch_t<BITS, AT, 32, 3, 2>(p, st, pdl);
        default: return launch_t<BITS, AT, 64, 4, 1>(p, st, pdl);
    }
}

}  // namespace tc

const char* wgemm_unsupported(int64_t m, int64_t n, int64_t k, int bits, int64_t g, int a_dtype) {
    (void)m;
    (void)n;
    if (a_dtype != RTNQ_BF16 && a_dtype != RTNQ_F16) return "activations must be bf16 or f16";
    if (k % 64 != 0) return "k must be a multiple of 64 for the tensor-core path";
    if (!(g >= k || g % 16 == 0)) return "group size must be a multiple of 16 (or span the row)";
    if (k >= (int64_t(1) << 29)) return "k too large";
    return nullptr;
}

// Workspace: [counters: fixed 64 KiB][stream-K partial slots].  The counters sit
// at a fixed offset so that, whatever shapes share one workspace, partial data
// never lands on a counter (they self-reset to zero and must start at zero).
constexpr size_t kCounterBytes = 64 * 1024;  // 16384 row-blocks (2M channels)

size_t wgemm_workspace_bytes(int64_t m, int64_t n, int64_t k, int bits, int64_t g) {
    (void)bits;
    const int64_t NB = (n + tc::kRows - 1) / tc::kRows;
    const int64_t U = NB * (k / 64 > 0 ? k / 64 : 1);
    size_t part = 0;
    for (int nt : {16, 32, 64}) {  // every tile a call may launch
        if (nt > tc::nt_for(m, g)) break;
        const int G = tc::ctas_for(U, nt);
        const size_t need = size_t(G) * 2 * tc::kRows * nt * sizeof(float);
        part = need > part ? need : part;
    }
    return kCounterBytes + part;
}

cudaError_t launch_wgemm(const WgemmArgs& A, cudaStream_t st) {
    tc::Params p{};
    p.codes = A.codes;
    p.scales = A.scales;
    p.N = A.n;
    p.K = A.k;
    p.NB = int((A.n + tc::kRows - 1) / tc::kRows);
    p.KBLK = int(A.k / 64);
    p.GPR = int(A.g >= A.k ? 1 : (A.k + A.g - 1) / A.g);
    p.log2g = A.g >= A.k ? 30 : __builtin_ctzll(uint64_t(A.g));
    p.out_dtype = A.out_dtype;
    if (const char* e = std::getenv("RTNQ_WGEMM_DEBUG")) p.debug = std::atoi(e);
    p.counters = static_cast<int*>(A.workspace);
    p.partials = reinterpret_cast<float*>(static_cast<char*>(A.workspace) + kCounterBytes);
    if (p.NB > int(kCounterBytes / 4) || int64_t(p.NB) * p.KBLK >= (int64_t(1) << 31))
        return cudaErrorInvalidValue;
    p.U = p.NB * p.KBLK;
    const int esz = A.out_dtype == RTNQ_F32 ? 4 : 2;
    const int nt_max = tc::nt_for(A.m, A.g);
    for (int64_t m0 = 0; m0 < A.m; m0 += nt_max) {  // one pass per token tile
        p.M = int(A.m - m0 < nt_max ? A.m - m0 : nt_max);
        p.a = static_cast<const char*>(A.a) + m0 * A.k * 2;
        p.out = static_cast<char*>(A.out) + m0 * A.n * esz;
        const int nt = tc::nt_for(p.M, A.g);
        p.G = tc::ctas_for(p.U, nt);
        const bool pdl = A.pdl || m0 > 0;
        cudaError_t e;
        if (A.bits == 4)
            e = A.a_dtype == RTNQ_BF16 ? tc::launch_bits<4, RTNQ_BF16>(p, nt, st, pdl)
                                       : tc::launch_bits<4, RTNQ_F16>(p, nt, st, pdl);
        else
            e = A.a_dtype == RTNQ_BF16 ? tc::launch_bits<8, RTNQ_BF16>(p, nt, st, pdl)
                                       : tc::launch_bits<8, RTNQ_F16>(p, nt, st, pdl);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace rtnq_b200
