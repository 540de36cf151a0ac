// wgemm_tc.cu -- W4A16 / W8A16 weight-only GEMM on the 5th-generation tensor cores.
//
// out[m][n] = sum_k a[m][k] * code[n][k] * S[n][k/g]   (gemm.hpp:18-27)
//
// One persistent CTA per SM computes 128-row (output channel) x NT-token tiles over
// a stream-K range of 64-code k-blocks, walked in units of 16 KiB of codes (4
// k-blocks at W4, 2 at W8): one stage, one TMEM A-ring slot, one synchronisation
// step.  Four decoupled warp roles joined by mbarriers:
//   warp 12    producer: per unit, one cp.async.bulk for the codes (the native layout
//              makes a row-block one contiguous run along K), one for the unit's f16
//              group scales, and one TMA tensor load for the activations, landing as
//              UMMA K-major core matrices; all three complete on the stage mbarrier.
//   warps 0-7  dequantizers: warp w owns TMEM lanes 32(w&3).. = rows 32(w&3)+lane of
//              the units with parity w>>2 (two warps per SM sub-partition hide each
//              other's latency).  Each thread turns its row's codes into exact bf16/f16
//              integers with LOP3/PRMT magic numbers and tcgen05.st's them into the
//              unit's TMEM A-ring slot.
//   warps 13-14 MMA issuers, one per unit parity: one elected lane issues
//              tcgen05.mma.cta_group::1.kind::f16 -- A (weights) from TMEM, B
//              (activations) from shared memory, D in TMEM, M=128, N=NT, K=16.  Every
//              unit owns one accumulator per quantization group it touches, so units
//              are independent and the two parities run as two pipelines.
//   warps 8-11 epilogue: per unit and group, tcgen05.ld of the f32 block sum and
//              acc += S[row][group] * block in registers -- the reference's
//              block-then-scale structure (gemm.cpp:69-87) with exact integer codes and
//              the f16 group scale applied in f32.
// Stream-K: the (row-block, k-block) units are split evenly over the grid; row-blocks
// shared by several CTAs are combined by the last CTA to arrive, summing partials in
// CTA order (deterministic; no float atomics).
// PDL (opt-in): weight prefetch for the first stages precedes griddepcontrol.wait.
#include <cuda.h>  // CUtensorMap
#include <cuda_runtime.h>

#include <cstdlib>

#include "../common.cuh"
#include "kernels.cuh"

// Profiling knobs (RTNQ_WGEMM_DEBUG bits) are compiled in only with -DRTNQ_KERNEL_DEBUG
// (RTNQ_KERNEL_DEBUG=1 at build time): even disabled, the checks cost a few % per launch.
#ifdef RTNQ_KERNEL_DEBUG
#define RTNQ_DBG(p) ((p).debug)
#else
#define RTNQ_DBG(p) 0
#endif

namespace rtnq_b200 {
namespace tc {

constexpr int kRows = kNativeRows;  // 128: UMMA M
constexpr int kKB = kNativeKB;      // 64 codes per k-block
constexpr int kDequantWarps = 8;    // warps 0-7: quadrant w & 3, unit parity w >> 2
constexpr int kEpiWarps = 4;        // warps 8-11: quadrant w & 3
constexpr int kEpiWarp0 = 8;
constexpr int kProducerWarp = 12;
constexpr int kMmaWarp = 13;        // warps 13..13+kMmaWarps-1: MMA issuers, unit i % kMmaWarps
constexpr int kMmaWarps = 2;  // <= 16 warps in all: 4 per SM sub-partition (its 16K-register file)
constexpr int kThreads = (13 + kMmaWarps) * 32;
constexpr int kTmemCols = 512;      // one CTA per SM owns all of TMEM
constexpr int kACols = 256;         // A ring; accumulators use the other 256 columns

struct Params {
    CUtensorMap tmap_a;  // activations as [k-chunk][token][8 elements]; OOB (m >= M, k >= K) -> 0
    const uint8_t* codes;
    const uint16_t* scales;
    void* out;
    float* partials;
    int* counters;
    int64_t N, K;
    int M;      // tokens in this launch (<= NT)
    int m0;     // first token of this launch (TMA coordinate)
    int NB;     // 128-row row-blocks
    int KBLK;   // 64-code k-blocks
    int GPR;    // scale groups per row
    int U;      // (row-block, k-block) pairs = NB * KBLK
    int G;      // CTAs
    int out_dtype;
    int log2g;  // log2(group); 30 when one group spans the row
    int csize;  // > 1: cluster split-K (csize CTAs per row-block, DSMEM reduction); 1: stream-K
    int debug;  // RTNQ_WGEMM_DEBUG bits (profiling only): 2 no copies, 4 no MMA, 8 no tcgen05.st,
                //   16 no tcgen05.ld, 32 per-role timing (rtnq_wgemm_debug_read)
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
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n"
        "@!P bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(10000000)  // suspend-time hint (ns): sleep, don't spin
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
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
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

__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t* d) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
        "%15}, [%16];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
          "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]),
          "=r"(d[14]), "=r"(d[15])
        : "r"(taddr)
        : "memory");
}

// Warp-uniform issue: every lane executes the asm, elect.sync picks one lane to issue,
// so the compiler sees no divergence (no per-MMA ELECT/R2UR loop).
__device__ __forceinline__ void umma_f16_elect(uint32_t d_addr, uint32_t a_addr, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_addr),
        "r"(a_addr), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// All k16 steps of a unit into one accumulator in one asm block: 4 (one k-block) or
// 8 (two) MMAs, a_addr advancing 8 TMEM columns and the B descriptor 256 bytes per step.
template <int STEPS, uint32_t BSTEP>
__device__ __forceinline__ void umma_unit_elect(uint32_t d_addr, uint32_t a_addr, uint64_t bdesc,
                                                uint32_t idesc, uint32_t accumulate) {
    static_assert(STEPS == 4 || STEPS == 8, "");
    if constexpr (STEPS == 4)
        asm volatile(
            "{\n.reg .pred e, p, t;\n.reg .b32 a1, a2, a3;\n.reg .b64 b1, b2, b3;\n"
            "elect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\nsetp.eq.b32 t, 0, 0;\n"
            "add.u32 a1, %1, 8;\nadd.u32 a2, %1, 16;\nadd.u32 a3, %1, 24;\n"
            "add.u64 b1, %2, %5;\nadd.u64 b2, b1, %5;\nadd.u64 b3, b2, %5;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, t;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, t;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, t;\n}\n" ::"r"(d_addr),
            "r"(a_addr), "l"(bdesc), "r"(idesc), "r"(accumulate), "n"(BSTEP)
            : "memory");
    else
        asm volatile(
            "{\n.reg .pred e, p, t;\n.reg .b32 a1, a2, a3, a4, a5, a6, a7;\n"
            ".reg .b64 b1, b2, b3, b4, b5, b6, b7;\n"
            "elect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\nsetp.eq.b32 t, 0, 0;\n"
            "add.u32 a1, %1, 8;\nadd.u32 a2, %1, 16;\nadd.u32 a3, %1, 24;\nadd.u32 a4, %1, 32;\n"
            "add.u32 a5, %1, 40;\nadd.u32 a6, %1, 48;\nadd.u32 a7, %1, 56;\n"
            "add.u64 b1, %2, %5;\nadd.u64 b2, b1, %5;\nadd.u64 b3, b2, %5;\nadd.u64 b4, b3, %5;\n"
            "add.u64 b5, b4, %5;\nadd.u64 b6, b5, %5;\nadd.u64 b7, b6, %5;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a1], b1, %3, t;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a2], b2, %3, t;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a3], b3, %3, t;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a4], b4, %3, t;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a5], b5, %3, t;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a6], b6, %3, t;\n"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a7], b7, %3, t;\n}\n" ::"r"(d_addr),
            "r"(a_addr), "l"(bdesc), "r"(idesc), "r"(accumulate), "n"(BSTEP)
            : "memory");
}

__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
            smem_u32(bar))
        : "memory");
}

// ---- geometry ------------------------------------------------------------------------------
template <int BITS, int NT>
struct Geo {
    static constexpr int KPU = BITS == 4 ? 4 : 2;                  // k-blocks per unit
    static constexpr int BLK = KPU * kKB;                          // codes per unit (aligned)
    static constexpr int LOG2BLK = BITS == 4 ? 8 : 7;
    static constexpr int STEPS = BLK / 16;                         // k16 MMA steps per unit
    static constexpr int CPR = BITS == 4 ? 2 : 4;                  // 16-B chunks / row / k-block
    static constexpr int CODE_BYTES = KPU * CPR * kRows * 16;      // 16 KiB
    static constexpr int SCALE_OFF = CODE_BYTES;                   // the unit's f16 group scales
    static constexpr int SCALE_BYTES = (BLK / 16) * kRows * 2;     // <= BLK/16 groups (g = 16)
    static constexpr int ACT_KCH = BLK / 8;                        // 16-B k-chunks per unit
    static constexpr int ACT_OFF = SCALE_OFF + SCALE_BYTES;
    static constexpr int ACT_BYTES = NT * ACT_KCH * 16;            // one TMA box [chunk][token][16 B]
    static constexpr int STAGE_BYTES = (ACT_OFF + ACT_BYTES + 1023) / 1024 * 1024;
    static constexpr int MB_BYTES = 12 * 1024;                     // scale mailbox (see kernel)
    static constexpr int STAGES_FIT = (220 * 1024 - MB_BYTES) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
    static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
    static constexpr int MB_OFF = BAR_OFF + 1024;
    static constexpr int SMEM = MB_OFF + MB_BYTES + 1024;          // + alignment slack
    static constexpr int SLOT_COLS = KPU * 32;                     // bf16x2 columns per unit
    static constexpr int RA_MAX = 8, ND_MAX = 16, MB_MAX = 24;     // barrier array sizes
    static_assert(STAGES >= 3, "tile does not fit");
};

// TMEM split between accumulators (nd x NT columns, nd a power of two with room for
// two units' worth when possible) and the A ring (the rest, ra slots).
struct TmemSplit {
    int nd, ra, d_col0;
};
__device__ __forceinline__ TmemSplit tmem_split(int nt, int slot_cols, int gpu) {
    int nd = nt == 16 ? 8 : 4;
    while (nd < 2 * gpu && nd * 2 * nt <= 256) nd *= 2;
    while (nd < gpu) nd *= 2;  // the host guarantees gpu * nt <= 256
    const int d_col0 = kTmemCols - nd * nt;
    int ra = d_col0 / slot_cols;
    ra = ra > 8 ? 8 : ra;
    return {nd, ra, d_col0};
}

__device__ __forceinline__ int cta_of(int64_t u, int64_t U, int G) {
    return int(((u + 1) * G - 1) / U);
}

// The unit sequence of a CTA: runs of <= KPU k-blocks that stay inside one KPU-aligned
// block and one row-block (segment).  Every role walks it alike.
template <int KPU>
struct Walker {
    int u, u1, b, kb, KBLK;
    __device__ Walker(int u0_, int u1_, int KBLK_) : u(u0_), u1(u1_), KBLK(KBLK_) {
        b = u0_ / KBLK_;
        kb = u0_ - b * KBLK_;
    }
    __device__ bool more() const { return u < u1; }
    __device__ int chunk() const {
        const int left_seg = KBLK - kb, left = u1 - u, cap = KPU - (kb & (KPU - 1));
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

// Accumulator slot j of a unit covers the intersection of the unit [kbase, kend) with
// the j-th group-sized piece of its aligned block; returns its first k16 step and count.
__device__ __forceinline__ void subgroup(int kbase, int kend, int blk, int lg, int j, int* k0,
                                         int* cnt) {
    const int lo0 = blk + (j << lg), hi0 = lo0 + (1 << lg);
    const int lo = lo0 > kbase ? lo0 : kbase, hi = hi0 < kend ? hi0 : kend;
    *k0 = (lo - kbase) >> 4;
    *cnt = hi > lo ? (hi - lo) >> 4 : 0;
}

// A position in a ring of n mbarrier-guarded slots, advanced incrementally: no runtime
// division on the per-unit critical path.  ph is the parity of the current use.
struct Ring {
    int idx = 0, n;
    uint32_t ph = 0;
    __device__ explicit Ring(int n_) : n(n_) {}
    __device__ void next() {
        if (++idx == n) idx = 0, ph ^= 1u;
    }
};

// Profiling-only instrumentation (RTNQ_WGEMM_DEBUG & 32): per-CTA globaltimer stamps and
// per-role blocked/total cycles, read back by rtnq_wgemm_debug_read.
__device__ unsigned long long g_wgemm_dbg[1024 * 64];
__device__ __forceinline__ void stamp(const Params& p, int slot) {
    if (!(RTNQ_DBG(p) & 32)) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_wgemm_dbg[blockIdx.x * 64 + slot] = t;
}
#define PWAIT(bar, par, slot)                                   \
    do {                                                        \
        if constexpr (PROF) {                                   \
            const long long t0_ = clock64();                    \
            mbar_wait(bar, par);                                \
            pacc[slot] += clock64() - t0_;                      \
        } else {                                                \
            mbar_wait(bar, par);                                \
        }                                                       \
    } while (0)

// Issue `cnt` k16 steps into one accumulator (the first step overwrites it).
template <uint32_t KSTEP>
__device__ __forceinline__ void issue_steps(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc,
                                            int cnt) {
    int done = 0;
    for (; cnt - done >= 8; done += 8)
        umma_unit_elect<8, KSTEP>(d, a + done * 8, bd + uint64_t(done * KSTEP), idesc, done);
    if (cnt - done >= 4) {
        umma_unit_elect<4, KSTEP>(d, a + done * 8, bd + uint64_t(done * KSTEP), idesc, done);
        done += 4;
    }
    for (; done < cnt; ++done)
        umma_f16_elect(d, a + done * 8, bd + uint64_t(done * KSTEP), idesc, done);
}

// A full, block-aligned unit: STEPS k16 MMAs, accumulator slot k / GS (GS steps per
// quantization group), every offset a compile-time constant added to three per-unit bases.
// One single-MMA asm per step keeps the issue stream short (measured: ~26 cycles/MMA,
// against ~70 for one asm block with runtime-derived operands).
template <int STEPS, int GS, int NT, uint32_t KSTEP>
__device__ __forceinline__ void issue_unit(uint32_t d0, uint32_t a0, uint64_t b0, uint32_t idesc) {
#pragma unroll
    for (int k = 0; k < STEPS; ++k)
        umma_f16_elect(d0 + uint32_t((k / GS) * NT), a0 + uint32_t(k * 8),
                       b0 + uint64_t(k * KSTEP), idesc, (k % GS) != 0 ? 1u : 0u);
}

template <int STEPS, int NT, uint32_t KSTEP>
__device__ __forceinline__ void issue_unit_lg(int lg, uint32_t d0, uint32_t a0, uint64_t b0,
                                              uint32_t idesc) {
    const int gs = (1 << lg) >> 4;  // k16 steps per group piece (<= STEPS)
    switch (gs) {
        case 16: if constexpr (STEPS >= 16) { issue_unit<STEPS, 16, NT, KSTEP>(d0, a0, b0, idesc); break; }
                 [[fallthrough]];
        case 8: issue_unit<STEPS, 8, NT, KSTEP>(d0, a0, b0, idesc); break;
        case 4: issue_unit<STEPS, 4, NT, KSTEP>(d0, a0, b0, idesc); break;
        case 2: issue_unit<STEPS, 2, NT, KSTEP>(d0, a0, b0, idesc); break;
        default: issue_unit<STEPS, 1, NT, KSTEP>(d0, a0, b0, idesc); break;
    }
}

// PROF=true (RTNQ_WGEMM_DEBUG & 32) accumulates per-role wait cycles in registers.
template <int BITS, int AT, int NT, bool PROF>
__global__ void __maxnreg__(128) wgemm_tc_kernel(const __grid_constant__ Params p) {
    using GG = Geo<BITS, NT>;
    constexpr int CPR = GG::CPR, STAGES = GG::STAGES, KPU = GG::KPU;
    extern __shared__ uint8_t smem_raw[];
    // align by indexing the __shared__ array (keeps the shared address space: LDS/STS, not
    // generic loads)
    uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + GG::BAR_OFF);
    // Barrier protocol (one tcgen05.commit per unit):
    //   full[s]    producer (TMA complete_tx) -> dequant, MMA
    //   a_full[r]  the unit's 4 dequant warps -> MMA (A-ring slot r written)
    //   done[u]    MMA commit of unit u -> producer (stage reusable), dequant (A slot
    //              reusable), epilogue (accumulators ready); u & 31, parity (u >> 5) & 1
    //   d_free[u]  epilogue (4 warps) -> MMA: unit u's accumulators have been read
    //   m_full[e]  dequant -> epilogue: the unit's group scales are in mailbox entry e
    // Rings indexed by the unit number modulo 32 are safe because no waiter ever lags the
    // newest completed phase of its slot by 32 units (stages <= 8, accumulators <= 16 units).
    uint64_t* full = bars;                    // [STAGES]
    uint64_t* a_full = full + STAGES;         // [RA]
    uint64_t* done = a_full + GG::RA_MAX;     // [32]
    uint64_t* d_free = done + 32;             // [32]
    uint64_t* m_full = d_free + 32;           // [MB]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(m_full + GG::MB_MAX);
    __half* mbox = reinterpret_cast<__half*>(smem + GG::MB_OFF);  // [MB][gpu][128 rows]
    volatile int* flag = reinterpret_cast<volatile int*>(tmem_slot + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    if (threadIdx.x == 0) stamp(p, 0);
    // stream-K: an even share of all (row-block, k-block) pairs; cluster split-K: row-block
    // c / csize, k-blocks [r, r + 1) * KBLK / csize of it for cluster rank r = c % csize
    int u0, u1;
    if (p.csize > 1) {
        const int b = c / p.csize, r = c % p.csize;
        u0 = b * p.KBLK + r * p.KBLK / p.csize;
        u1 = b * p.KBLK + (r + 1) * p.KBLK / p.csize;
    } else {
        u0 = int(int64_t(c) * p.U / p.G);
        u1 = int(int64_t(c + 1) * p.U / p.G);
    }
    // accumulator slots per unit: one per group-sized piece of the aligned block
    const int lg = p.log2g < GG::LOG2BLK ? p.log2g : GG::LOG2BLK;
    const int gpu = 1 << (GG::LOG2BLK - lg);
    const TmemSplit tsp = tmem_split(NT, GG::SLOT_COLS, gpu);
    const int ND = tsp.nd, RA = tsp.ra;
    const int NU = ND / gpu;  // units whose accumulators can be in flight
    // Mailbox entry e = unit % MB carries the unit's group scales from its dequant warps
    // to the epilogue.  Reusing it for unit i needs the epilogue done with unit i - MB:
    // dequant(i) follows done(i - RA) <- MMA(i - RA) <- d_free(i - RA - NU).
    const int MB = RA + NU;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);  // producer's arrive.expect_tx
        for (int i = 0; i < RA; ++i) mbar_init(&a_full[i], 4);
        for (int i = 0; i < 32; ++i) {
            mbar_init(&done[i], 1);
            mbar_init(&d_free[i], kEpiWarps);
        }
        for (int i = 0; i < MB; ++i) mbar_init(&m_full[i], 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {  // the first MMA warp owns the TMEM allocation
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    grid_dep_launch();
    if (threadIdx.x == 0) stamp(p, 1);
    long long pacc[4] = {0, 0, 0, 0};
#define PT_BEGIN(v) long long v = PROF ? clock64() : 0
#define PT_END(v, slot) do { if constexpr (PROF) pacc[slot] += clock64() - v; } while (0)
    const long long prof_t0 = PROF ? clock64() : 0;
    auto prof_store = [&](int base) {  // slots base..base+3 = waits, base+4 = role time
        if constexpr (PROF) {
            for (int i = 0; i < 4; ++i) g_wgemm_dbg[blockIdx.x * 64 + base + i] = pacc[i];
            g_wgemm_dbg[blockIdx.x * 64 + base + 4] = clock64() - prof_t0;
        }
    };

    if (RTNQ_DBG(p) & 1024) {
        // profiling: the MMA issue stream alone (no other role, no barrier waits)
        if (warp == kMmaWarp) {
            constexpr uint32_t fmt = AT == RTNQ_BF16 ? 1u : 0u;
            constexpr uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) |
                                       (uint32_t(NT >> 3) << 17) | (uint32_t(kRows >> 4) << 24);
            constexpr uint64_t bdesc_hi = (uint64_t((NT * 16) >> 4) << 16) |
                                          (uint64_t(128 >> 4) << 32) | (1ull << 46);
            constexpr uint32_t kStep = (2 * NT * 16) >> 4;
            const uint32_t act0 = smem_u32(smem + GG::ACT_OFF);
            const long long t0 = clock64();
            const int units = (u1 - u0 + KPU - 1) / KPU;
            if (RTNQ_DBG(p) & 65536) {
                // the microbenchmark's loop verbatim (scratch/tc_micro.cu "rotating")
                const uint64_t bdesc = bdesc_hi | uint64_t((act0 >> 4) & 0x3FFFu);
                for (int i = 0; i < units; ++i)
                    for (int k = 0; k < 16; ++k)
                        umma_f16_elect(tmem + 256 + ((k >> 3) & 1) * NT, tmem + (k & 31) * 8,
                                       bdesc + ((k * 2 * NT) & 1023), idesc, (k & 7) != 0);
            } else
            for (int i = 0; i < units; ++i) {
                const int s = (RTNQ_DBG(p) & 4096) ? 0 : i % STAGES;
                const int slot = (RTNQ_DBG(p) & 8192) ? 0 : i % RA;
                const uint64_t bdesc0 = bdesc_hi | uint64_t(((act0 + s * GG::STAGE_BYTES) >> 4) & 0x3FFFu);
                for (int j = 0; j < gpu; ++j)
                    issue_steps<kStep>(tmem + tsp.d_col0 + (((RTNQ_DBG(p) & 16384) ? 0 : (i * gpu + j)) & (ND - 1)) * NT,
                                       tmem + slot * GG::SLOT_COLS + j * (GG::STEPS / gpu) * 8,
                                       bdesc0 + uint64_t(j * (GG::STEPS / gpu) * kStep), idesc,
                                       GG::STEPS / gpu);
                if (!(RTNQ_DBG(p) & 2048)) {
                    tc_commit_elect(&done[i & 31]);
                    if (i >= 4) mbar_wait(&done[(i - 4) & 31], uint32_t((i - 4) >> 5) & 1u);
                }
            }
            tc_commit_elect(&done[31]);
            mbar_wait(&done[31], (RTNQ_DBG(p) & 2048) ? 0u : uint32_t(units > 31 ? 1 : 0));
            const long long t1 = clock64();
            if (lane == 0 && (RTNQ_DBG(p) & 32)) g_wgemm_dbg[blockIdx.x * 64 + 60] = (t1 - t0) / (units ? units : 1);
        }
    } else if (warp == kProducerWarp) {
        // ===================== producer =====================
        // Codes and the unit's group scales: bulk copies of contiguous runs.  Activations:
        // one TMA box of BLK/8 k-chunks x NT tokens.  All complete on full[s].
        auto weights = [&](const Walker<KPU>& w, int n, int s) {
            if (lane != 0 || (RTNQ_DBG(p) & 2)) return;
            const int rows = min(kRows, int(p.N - int64_t(w.b) * kRows));
            const int rows8 = (rows + 7) / 8 * 8, kbase = w.kb * kKB;
            const uint32_t code_bytes = uint32_t(n * CPR * rows * 16);
            const int g0 = kbase >> p.log2g;
            int g1 = (kbase + n * kKB - 1) >> p.log2g;
            g1 = g1 < p.GPR ? g1 : p.GPR - 1;
            const uint32_t scale_bytes = uint32_t((g1 - g0 + 1) * rows8 * 2);
            uint8_t* st = smem + s * GG::STAGE_BYTES;
            mbar_expect_tx_only(&full[s], code_bytes + scale_bytes);
            bulk_g2s(st,
                     p.codes + (int64_t(w.b) * kRows * p.KBLK * CPR + int64_t(w.kb) * CPR * rows) * 16,
                     code_bytes, &full[s]);
            bulk_g2s(st + GG::SCALE_OFF,
                     p.scales + int64_t(w.b) * kRows * p.GPR + int64_t(g0) * rows8, scale_bytes,
                     &full[s]);
        };
        auto acts = [&](const Walker<KPU>& w, int s) {
            if (lane != 0) return;
            if (RTNQ_DBG(p) & 2) {
                mbar_arrive(&full[s]);
                return;
            }
            mbar_expect_tx(&full[s], GG::ACT_BYTES);
            tma_load_3d(smem + s * GG::STAGE_BYTES + GG::ACT_OFF, &p.tmap_a, 0, p.m0,
                        w.kb * (kKB / 8), &full[s]);
        };
        Walker<KPU> w(u0, u1, p.KBLK);
        int pro = 0;
        {
            Walker<KPU> t = w;
            for (; pro < STAGES && t.more(); ++pro) {
                const int n = t.chunk();
                weights(t, n, pro);
                t.advance(n);
            }
        }
        grid_dep_wait();  // activations come from the previous kernel
        for (int i = 0; i < pro; ++i) {
            acts(w, i);
            w.advance(w.chunk());
        }
        Ring st(STAGES);  // stage ring position of unit `pro` onward
        for (int i = 0; i < pro; ++i) st.next();
        int iu = pro;     // unit number
        // L2 prefetch runs kPrefetch units ahead of the stage ring, so DRAM latency is
        // covered by L2 rather than by shared-memory stages
        constexpr int kPrefetch = 8;
        Walker<KPU> pf = w;
        auto prefetch_unit = [&](const Walker<KPU>& x) {
            const int n = x.chunk(), rows = min(kRows, int(p.N - int64_t(x.b) * kRows));
            if (lane == 0 && !(RTNQ_DBG(p) & 2))
                prefetch_l2(p.codes + (int64_t(x.b) * kRows * p.KBLK * CPR + int64_t(x.kb) * CPR * rows) * 16,
                            uint32_t(n * CPR * rows * 16));
        };
        for (int i = 0; i < kPrefetch && pf.more(); ++i) {
            prefetch_unit(pf);
            pf.advance(pf.chunk());
        }
        while (w.more()) {
            const int n = w.chunk(), s = st.idx;
            if (pf.more()) {
                prefetch_unit(pf);
                pf.advance(pf.chunk());
            }
            {  // the previous use of this stage (unit iu - STAGES) is done
                const int v = iu - STAGES;
                PWAIT(&done[v & 31], uint32_t(v >> 5) & 1u, 0);
            }
            weights(w, n, s);
            acts(w, s);
            w.advance(n);
            st.next();
            ++iu;
        }
        if (lane == 0) stamp(p, 2), prof_store(8);
    } else if (warp >= kMmaWarp) {
        // ===================== MMA issuers (warp-uniform, one lane issues) =====================
        const int par = warp - kMmaWarp;
        const int nmma = (RTNQ_DBG(p) & 512) ? 1 : kMmaWarps;  // profiling: one warp issues all
        constexpr uint32_t fmt = AT == RTNQ_BF16 ? 1u : 0u;
        constexpr uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) |
                                   (uint32_t(NT >> 3) << 17) | (uint32_t(kRows >> 4) << 24);
        // B descriptor: K-major, no swizzle, smem [k-chunk][token][16 B]: LBO = NT*16 B
        // (next k core matrix), SBO = 128 B (next 8 tokens); start address per stage/step.
        constexpr uint64_t bdesc_hi = (uint64_t((NT * 16) >> 4) << 16) |
                                      (uint64_t(128 >> 4) << 32) | (1ull << 46);
        constexpr uint32_t kStep = (2 * NT * 16) >> 4;  // one k16 step = 2 k-chunks
        const uint32_t act0 = smem_u32(smem + GG::ACT_OFF);
        const uint32_t d_base = tmem + tsp.d_col0;
        Walker<KPU> w(u0, u1, p.KBLK);
        Ring st(STAGES), sl(RA);
        int ob0 = 0;  // first accumulator ordinal of the unit (gpu per unit)
        int mi = 0;  // i % nmma, kept incrementally
        for (int i = 0; w.more(); ++i, st.next(), sl.next(), ob0 += gpu, mi = mi + 1 == nmma ? 0 : mi + 1) {
            const int n = w.chunk();
            if (mi == par) {
                const int s = st.idx, slot = sl.idx;
                const int kbase = w.kb * kKB, kend = kbase + n * kKB, blk = kbase & ~(GG::BLK - 1);
                PWAIT(&full[s], st.ph, 0);
                PWAIT(&a_full[slot], sl.ph, 1);
                tc_fence_after();
                const uint64_t bdesc0 =
                    bdesc_hi | uint64_t(((act0 + s * GG::STAGE_BYTES) >> 4) & 0x3FFFu);
                const uint32_t a_base = tmem + slot * GG::SLOT_COLS;
                if (i >= NU) {  // accumulator reuse: the epilogue has read unit i - NU
                    const int v = i - NU;
                    PWAIT(&d_free[v & 31], uint32_t(v >> 5) & 1u, 2);
                    tc_fence_after();
                }
                PT_BEGIN(tiss);
                if (RTNQ_DBG(p) & 4) {
                } else if (n == KPU && kbase == blk) {  // full aligned unit: unrolled issue
                    const uint32_t a_use = (RTNQ_DBG(p) & 131072) ? tmem : a_base;  // profiling knobs
                    const uint64_t b_use =
                        (RTNQ_DBG(p) & 262144) ? (bdesc_hi | uint64_t((act0 >> 4) & 0x3FFFu)) : bdesc0;
                    issue_unit_lg<GG::STEPS, NT, kStep>(lg, d_base + (ob0 & (ND - 1)) * NT, a_use,
                                                        b_use, idesc);
                } else {
                    for (int j = 0; j < gpu; ++j) {
                        const int buf = (ob0 + j) & (ND - 1);
                        int k0, cnt;
                        subgroup(kbase, kend, blk, lg, j, &k0, &cnt);
                        if (cnt > 0)
                            issue_steps<kStep>(d_base + buf * NT, a_base + k0 * 8,
                                               bdesc0 + uint64_t(k0 * kStep), idesc, cnt);
                    }
                }
                // one commit: stage, A slot and accumulators of unit i all complete together
                tc_commit_elect(&done[i & 31]);
                PT_END(tiss, 3);
            }
            w.advance(n);
        }
        if (lane == 0 && par == 0) stamp(p, 3), prof_store(20);
    } else if (warp < kDequantWarps) {
        // ===================== dequantizers =====================
        const int q = warp & 3, par = warp >> 2;
        const int row = q * 32 + lane;  // row within the row-block = TMEM lane
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        Walker<KPU> w(u0, u1, p.KBLK);
        Ring st(STAGES), sl(RA), me(MB);
        for (int i = 0; w.more(); ++i, st.next(), sl.next(), me.next()) {
            const int n = w.chunk();
            if ((i & 1) == par) {
                const int s = st.idx, slot = sl.idx;
                const int rows = min(kRows, int(p.N - int64_t(w.b) * kRows));
                PWAIT(&full[s], st.ph, 0);
                const uint8_t* st = smem + s * GG::STAGE_BYTES + row * 16;
                const uint32_t ta = tmem + lane_base + slot * GG::SLOT_COLS;
#pragma unroll
                if (RTNQ_DBG(p) & 256) {  // profiling: barrier protocol only
                    if (i >= RA) PWAIT(&done[(i - RA) & 31], uint32_t((i - RA) >> 5) & 1u, 1);
                } else
                for (int h = 0; h < KPU / 2; ++h) {  // two k-blocks (64 columns) at a time
                    if (2 * h < n) {
                        PT_BEGIN(tq);
                        uint4 v[2 * CPR];
#pragma unroll
                        for (int j = 0; j < 2 * CPR; ++j)
                            if (2 * h * CPR + j < n * CPR)
                                v[j] = *reinterpret_cast<const uint4*>(st + (2 * h * CPR + j) * rows * 16);
                        uint32_t col[64];
#pragma unroll
                        for (int j = 0; j < 2 * CPR; ++j) {
                            if constexpr (BITS == 4) {
                                dequant4<AT>(v[j].x, col + j * 16 + 0);
                                dequant4<AT>(v[j].y, col + j * 16 + 4);
                                dequant4<AT>(v[j].z, col + j * 16 + 8);
                                dequant4<AT>(v[j].w, col + j * 16 + 12);
                            } else {
                                dequant8<AT>(v[j].x, col + j * 8 + 0);
                                dequant8<AT>(v[j].y, col + j * 8 + 2);
                                dequant8<AT>(v[j].z, col + j * 8 + 4);
                                dequant8<AT>(v[j].w, col + j * 8 + 6);
                            }
                        }
                        if constexpr (PROF) asm volatile("" ::"r"(col[0]), "r"(col[63]));
                        PT_END(tq, 2);
                        if (h == 0) {
                            if (i >= RA) {  // slot free? (its MMA overlapped this dequant)
                                PWAIT(&done[(i - RA) & 31], uint32_t((i - RA) >> 5) & 1u, 1);
                                tc_fence_after();
                            }
                            // this row's group scales -> the epilogue's mailbox entry
                            const int kbase = w.kb * kKB, kend = kbase + n * kKB;
                            const int blk = kbase & ~(GG::BLK - 1), g0 = kbase >> p.log2g;
                            const int rows8 = (rows + 7) / 8 * 8;
                            const __half* sc_st = reinterpret_cast<const __half*>(
                                                      smem + s * GG::STAGE_BYTES + GG::SCALE_OFF) + row;
                            __half* mb = mbox + me.idx * gpu * kRows + row;
                            for (int j = 0; j < gpu; ++j) {
                                int k0, cnt;
                                subgroup(kbase, kend, blk, lg, j, &k0, &cnt);
                                int grp = (blk + (j << lg)) >> p.log2g;
                                grp = grp < p.GPR ? grp : p.GPR - 1;
                                mb[j * kRows] = cnt > 0 && row < rows ? sc_st[(grp - g0) * rows8]
                                                                      : __float2half(0.0f);
                            }
                        }
                        PT_BEGIN(tw);
                        if (!(RTNQ_DBG(p) & 8)) {
                            tmem_st32(ta + h * 64, col);
                            if (2 * h + 1 < n) tmem_st32(ta + h * 64 + 32, col + 32);
                        }
                        PT_END(tw, 3);
                    }
                }
                PT_BEGIN(tw2);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                PT_END(tw2, 3);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&a_full[slot]);
                    mbar_arrive(&m_full[me.idx]);
                }
            }
            w.advance(n);
        }
        if (threadIdx.x == 0) stamp(p, 4), prof_store(32);
    } else if (warp < kEpiWarp0 + kEpiWarps) {
        // ===================== epilogue =====================
        const int q = warp & 3;  // TMEM lane quadrant
        const int row = q * 32 + lane;
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        const int et = threadIdx.x - kEpiWarp0 * 32;  // 0..127
        float acc[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[j] = 0.0f;

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
            for (int j = 0; j < NT / 4; ++j)
                mine[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int c_first = cta_of(int64_t(b) * p.KBLK, p.U, p.G);
            const int c_last = cta_of(int64_t(b + 1) * p.KBLK - 1, p.U, p.G);
            if (et == 0) {
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
            for (int j = 0; j < NT; ++j) sum[j] = 0.0f;
            const int first_bit = int(int64_t(c_first) * p.U / p.G) / p.KBLK == b ? 0 : 1;
            // partials in batches of PB: all loads of a batch are in flight together (one L2
            // round trip per batch), then summed in CTA order -- deterministic
            constexpr int PB = NT <= 16 ? 4 : NT <= 32 ? 2 : 1;
            for (int c0 = c_first; c0 <= c_last; c0 += PB) {
                float4 x[PB][NT / 4];
#pragma unroll
                for (int q = 0; q < PB; ++q) {
                    const int cc = c0 + q;
                    if (cc > c_last) break;
                    const int cs = 2 * cc + (cc == c_first ? first_bit : 0);
                    const float4* src =
                        reinterpret_cast<const float4*>(p.partials + (int64_t(cs) * kRows + row) * NT);
#pragma unroll
                    for (int j = 0; j < NT / 4; ++j) x[q][j] = __ldcg(src + j);
                }
#pragma unroll
                for (int q = 0; q < PB; ++q) {
                    if (c0 + q > c_last) break;
#pragma unroll
                    for (int j = 0; j < NT / 4; ++j) {
                        sum[4 * j] += x[q][j].x;
                        sum[4 * j + 1] += x[q][j].y;
                        sum[4 * j + 2] += x[q][j].z;
                        sum[4 * j + 3] += x[q][j].w;
                    }
                }
            }
            write(sum);
        };

        Walker<KPU> w(u0, u1, p.KBLK);
        int seg_kb0 = w.kb;
        Ring me(MB);
        int ob0 = 0;
        for (int i = 0; w.more(); ++i, me.next(), ob0 += gpu) {
            const int n = w.chunk();
            const bool seg_end = w.seg_end(n);
            const int kbase = w.kb * kKB, kend = kbase + n * kKB, blk = kbase & ~(GG::BLK - 1);
            // this unit's scales, handed over by its dequant warps, then its accumulators
            PWAIT(&m_full[me.idx], me.ph, 1);
            const __half* mb = mbox + me.idx * gpu * kRows + row;
            PWAIT(&done[i & 31], uint32_t(i >> 5) & 1u, 0);
            tc_fence_after();
            for (int j = 0; j < gpu; ++j) {
                int k0, cnt;
                subgroup(kbase, kend, blk, lg, j, &k0, &cnt);
                if (cnt == 0) continue;
                const int buf = (ob0 + j) & (ND - 1);
                const float sc = __half2float(mb[j * kRows]);
#pragma unroll
                for (int jj = 0; jj < NT; jj += 32) {
                    uint32_t v[32];
                    if (!(RTNQ_DBG(p) & 16)) {
                        tmem_ld16_nw(tmem + lane_base + tsp.d_col0 + buf * NT + jj, v);
                        if constexpr (NT >= 32)
                            tmem_ld16_nw(tmem + lane_base + tsp.d_col0 + buf * NT + jj + 16, v + 16);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    } else {
#pragma unroll
                        for (int e = 0; e < 32; ++e) v[e] = 0;
                    }
                    constexpr int W = NT < 32 ? NT : 32;
#pragma unroll
                    for (int e = 0; e < W; ++e)
                        acc[jj + e] = fmaf(sc, __uint_as_float(v[e]), acc[jj + e]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&d_free[i & 31]);  // accumulators of unit i read
            if (seg_end && p.csize > 1) {
                // cluster split-K: park this CTA's partial in its own shared memory (stage 0
                // is idle once the last unit is done); the cluster reduces it below
                float* red = reinterpret_cast<float*>(smem);
#pragma unroll
                for (int m = 0; m < NT; ++m) red[m * kRows + row] = acc[m];
                w.advance(n);
            } else if (seg_end) {
                if (et == 0) stamp(p, 5);
                epilogue(w.b, seg_kb0 == 0 && w.kb + n == p.KBLK);
                if (et == 0) stamp(p, 6), prof_store(44);
#pragma unroll
                for (int j = 0; j < NT; ++j) acc[j] = 0.0f;
                w.advance(n);
                seg_kb0 = w.kb;
            } else {
                w.advance(n);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (p.csize > 1) {
        // DSMEM reduction: rank 0 of the cluster sums every rank's partial, in rank order
        // (deterministic), and writes the row-block's output; the second barrier keeps the
        // other ranks' shared memory alive until rank 0 has read it.
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (c % p.csize == 0 && warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps) {
            const int row = (warp & 3) * 32 + lane;
            const int b = c / p.csize;
            const int rows = min(kRows, int(p.N - int64_t(b) * kRows));
            float sum[NT];
#pragma unroll
            for (int m = 0; m < NT; ++m) sum[m] = 0.0f;
            const uint32_t red = smem_u32(smem);
            for (int r = 0; r < p.csize; ++r) {
                uint32_t rbase;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbase) : "r"(red), "r"(r));
#pragma unroll
                for (int m = 0; m < NT; ++m) {
                    float v;
                    asm volatile("ld.shared::cluster.f32 %0, [%1];"
                                 : "=f"(v)
                                 : "r"(rbase + uint32_t((m * kRows + row) * 4)));
                    sum[m] += v;
                }
            }
            if (row < rows)
#pragma unroll
                for (int m = 0; m < NT; ++m)
                    if (m < p.M)
                        store_out(p.out, p.out_dtype, int64_t(m) * p.N + int64_t(b) * kRows + row, sum[m]);
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kTmemCols));
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

// Token tile = the MMA N (M=128 UMMA needs N % 16 == 0).  A unit needs one accumulator
// per group-sized piece of its block (blk/g), and TMEM holds 256/NT of them.
int nt_for(int64_t m, int64_t g, int bits) {
    const int64_t blk = bits == 4 ? 256 : 128;
    const int64_t per_unit = g >= blk ? 1 : blk / g;
    int nt = m <= 16 ? 16 : m <= 32 ? 32 : 64;
    while (nt > 16 && 256 / nt < per_unit) nt /= 2;
    return nt;
}

// Cluster split-K when the row-blocks are few (at most half the SMs): S CTAs per row-block,
// S <= 8 (portable cluster), S <= k-blocks.  0/1 = stream-K.  RTNQ_WGEMM_CTAS (an explicit
// stream-K grid, used by the split-invariance tests) or RTNQ_WGEMM_CLUSTER=0 disable it.
int cluster_size_for(int64_t NB, int64_t KBLK) {
    if (std::getenv("RTNQ_WGEMM_CTAS")) return 1;
    if (const char* e = std::getenv("RTNQ_WGEMM_CLUSTER"))
        if (std::atoi(e) == 0) return 1;
    const int sms = sm_count();
    if (NB * 2 > sms) return 1;
    int S = int(sms / NB);
    S = S > 8 ? 8 : S;
    S = S > KBLK ? int(KBLK) : S;
    return S < 2 ? 1 : S;
}

int ctas_for(int64_t U) {
    int G = sm_count();  // persistent: one CTA per SM (it owns all 512 TMEM columns)
    if (const char* e = std::getenv("RTNQ_WGEMM_CTAS")) G = std::atoi(e);
    if (G < 1) G = 1;
    return int(U < G ? U : G);
}

template <int BITS, int AT, int NT, bool PROF>
cudaError_t launch_t(const Params& p_in, cudaStream_t st, bool pdl) {
    using GG = Geo<BITS, NT>;
    auto kern = wgemm_tc_kernel<BITS, AT, NT, PROF>;
    static unsigned long long configured = 0;  // per device
    static int max_clusters_dev[64][9] = {};
    int* max_clusters = max_clusters_dev[current_device_index()];  // per cluster size: clusters resident at once
    if (!(configured & current_device_bit())) {
        cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, GG::SMEM);
        if (e != cudaSuccess) return e;
        configured |= current_device_bit();
    }
    Params p = p_in;
    // cluster split-K only if all NB clusters are resident at once; else a smaller cluster
    while (p.csize > 1) {
        int& mc = max_clusters[p.csize];
        if (mc == 0) {
            cudaLaunchConfig_t q{};
            q.gridDim = dim3(unsigned(p.NB * p.csize));
            q.blockDim = dim3(kThreads);
            q.dynamicSmemBytes = GG::SMEM;
            cudaLaunchAttribute ca;
            ca.id = cudaLaunchAttributeClusterDimension;
            ca.val.clusterDim.x = unsigned(p.csize);
            ca.val.clusterDim.y = ca.val.clusterDim.z = 1;
            q.attrs = &ca;
            q.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&mc, kern, &q) != cudaSuccess || mc < 1) mc = -1;
            cudaGetLastError();
        }
        if (mc >= p.NB) break;
        --p.csize;
    }
    if (p.csize > 1) p.G = p.NB * p.csize;
    else p.csize = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(p.G));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = GG::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (p.csize > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = unsigned(p.csize);
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

template <int BITS, int AT>
cudaError_t launch_bits(const Params& p, int nt, cudaStream_t st, bool pdl) {
    if (p.debug & 32) {
        switch (nt) {
            case 16: return launch_t<BITS, AT, 16, true>(p, st, pdl);
            case 32: return launch_t<BITS, AT, 32, true>(p, st, pdl);
            default: return launch_t<BITS, AT, 64, true>(p, st, pdl);
        }
    }
    switch (nt) {
        case 16: return launch_t<BITS, AT, 16, false>(p, st, pdl);
        case 32: return launch_t<BITS, AT, 32, false>(p, st, pdl);
        default: return launch_t<BITS, AT, 64, false>(p, st, pdl);
    }
}

}  // namespace tc

extern "C" int rtnq_wgemm_debug_read(void* host, size_t bytes, int reset) {
    if (bytes > sizeof(tc::g_wgemm_dbg)) bytes = sizeof(tc::g_wgemm_dbg);
    if (cudaMemcpyFromSymbol(host, tc::g_wgemm_dbg, bytes) != cudaSuccess) return 1;
    if (reset) {
        static unsigned long long zeros[1024 * 64];
        if (cudaMemcpyToSymbol(tc::g_wgemm_dbg, zeros, sizeof(zeros)) != cudaSuccess) return 1;
    }
    return 0;
}

const char* wgemm_unsupported(int64_t m, int64_t n, int64_t k, int bits, int64_t g, int a_dtype) {
    (void)m;
    (void)n;
    if (a_dtype != RTNQ_BF16 && a_dtype != RTNQ_F16) return "activations must be bf16 or f16";
    if (k % 8 != 0) return "k must be a multiple of 8 for the tensor-core path";
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
    const int64_t U = NB * ((k + 63) / 64 > 0 ? (k + 63) / 64 : 1);
    size_t part = 0;
    for (int nt : {16, 32, 64}) {  // every tile a call may launch
        if (nt > tc::nt_for(m, g, bits)) break;
        const int G = tc::ctas_for(U);
        const size_t need = size_t(G) * 2 * tc::kRows * nt * sizeof(float);
        part = need > part ? need : part;
    }
    return kCounterBytes + part;
}

// Activations [m][k] viewed as a 3-D tensor (8 elements, token, k-chunk) so one TMA box
// {8, nt, chunks per unit} lands in shared memory as [k-chunk][token][16 B] -- UMMA K-major core
// matrices.  Tokens >= m and chunks past k are out of bounds and arrive as zeros.
static cudaError_t encode_act_map(CUtensorMap* map, const void* a, int a_dtype, int64_t m,
                                  int64_t k, int nt, int chunks) {
    const cuuint64_t dims[3] = {8, cuuint64_t(m), cuuint64_t(k / 8)};
    const cuuint64_t strides[2] = {cuuint64_t(k * 2), 16};
    const cuuint32_t box[3] = {8, cuuint32_t(nt), cuuint32_t(chunks)};
    const cuuint32_t estr[3] = {1, 1, 1};
    // the driver entry point is fetched through the runtime, so the library does not link
    // libcuda (it must load on a machine without a driver, e.g. for the CPU test suite)
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<EncodeFn>(fn);
    }();
    if (!encode) return cudaErrorNotSupported;
    const CUresult r = encode(
        map, a_dtype == RTNQ_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
        3, const_cast<void*>(a), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t launch_wgemm(const WgemmArgs& A, cudaStream_t st) {
    tc::Params p{};
    p.codes = A.codes;
    p.scales = A.scales;
    p.N = A.n;
    p.K = A.k;
    p.NB = int((A.n + tc::kRows - 1) / tc::kRows);
    p.KBLK = int((A.k + 63) / 64);
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
    const int nt_max = tc::nt_for(A.m, A.g, A.bits);
    for (int64_t m0 = 0; m0 < A.m; m0 += nt_max) {  // one pass per token tile
        p.M = int(A.m - m0 < nt_max ? A.m - m0 : nt_max);
        p.out = static_cast<char*>(A.out) + m0 * A.n * esz;
        const int nt = tc::nt_for(p.M, A.g, A.bits);
        p.m0 = int(m0);
        if (cudaError_t e = encode_act_map(&p.tmap_a, A.a, A.a_dtype, A.m, A.k, nt,
                                             A.bits == 4 ? 32 : 16)) return e;
        p.G = tc::ctas_for(p.U);
        p.csize = tc::cluster_size_for(p.NB, p.KBLK);
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
