// wgemm_i4.cu -- W4A16 group-128 linear on tcgen05.mma.kind::i8.
//
// out[m][n] = sum_g S[n][g] * sum_{k in g} a[m][k] * code[n][k]     (gemm.hpp:18-27, g = 128)
//
// Weights: RTNQ_NATIVE_I4 (common.cuh), one 8 KiB nibble tile per 128 rows x one group.  Each
// byte carries two codes as 4-bit two's complement, so the expansion to the s8 A operand is
// three ALU ops per 4 bytes and needs no offset correction:
//   hi = w & 0xF0F0F0F0          -> 16 * code(r, p)        (k = p)
//   lo = (w << 4) & 0xF0F0F0F0   -> 16 * code(r, 64 + p)   (k = 64 + p)
// The factor 16 is folded into the group scale.
//
// Activations: the three exact int8 planes of int8_mma.cuh (a = 2^s (P0 + P1/2^7 + P2/2^14)),
// the s8 B operand.  PT tokens per launch chunk (5, 10, 16, 32 or 64): B row p * PT + t is plane
// p of token t, N = 3 * PT rounded up to 16 (the rows past 3 * PT are zero).  Small batches
// get small N: the epilogue reads back N accumulator columns per group, and TMEM reads (64 B
// per clock per SM) are the budget that binds this kernel (A reads of the MMA + readback).
//
// Each group has its own int32 accumulator in TMEM (a ring of NS slots): the epilogue reads
// it once, applies S[n][g] / 16 * 2^s and adds into per-row float accumulators.
//
// Warp roles (384 threads):
//   warp 0      TMA producer: codes (contiguous tiles) + the group scales of the stage
//   warp 2      TMA producer: activation planes (after the planes kernel, PDL)
//   warp 1      MMA issuer: 4 x (M128, N, K32) per group, A = expanded tile (TMEM)
//   warps 8-11  expansion: nibble tile (smem) -> registers -> tcgen05.st into a TMEM A slot
//               (32 columns of 4 s8 each per row); group scale / 16 into the scale ring
//
// Shared-memory bandwidth (128 B/clk/SM) is the budget that shapes this: per 8 KiB group the
// smem carries the TMA writes (codes 8 KiB + planes N*128) and the reads (codes 8 KiB +
// planes by the MMA).  An expanded A tile staged in smem would add 32 KiB more per group;
// in TMEM it costs no smem bandwidth at all.
//   warps 4-7   epilogue: per-group TMEM reads, scaling, stream-K / cluster output
//   warps 12-15 (batch >= 16) a second epilogue warpgroup: the other half of the tokens
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "int8_mma.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {
namespace i4 {
using namespace imma;

constexpr int kKB = 128;              // k-block = one quantization group = one tile
constexpr int kTile = kRows * 64;     // 8 KiB of nibbles
constexpr int kEpi0 = 4, kExp0 = 8, kEpiB0 = 12;  // epilogue warpgroup B (EH = 2): warps 12-15

struct Params {
    CUtensorMap tmap_p;      // planes [3][M][K] s8, box {128, PT, 3}, SWIZZLE_128B
    const uint8_t* codes;    // RTNQ_NATIVE_I4
    const uint16_t* scales;  // f16, native order [row-block][group][rows8]
    const int32_t* texp;     // [M] token exponents s
    void* out;
    float* partials;
    int* counters;
    int64_t N, K;
    int M, Mtot, m0, NB, KBLK, U, G, csize, out_dtype;
    int debug;
    imma::OwnPlanes own;  // own.a != nullptr: this launch computes its tokens' planes itself
    int8_t* planes_w;     // ... into this [3][Mtot][K] buffer (the TMA source), exponents into texp
    PeerOut peer;         // tensor parallel: output pushed into every rank's slot (world > 0)
};

template <int PT, int BITS = 4>
struct Geo {
    // W4: one 8 KiB NATIVE_I4 nibble tile per 128 rows x group, expanded to s8 in TMEM;
    // W8 group 128: one 16 KiB NATIVE_I8 tile (pre-swizzled s8, the MMA reads it from smem)
    static constexpr int TILE = BITS == 4 ? kTile : kRows * 128;
    static constexpr int ACC = (PT + 3) / 4 * 4;            // per-row accumulators (float4 I/O)
    static constexpr int DN = (3 * PT + 15) / 16 * 16;      // accumulator columns per group
    static constexpr int BOX_BYTES = 3 * PT * 128;          // one group's planes box
    static constexpr int PLANE_BYTES = DN * 128;            // ... its smem slot (zero rows past it)
    // groups (tiles) per stage: every stage costs each role a fixed few hundred cycles of
    // barrier hand-offs (measured: the stage period stays ~1000 cycles with all memory traffic
    // switched off), so batch <= 16 moves four groups (32 KiB of codes) per stage
#ifndef RTNQ_I4_TPS16
#define RTNQ_I4_TPS16 4
#endif
    static constexpr int TPS = BITS == 8 ? (PT <= 32 ? 2 : 1) : PT <= 16 ? RTNQ_I4_TPS16 : PT <= 32 ? 2 : 1;
    static constexpr int CODE_OFF = TPS * PLANE_BYTES;      // planes first: 1024-aligned
    static constexpr int SC_OFF = CODE_OFF + TPS * TILE;
    static constexpr int STAGE_BYTES = (SC_OFF + TPS * 256 + 1023) / 1024 * 1024;
    // epilogue warpgroups: two (each with half of the tokens) from 16 tokens up
#ifndef RTNQ_I4_EH
#define RTNQ_I4_EH 2
#endif
    static constexpr int EH = PT >= 16 ? RTNQ_I4_EH : 1;
    static constexpr int THREADS = EH == 2 ? 512 : 384;
    // The A operand of a group is 4 k-steps of 32 codes.  The first KT come from TMEM (tcgen05.st
    // by the expansion; the MMA's A reads share the 64 B/clk TMEM read port with the epilogue's
    // accumulator readback), the rest from a 128B-swizzled smem tile (128 B/clk smem port,
    // shared with TMA and the planes).  KT balances the two ports for the batch size.
    static constexpr int KT = 4;
    // expanded A slots (groups); TMEM = AS * 32 A columns + NS * DN accumulator columns
    static constexpr int AS = BITS == 8 ? 0 : TPS == 4 ? (PT <= 10 ? 8 : 4) : PT <= 16 ? 6 : PT <= 32 ? 4 : 2;
    static constexpr int AP = BITS == 8 ? 1 : AS / TPS;     // ... in stage-sized slots (W8: unused)
    static constexpr int A_SMEM = KT < 4 ? kRows * 128 : 0;  // smem A tile per slot (16 KiB)
#ifndef RTNQ_I4_SMEM_KB
#define RTNQ_I4_SMEM_KB 212
#endif
    static constexpr int STAGES_FIT = ((PT <= 16 ? RTNQ_I4_SMEM_KB : 212) * 1024 - AS * A_SMEM) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_FIT > 12 ? 12 : STAGES_FIT;
    static constexpr int A_OFF = STAGES * STAGE_BYTES;      // smem A slots (1024-aligned)
    static constexpr int A_COL = 512 - AS * KT * 8;         // TMEM A slots: 8 columns per k-step
    static constexpr int NS_FIT = A_COL / DN;
    static constexpr int NS = NS_FIT > 12 ? 12 : NS_FIT;    // TMEM group accumulators
    static constexpr int NP = NS / TPS;                     // ... in stage-sized slots
    static constexpr int BAR_OFF = A_OFF + AS * A_SMEM;
    static constexpr int SR_OFF = BAR_OFF + 1024;           // [NS][128] f32 group scale / 16
    static constexpr int SMEM = SR_OFF + NS * kRows * 4 + 1024;
    static constexpr int MAXC_FIT = 1 + STAGES * STAGE_BYTES / (ACC * kRows * 4);
    static constexpr int MAXC = MAXC_FIT > 8 ? 8 : MAXC_FIT;
    static_assert(STAGES >= 3, "");
    static_assert(SMEM <= 227 * 1024, "");
};

__device__ unsigned long long g_i4_dbg[1024 * 16];  // profiling (debug & 64: globaltimer stamps)
// profiling (debug & 512): per-stage clock64 timeline of CTA p.debug >> 16 -- [stage][event]:
// 0 codes TMA issued, 1 MMAs issued (before the commits), 2 expansion start, 3 expansion done, 4 MMA start,
// 5 MMA issued, 6 epilogue start, 7 epilogue done
__device__ long long g_i4_tl[64 * 16];
#define I4_TL(si, ev) \
    if ((dbg_ & 512) && c == (dbg_ >> 16) && (si) < 64 && lane == 0) g_i4_tl[(si) * 16 + (ev)] = clock64() - tl0

// A from TMEM (32-bit columns of 4 s8 along K), B from shared memory
__device__ __forceinline__ void mma_i8_ts_elect(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc,
                                                uint32_t acc) {
    asm volatile(
        "{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
        "r"(a), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}
// Plain TS issue (the caller is the one elected thread).
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
        "r"(a), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
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
__device__ __forceinline__ void elect_bulk_tx(void* dst, const void* src, uint64_t* b, uint32_t bytes) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n}\n" ::"r"(
            su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(b))
        : "memory");
}

// debug & 32: per-role blocked/busy cycles (lane 0 of the first warp of each role)
#define I4_T0() const long long _t0 = (dbg_ & 32) ? clock64() : 0
#define I4_ACC(var) if (dbg_ & 32) var += clock64() - _t0

// PEER: the output goes to the tensor-parallel peers' slots (a separate instantiation: the peer
// store path compiled into the plain kernel measured +1-2.5 us per launch, never executed)
template <int PT, int BITS, bool PEER>
__global__ void __launch_bounds__(Geo<PT, BITS>::THREADS, 1) wgemm_i4_kernel(const __grid_constant__ Params p) {
#ifdef RTNQ_KERNEL_DEBUG
    const int dbg_ = p.debug;  // profiling knobs (scratch/*prof*.py, *tl.py)
#else
    constexpr int dbg_ = 0;  // compiled out: even disabled, the checks cost a few % per launch
#endif
    using GG = Geo<PT, BITS>;
    constexpr int NT = GG::ACC;
    constexpr int STAGES = GG::STAGES, DN = GG::DN, AP = GG::AP, NP = GG::NP, TPS = GG::TPS, EH = GG::EH;
    extern __shared__ uint8_t smem_raw[];
    // align by indexing the __shared__ array (keeps the shared address space: LDS/STS, not
    // generic loads)
    uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + GG::BAR_OFF);  // [STAGES] TMA landed
    uint64_t* empty = full + STAGES;    // [STAGES] expansion (4) + MMA commit (1) done with it
    uint64_t* afull = empty + STAGES;   // [AP] a stage's expanded tiles ready (4 warps)
    uint64_t* aempty = afull + AP;      // [AP] MMA done reading them (commit)
    uint64_t* tfull = aempty + AP;      // [NP] a stage's group accumulators ready (commit)
    uint64_t* tfree = tfull + NP;       // [NP] epilogue has read them (4 warps)
    uint64_t* sfull = tfree + NP;       // [NP] their group scales in the scale ring (4 warps)
    uint64_t* go = sfull + NP;          // cluster split-K: leader ready for partials
    uint64_t* rfull = go + 1;           // cluster split-K: partials landed in the leader
    uint64_t* pub = rfull + 1;          // stream-K contributor partials stored (4 warps)
    uint64_t* pready = pub + 1;         // own planes: this launch's planes / exponents published
    uint32_t* tslot = reinterpret_cast<uint32_t*>(pready + 1);
    float* sring = reinterpret_cast<float*>(smem + GG::SR_OFF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, c = blockIdx.x;
    const long long tl0 = (dbg_ & 512) ? clock64() : 0;
    if ((dbg_ & 64) && threadIdx.x == 0) g_i4_dbg[c * 16 + 5] = gtime();

    int u0, u1;
    if (p.csize > 1) {
        const int b = c / p.csize, r = c % p.csize;
        u0 = b * p.KBLK + r * p.KBLK / p.csize;
        u1 = b * p.KBLK + (r + 1) * p.KBLK / p.csize;
    } else {
        u0 = int(int64_t(c) * p.U / p.G);
        u1 = int(int64_t(c + 1) * p.U / p.G);
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 2), mbar_init(&empty[s], 5);
        for (int i = 0; i < AP; ++i) mbar_init(&afull[i], 4), mbar_init(&aempty[i], 1);
        for (int i = 0; i < NP; ++i) mbar_init(&tfull[i], 1), mbar_init(&tfree[i], 4 * EH), mbar_init(&sfull[i], 4);
        mbar_init(go, 1), mbar_init(rfull, 1), mbar_init(pub, 4 * EH), mbar_init(pready, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if ((dbg_ & 512) && c == (dbg_ >> 16)) g_i4_tl[63 * 16 + 13] = clock64() - tl0;
    }
    if constexpr (GG::DN > 3 * PT) {  // B rows past 3 * PT: zero once, never written by TMA
        constexpr int PAD = (GG::DN - 3 * PT) * 128 / 16;  // uint4 per slot
        for (int i = threadIdx.x; i < STAGES * TPS * PAD; i += blockDim.x) {
            const int slot = i / PAD, k = i % PAD;
            uint8_t* dst = smem + (slot / TPS) * GG::STAGE_BYTES + (slot % TPS) * GG::PLANE_BYTES + 3 * PT * 128;
            reinterpret_cast<uint4*>(dst)[k] = make_uint4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            su32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        if ((dbg_ & 512) && c == (dbg_ >> 16) && lane == 0) g_i4_tl[63 * 16 + 14] = clock64() - tl0;
    }
    fence_before();
    __syncthreads();
    fence_after();
    if ((dbg_ & 512) && c == (dbg_ >> 16) && threadIdx.x == 0) g_i4_tl[63 * 16 + 15] = clock64() - tl0;
    if (p.csize > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    const uint32_t tmem = *tslot;
    asm volatile("griddepcontrol.launch_dependents;");
    if (p.own.a && warp >= kEpi0 && warp < kExp0 + 4) {
        // the epilogue + expansion warps (idle until the first weights land) compute this CTA's
        // share of the launch's activation planes (int8_mma.cuh, own_planes_produce)
        __shared__ float pred[8];
        if ((dbg_ & 512) && c == (dbg_ >> 16) && threadIdx.x == kEpi0 * 32) g_i4_tl[62 * 16 + 5] = clock64() - tl0;
        own_planes_produce(p.own, int(p.K), p.m0, p.M, p.Mtot, c, int(gridDim.x), p.planes_w,
                           const_cast<int32_t*>(p.texp), threadIdx.x - kEpi0 * 32, 256, 3, pred,
                           (dbg_ & 512) && c == (dbg_ >> 16) ? &g_i4_tl[61 * 16] : nullptr, tl0);
        if ((dbg_ & 512) && c == (dbg_ >> 16) && threadIdx.x == kEpi0 * 32) g_i4_tl[62 * 16 + 6] = clock64() - tl0;
    }

    // ===================== expansion: nibbles -> s8 (16 x code) in TMEM ===============
    // One handshake per stage (TPS groups): A pair slot xsi % AP, accumulator slot xsi % NP.
    // exp_step() expands one stage; run by warps 8-11.
    const int xrow = threadIdx.x - kExp0 * 32;  // one xrow of the tile per thread = TMEM lane
    const uint32_t sw_in = uint32_t((xrow >> 1) & 3);
    const uint32_t xlane_base = uint32_t((warp & 3) * 32) << 16;
    Cursor<TPS> xcu(u0, u1, p.KBLK);
    int xs = 0, xsi = 0;
    uint32_t xph = 0;
    long long x_full = 0, x_aempty = 0, x_tfree = 0, x_work = 0;
    auto exp_step = [&]() {
        const int n = xcu.chunk();
        const int slot0 = xcu.kb & (TPS - 1);
        const int64_t left = p.N - int64_t(xcu.b) * kRows;
        const int r8 = left >= kRows ? kRows : int((left + 7) / 8 * 8);
        const int ap = xsi % AP, np = xsi % NP;
        {
            I4_T0();
            mbar_wait(&full[xs], xph);
            I4_ACC(x_full);
        }
        if (warp == kExp0) I4_TL(xsi, 11);
        {
            I4_T0();
            if (BITS == 4 && xsi >= AP) mbar_wait(&aempty[ap], uint32_t(xsi / AP - 1) & 1u);
            I4_ACC(x_aempty);
        }
        if (warp == kExp0) I4_TL(xsi, 12);
        {
            I4_T0();
            if (xsi >= NP) mbar_wait(&tfree[np], uint32_t(xsi / NP - 1) & 1u);
            I4_ACC(x_tfree);
        }
        const long long _tw = (dbg_ & 32) ? clock64() : 0;
        if (warp == kExp0) I4_TL(xsi, 2);
        const uint8_t* st = smem + xs * GG::STAGE_BYTES;
        if (BITS == 8) {
            // W8: the MMA reads the s8 tiles from shared memory; only the group scales move
#pragma unroll
            for (int j = 0; j < TPS; ++j) {
                if (j >= n) break;
                const uint16_t* sc = reinterpret_cast<const uint16_t*>(st + GG::SC_OFF + slot0 * 256) + j * r8;
                sring[(np * TPS + j) * kRows + xrow] = xrow < r8 ? __half2float(__ushort_as_half(sc[xrow])) : 0.0f;
            }
        } else if (!(dbg_ & 65536)) {
            // two groups at a time: their code loads first (latency overlap), then expand and store
            constexpr int JP = TPS < 2 ? TPS : 2;
#pragma unroll
            for (int j0 = 0; j0 < TPS; j0 += JP) {
                if (j0 >= n) break;
                uint4 w[JP][4];
#pragma unroll
                for (int jj = 0; jj < JP; ++jj)
                    if (j0 + jj < n) {
                        const uint8_t* src = st + GG::CODE_OFF + (slot0 + j0 + jj) * GG::TILE + xrow * 64;
#pragma unroll
                        for (uint32_t q = 0; q < 4; ++q)
                            w[jj][q] = *reinterpret_cast<const uint4*>(src + ((q ^ sw_in) << 4));
                    }
                float scv[JP];
#pragma unroll
                for (int jj = 0; jj < JP; ++jj) {
                    const uint16_t* sc =
                        reinterpret_cast<const uint16_t*>(st + GG::SC_OFF + slot0 * 256) + (j0 + jj) * r8;
                    scv[jj] = (j0 + jj < n && xrow < r8) ? __half2float(__ushort_as_half(sc[xrow])) * 0.0625f : 0.0f;
                }
#pragma unroll
                for (int jj = 0; jj < JP; ++jj) {
                    const int j = j0 + jj;
                    if (j >= n) break;
                    uint32_t v[32];  // TMEM column c of this xrow holds k = 4c .. 4c + 3
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q) {
                        const uint32_t ww[4] = {w[jj][q].x, w[jj][q].y, w[jj][q].z, w[jj][q].w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            v[4 * q + e] = ww[e] & 0xF0F0F0F0u;               // k = 16q + 4e ..
                            v[16 + 4 * q + e] = (ww[e] & 0x0F0F0F0Fu) * 16u;  // k = 64 + 16q + 4e ..
                        }
                    }
                    const int slot = ap * TPS + j;
                    static_assert(GG::KT == 4, "A operand entirely from TMEM");
                    if (!(dbg_ & 8)) {
                        tmem_st32(tmem + xlane_base + uint32_t(GG::A_COL + slot * 32), v);
                    } else if (v[0] == 0x12345u) {
                        g_i4_dbg[0] = v[1] + v[31];  // keep the expansion alive
                    }
                    sring[(np * TPS + j) * kRows + xrow] = scv[jj];
                }
            }
        }
        if constexpr (BITS == 4) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[ap]), mbar_arrive(&sfull[np]), mbar_arrive(&empty[xs]);
        if (warp == kExp0) I4_TL(xsi, 3);
        if (dbg_ & 32) x_work += clock64() - _tw;
        xcu.advance(n);
        ++xsi;
        if (++xs == STAGES) xs = 0, xph ^= 1u;
    };
    if (warp == 0 || warp == 2) {
        // ===================== producers: warp 0 codes + scales, warp 2 planes ============
        const bool codes = warp == 0;
        Cursor<TPS> cu(u0, u1, p.KBLK);
        int s = 0;
        uint32_t ph = 0;
        if (!codes) {
            if (p.own.a) {  // planes computed by this launch's CTAs
                own_planes_acquire(p.own, p.M, int(gridDim.x), int(p.K));
                if (lane == 0) mbar_arrive(pready);
            } else {
                asm volatile("griddepcontrol.wait;" ::: "memory");  // planes kernel / fused producer
            }
        }
        long long w_empty = 0;
        if ((dbg_ & 512) && c == (dbg_ >> 16) && lane == 0) g_i4_tl[62 * 16 + 13 + codes] = clock64() - tl0;
        for (int i = 0; cu.more(); ++i) {
            const int n = cu.chunk();
            if (i >= STAGES) {
                I4_T0();
                mbar_wait(&empty[s], ph ^ 1u);
                I4_ACC(w_empty);
            }
            uint8_t* st = smem + s * GG::STAGE_BYTES;
            const int slot0 = cu.kb & (TPS - 1);
            if ((dbg_ & 2) || (codes && (dbg_ & 8192)) || (!codes && (dbg_ & 4096))) {
                elect_arrive(&full[s]);  // profiling: no copy
            } else if (codes) {
                // the row-block's rows padded to 8: the stride of its native scale groups
                const int64_t left = p.N - int64_t(cu.b) * kRows;
                const int r8 = left >= kRows ? kRows : int((left + 7) / 8 * 8);
                if (i == 0 && (dbg_ & 512) && c == (dbg_ >> 16) && lane == 0) g_i4_tl[62 * 16 + 10] = clock64() - tl0;
                elect_expect(&full[s], uint32_t(n) * (GG::TILE + uint32_t(r8) * 2));
                if (i == 0 && (dbg_ & 512) && c == (dbg_ >> 16) && lane == 0) g_i4_tl[62 * 16 + 11] = clock64() - tl0;
                elect_bulk_tx(st + GG::CODE_OFF + slot0 * GG::TILE,
                              p.codes + (int64_t(cu.b) * p.KBLK + cu.kb) * GG::TILE, &full[s], uint32_t(n) * GG::TILE);
                if (i == 0 && (dbg_ & 512) && c == (dbg_ >> 16) && lane == 0) g_i4_tl[62 * 16 + 12] = clock64() - tl0;
                elect_bulk_tx(st + GG::SC_OFF + slot0 * 256,
                              p.scales + int64_t(cu.b) * kRows * p.KBLK + int64_t(cu.kb) * r8, &full[s],
                              uint32_t(n * r8 * 2));
            } else {
                elect_expect(&full[s], uint32_t(n) * GG::BOX_BYTES);
                for (int j = 0; j < n; ++j)
                    elect_tma3d_tx(st + (slot0 + j) * GG::PLANE_BYTES, &p.tmap_p, (cu.kb + j) * kKB, p.m0, 0,
                                   &full[s]);
            }
            if (codes) I4_TL(i, 0);
            cu.advance(n);
            if (++s == STAGES) s = 0, ph ^= 1u;
        }
        if ((dbg_ & 32) && lane == 0 && codes) g_i4_dbg[c * 16] = w_empty;
    } else if (warp == 3) {
        // ===================== stream-K publisher =====================
        if (p.csize == 1 && u0 < u1 && u0 % p.KBLK != 0) {
            mbar_wait(pub, 0);
            if (lane == 0) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(p.counters + u0 / p.KBLK) : "memory");
            }
        }
    } else if (warp >= kExp0 && warp < kExp0 + 4) {
        while (xcu.more()) exp_step();
        if ((dbg_ & 32) && threadIdx.x == kExp0 * 32) {
            g_i4_dbg[c * 16 + 2] = x_full, g_i4_dbg[c * 16 + 3] = x_aempty;
            g_i4_dbg[c * 16 + 4] = x_tfree, g_i4_dbg[c * 16 + 6] = x_work;
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (warp-uniform, one elected lane issues) ==========
        // D s32, A s8 (16 x codes, TMEM), B s8 (planes, smem), M = 128, N = DN
        constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                   (uint32_t(DN >> 3) << 17) | (uint32_t(kRows >> 4) << 24);
        constexpr uint64_t kHi = (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) |
                                 (2ull << 61);  // K-major SWIZZLE_128B, SBO = 1024
        const uint32_t base = su32(smem) >> 4;
        Cursor<TPS> cu(u0, u1, p.KBLK);
        int s = 0, si = 0;
        uint32_t ph = 0;
        long long m_full = 0, m_afull = 0, m_tfree = 0, m_issue = 0;
        while (cu.more()) {
            const int n = cu.chunk();
            const int slot0 = cu.kb & (TPS - 1);
            const int ap = si % AP, np = si % NP;
            {
                I4_T0();
                mbar_wait(&full[s], ph);  // the planes of this stage
                I4_ACC(m_full);
            }
            I4_TL(si, 8);
            if ((dbg_ & 64) && si == 0 && lane == 0) g_i4_dbg[c * 16 + 6] = gtime();
            if (BITS == 4) {
                I4_T0();
                mbar_wait(&afull[ap], uint32_t(si / AP) & 1u);
                I4_ACC(m_afull);
            }
            I4_TL(si, 9);
            {
                I4_T0();
                if (si >= NP) mbar_wait(&tfree[np], uint32_t(si / NP - 1) & 1u);
                I4_ACC(m_tfree);
            }
            fence_after();
            I4_TL(si, 4);
            const long long _ti = (dbg_ & 32) ? clock64() : 0;
            const uint32_t stage_lo = base + uint32_t(s * GG::STAGE_BYTES >> 4);
            // the whole warp issues the stage's MMAs (one elected lane, warp-uniform asm blocks of
            // a group's 4 k-steps) and their commits
            static_assert(GG::KT == 4, "A operand entirely from TMEM");
            if (!(dbg_ & 4)) {
                for (int j = 0; j < n; ++j) {
                    const uint32_t blo = stage_lo + uint32_t((slot0 + j) * GG::PLANE_BYTES >> 4);
                    const uint32_t d = tmem + uint32_t((np * TPS + j) * DN);
                    if constexpr (BITS == 4) {
                        const uint32_t a = tmem + uint32_t(GG::A_COL + (ap * TPS + j) * GG::KT * 8);
                        mma4_i8_ts_warp(d, a, kHi | blo, idesc, 0u);
                    } else {  // the pre-swizzled 128 x 128 s8 tile: K-major SWIZZLE_128B, like the planes
                        const uint32_t alo = stage_lo + uint32_t((GG::CODE_OFF + (slot0 + j) * GG::TILE) >> 4);
                        mma2_i8_ss_warp(d, kHi | alo, kHi | blo, idesc, 0u);
                        mma2_i8_ss_warp(d, kHi | (alo + 4), kHi | (blo + 4), idesc, 1u);
                    }
                }
            }
            I4_TL(si, 1);
            commit_elect(&aempty[ap]);
            commit_elect(&tfull[np]);
            commit_elect(&empty[s]);
            __syncwarp();
            I4_TL(si, 5);
            if (dbg_ & 32) m_issue += clock64() - _ti;
            cu.advance(n);
            ++si;
            if (++s == STAGES) s = 0, ph ^= 1u;
        }
        if ((dbg_ & 32) && lane == 0)
            g_i4_dbg[c * 16 + 8] = m_full, g_i4_dbg[c * 16 + 9] = m_afull, g_i4_dbg[c * 16 + 10] = m_tfree,
            g_i4_dbg[c * 16 + 1] = m_issue;
    } else if (warp >= kEpi0) {
        // ===================== epilogue =====================
        // EH warpgroups (warps 4-7; and 12-15 when EH = 2), each owning NH of the tokens: a
        // warpgroup's TMEM loads of a group are 3 planes x NH columns, so the two warpgroups'
        // load latencies overlap (measured: the epilogue's ~200-cycle tcgen05.ld round trips bound
        // the batch-16 stage period with one warpgroup, profiles/r2_w4_limiter.md)
        constexpr int EH = GG::EH, NH = NT / EH;
        const int eh = warp >= kEpiB0 ? 1 : 0, t0 = eh * NH;
        const int q = warp & 3, row = q * 32 + lane, et = threadIdx.x - (eh ? kEpiB0 : kEpi0) * 32;
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        __shared__ float pow_s[NT];  // 2^s per token, 0 for padding tokens
        if (eh == 0) {
            if (p.own.a) mbar_wait(pready, 0);  // texp published by this launch
            else asm volatile("griddepcontrol.wait;" ::: "memory");  // texp from the planes producer
            for (int t = et; t < NT; t += 128) pow_s[t] = t < p.M ? ldexpf(1.0f, __ldg(p.texp + p.m0 + t)) : 0.0f;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(128 * EH) : "memory");
        // the output: local, or (tensor parallel) this rank's slot of every rank's buffer; the
        // peer round is read once the previous grid is done (warpgroup A waited for it above)
        int pe = 0;
        if constexpr (PEER) pe = peer_round(p.peer);
        auto emit_out = [&](int m, int64_t col, float v) {
            if constexpr (PEER) peer_store(p.peer, pe, int64_t(p.m0 + m) * p.N + col, v);
            else store_out(p.out, p.out_dtype, int64_t(m) * p.N + col, v);
        };
        float acc[NH];
#pragma unroll
        for (int t = 0; t < NH; ++t) acc[t] = 0.0f;
        Cursor<TPS> cu(u0, u1, p.KBLK);
        int si = 0, seg_kb0 = cu.kb;
        long long e_wait = 0, e_work = 0, e_ld = 0;
        const long long e_t0 = clock64();
        // one stage of this warpgroup's epilogue
        auto epi_step = [&]() {
        const int n = cu.chunk();
        const bool seg_end = cu.seg_end(n);
        const int b = cu.b;
        const int np = si % NP;
        {
            I4_T0();
            mbar_wait(&sfull[np], uint32_t(si / NP) & 1u);
            mbar_wait(&tfull[np], uint32_t(si / NP) & 1u);
            I4_ACC(e_wait);
        }
        const long long _tw = (dbg_ & 32) ? clock64() : 0;
        if (warp == kEpi0) I4_TL(si, 6);
        fence_after();
        float scg[TPS];
#pragma unroll
        for (int j = 0; j < TPS; ++j) scg[j] = j < n ? sring[(np * TPS + j) * kRows + row] : 0.0f;
        // token chunks of CH: plane p3 of token t is accumulator column p3 * PT + t
        // (the accumulators of padding tokens past PT are never combined)
        constexpr int NHR = EH == 2 ? NH : PT;  // real tokens of this warpgroup
        constexpr int CH = NHR >= 16 ? 16 : NHR;
        constexpr bool SPLIT = PT >= 16;           // planes loaded separately (CH columns each)
        constexpr int LDC = SPLIT ? CH : GG::DN;   // columns per load buffer
        // TMEM loads in batches of GL groups per tcgen05.wait::ld, double-buffered when the
        // registers allow
        constexpr int PGR = SPLIT ? 3 * CH : LDC;  // registers per group of a chunk
#ifndef RTNQ_I4_GL
#define RTNQ_I4_GL 1
#endif
        // (measured: one group per round trip, double-buffered, is the fastest at batch 1 and 16;
        // RTNQ_I4_GL=4 batches up to four groups per round trip)
        constexpr int GL = RTNQ_I4_GL >= 4 && TPS >= 4 && 4 * PGR <= 96 ? 4
                           : RTNQ_I4_GL >= 2 && TPS >= 2 && 2 * PGR <= 96 ? 2 : 1;
        constexpr int NBT = (TPS + GL - 1) / GL;
        constexpr int NB = NBT > 1 && 2 * GL * PGR <= 96 ? 2 : 1;
#pragma unroll
        for (int jj = 0; jj < NHR; jj += CH) {
            if (dbg_ & 131072) break;
            uint32_t d[NB][GL][SPLIT ? 3 : 1][LDC];
            auto load = [&](int bi) {
#pragma unroll
                for (int g = 0; g < GL; ++g) {
                    const int j = bi * GL + g;
                    if (j >= n) break;
                    const uint32_t ta = tmem + lane_base + uint32_t((np * TPS + j) * DN + t0 + jj);
                    uint32_t(&dd)[SPLIT ? 3 : 1][LDC] = d[bi % NB][g];
                    if (!(dbg_ & 16)) {
                        if constexpr (SPLIT) {
#pragma unroll
                            for (int p3 = 0; p3 < 3; ++p3) {
                                if constexpr (CH == 16) ld16(ta + p3 * PT, dd[p3]);
                                else ld8(ta + p3 * PT, dd[p3]);
                            }
                        } else {
#pragma unroll
                            for (int h = 0; h < GG::DN / 16; ++h) ld16(ta + 16 * h, dd[0] + 16 * h);
                        }
                    } else {
#pragma unroll
                        for (int e = 0; e < LDC; ++e)
#pragma unroll
                            for (int q3 = 0; q3 < (SPLIT ? 3 : 1); ++q3) dd[q3][e] = uint32_t(row + e);
                    }
                }
            };
            auto combine = [&](int bi) {
#pragma unroll
                for (int g = 0; g < GL; ++g) {
                    const int j = bi * GL + g;
                    if (j >= n) break;
                    const uint32_t(&dd)[SPLIT ? 3 : 1][LDC] = d[bi % NB][g];
                    // two tokens per packed FP32 FMA pair (__ffma2_rn: the same two roundings as
                    // scalar FMAs; measured -1 to -3 % per launch: the epilogue is issue-bound)
                    auto plane = [&](int p3, int e) -> uint32_t {
                        if constexpr (SPLIT) return dd[p3][e];
                        else return dd[0][(p3 * PT + e) % LDC];
                    };
                    const float2 c14 = make_float2(6.103515625e-05f, 6.103515625e-05f);
                    const float2 sg = make_float2(scg[j], scg[j]);
#pragma unroll
                    for (int e = 0; e + 1 < CH; e += 2) {
                        const float2 x0 = make_float2(float(int32_t(plane(0, e))), float(int32_t(plane(0, e + 1))));
                        const float2 x12 = make_float2(float(int32_t(plane(1, e)) * 128 + int32_t(plane(2, e))),
                                                       float(int32_t(plane(1, e + 1)) * 128 + int32_t(plane(2, e + 1))));
                        const float2 r = __ffma2_rn(__ffma2_rn(x12, c14, x0), sg, make_float2(acc[jj + e], acc[jj + e + 1]));
                        acc[jj + e] = r.x, acc[jj + e + 1] = r.y;
                    }
                    if constexpr ((CH & 1) == 0) continue;
#pragma unroll
                    for (int e = CH & ~1; e < CH; ++e) {  // odd tail; 2^s per token at the segment end
                        uint32_t u0v, u1v, u2v;
                        if constexpr (SPLIT) {
                            u0v = dd[0][e], u1v = dd[SPLIT ? 1 : 0][e], u2v = dd[SPLIT ? 2 : 0][e];
                        } else {
                            u0v = dd[0][e], u1v = dd[0][(PT + e) % LDC], u2v = dd[0][(2 * PT + e) % LDC];
                        }
                        // planes 1 and 2 combined exactly in int32 (|D1 * 128 + D2| < 2^28); D0
                        // (< 2^21) converts exactly, D12's rounding (2^-24 of it) sits 2^-30 below
                        // D0 after the 2^-14 weight
                        const float x0 = float(int32_t(u0v));
                        const float x12 = float(int32_t(u1v) * 128 + int32_t(u2v));
                        acc[jj + e] = fmaf(fmaf(x12, 6.103515625e-05f, x0), scg[j], acc[jj + e]);
                    }
                }
            };
            if (n > 0) {
                load(0);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (dbg_ & 32) {
                    const long long t = clock64();
                    e_ld += t - _tw;
                }
#pragma unroll
                for (int bi = 0; bi < NBT; ++bi) {
                    if (bi * GL >= n) break;
                    const bool next = (bi + 1) * GL < n;
                    if (NB == 2 && next) load(bi + 1);
                    combine(bi);
                    if (NB == 1 && next) load(bi + 1);
                    if (next) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                }
            }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tfree[np]);
        if (warp == kEpi0) I4_TL(si, 7);
        if (dbg_ & 32) e_work += clock64() - _tw;
        ++si;
        if (seg_end) {
#pragma unroll
            for (int t = 0; t < NH; ++t) acc[t] *= pow_s[t0 + t];
            const int kbe = cu.kb + n;
            const bool sole = seg_kb0 == 0 && kbe == p.KBLK;
            const int rows = min(kRows, int(p.N - int64_t(b) * kRows));
            const int64_t n0 = int64_t(b) * kRows;
            auto emit_all = [&]() {
                if (row < rows)
#pragma unroll
                    for (int m = 0; m < NH; ++m)
                        if (t0 + m < p.M) emit_out(t0 + m, n0 + row, acc[m]);
            };
            if (p.csize > 1) {
                // cluster split-K (one segment per CTA): push partials into the leader
                const int rank = c % p.csize;
                constexpr uint32_t kSlot = uint32_t(NT) * kRows * 4;
                asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
                if (rank == 0) {
                    if (et == 0 && eh == 0) {
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(rfull)),
                                     "r"(uint32_t(p.csize - 1) * kSlot)
                                     : "memory");
                        for (int r = 1; r < p.csize; ++r) {
                            uint32_t ra;
                            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(su32(go)), "r"(r));
                            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra)
                                         : "memory");
                        }
                    }
                    mbar_wait(rfull, 0);
                    const float4* red = reinterpret_cast<const float4*>(smem);
                    for (int r = 1; r < p.csize; ++r) {  // rank order: deterministic
#pragma unroll
                        for (int j = 0; j < NH / 4; ++j) {
                            const float4 x = red[((r - 1) * kRows + row) * (NT / 4) + t0 / 4 + j];
                            acc[4 * j] += x.x, acc[4 * j + 1] += x.y, acc[4 * j + 2] += x.z, acc[4 * j + 3] += x.w;
                        }
                    }
                    emit_all();
                } else {
                    mbar_wait(go, 0);
                    uint32_t dst, rb;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(dst)
                                 : "r"(su32(smem) + uint32_t((((rank - 1) * kRows + row) * NT + t0) * 4)));
                    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rb) : "r"(su32(rfull)));
#pragma unroll
                    for (int j = 0; j < NH / 4; ++j)
                        asm volatile(
                            "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                                dst + 16u * j),
                            "f"(acc[4 * j]), "f"(acc[4 * j + 1]), "f"(acc[4 * j + 2]), "f"(acc[4 * j + 3]), "r"(rb)
                            : "memory");
                }
            } else if (sole) {
                emit_all();
            } else {
                // stream-K: the owner holds the row-block's first k-block (its last segment);
                // the others hand over partials from their first segment (slot = CTA)
                const int c_first = cta_of(int64_t(b) * p.KBLK, p.U, p.G);
                const int c_last = cta_of(int64_t(b + 1) * p.KBLK - 1, p.U, p.G);
                if (c == c_first) {
                    if (et == 0 && eh == 0) {
                        const int want = c_last - c_first;
                        int got;
                        do {
                            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(got) : "l"(p.counters + b) : "memory");
                        } while (got < want);
                        p.counters[b] = 0;  // ready for the next launch (stream-ordered)
                    }
                    asm volatile("bar.sync 3, %0;" ::"r"(128 * EH) : "memory");
                    for (int cc = c_first + 1; cc <= c_last; ++cc) {  // fixed order: deterministic
                        const float4* src =
                            reinterpret_cast<const float4*>(p.partials + (int64_t(cc) * kRows + row) * NT + t0);
#pragma unroll
                        for (int j = 0; j < NH / 4; ++j) {
                            const float4 x = __ldcg(src + j);
                            acc[4 * j] += x.x, acc[4 * j + 1] += x.y, acc[4 * j + 2] += x.z, acc[4 * j + 3] += x.w;
                        }
                    }
                    emit_all();
                } else {
                    // contributor (its first segment): store the partial; warp 3 publishes it
                    // (gpu-scope fence + counter), off this pipeline's critical path
                    float4* mine = reinterpret_cast<float4*>(p.partials + (int64_t(c) * kRows + row) * NT + t0);
#pragma unroll
                    for (int j = 0; j < NH / 4; ++j)
                        mine[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(pub);
                }
            }
#pragma unroll
            for (int t = 0; t < NH; ++t) acc[t] = 0.0f;
            seg_kb0 = kbe == p.KBLK ? 0 : kbe;
        }
        cu.advance(n);
        };
        while (cu.more()) epi_step();
        if ((dbg_ & 64) && et == 0 && eh == 0) g_i4_dbg[c * 16 + 4] = gtime();
        if ((dbg_ & 32) && et == 0 && eh == 0)
            g_i4_dbg[c * 16 + 11] = e_wait, g_i4_dbg[c * 16 + 12] = e_work, g_i4_dbg[c * 16 + 13] = clock64() - e_t0,
            g_i4_dbg[c * 16 + 14] = si, g_i4_dbg[c * 16 + 15] = e_ld;
    }
    fence_before();
    __syncthreads();
    if ((dbg_ & 64) && threadIdx.x == 0) g_i4_dbg[c * 16 + 7] = gtime();
    if constexpr (PEER)
        if (threadIdx.x == 0) peer_complete(p.peer, peer_round(p.peer), int(gridDim.x));
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int PT, int BITS, bool PEER>
cudaError_t launch_nt(Params p, cudaStream_t st) {
    using GG = Geo<PT, BITS>;
    auto kern = wgemm_i4_kernel<PT, BITS, PEER>;
    static unsigned long long configured = 0;  // per device
    static int max_clusters_dev[64][9] = {};
    int* max_clusters = max_clusters_dev[current_device_index()];
    if (!(configured & current_device_bit())) {
        if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, GG::SMEM))
            return e;
        configured |= current_device_bit();
    }
    if (p.csize > GG::MAXC) p.csize = GG::MAXC;
    while (p.csize > 1) {
        int& mc = max_clusters[p.csize];
        if (mc == 0) {
            cudaLaunchConfig_t q{};
            q.gridDim = dim3(unsigned(p.NB * p.csize));
            q.blockDim = dim3(GG::THREADS);
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
    cfg.blockDim = dim3(GG::THREADS);
    cfg.dynamicSmemBytes = GG::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (p.csize > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = unsigned(p.csize);
        attr[na].val.clusterDim.y = attr[na].val.clusterDim.z = 1;
        ++na;
    }
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // after the planes kernel
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

}  // namespace i4

constexpr size_t kI4Counters = 64 * 1024;

extern "C" int rtnq_i4_timeline_read(void* host, size_t bytes) {
    if (bytes > sizeof(i4::g_i4_tl)) bytes = sizeof(i4::g_i4_tl);
    return cudaMemcpyFromSymbol(host, i4::g_i4_tl, bytes) == cudaSuccess ? 0 : 1;
}

extern "C" int rtnq_i4_debug_read(void* host, size_t bytes) {
    if (bytes > sizeof(i4::g_i4_dbg)) bytes = sizeof(i4::g_i4_dbg);
    return cudaMemcpyFromSymbol(host, i4::g_i4_dbg, bytes) == cudaSuccess ? 0 : 1;
}

static size_t align256_i4(size_t x) { return (x + 255) / 256 * 256; }

size_t wgemm_i4_workspace_bytes(int64_t m, int64_t n, int64_t k) {
    (void)n;
    const size_t part = size_t(imma::sms()) * i4::kRows * 64 * sizeof(float);
    return kI4Counters + align256_i4(part) + align256_i4(size_t(3 * m * k)) + align256_i4(size_t(m) * 4);
}

const char* wgemm_i4_unsupported(int64_t m, int64_t n, int64_t k, int bits, int64_t g, int a_dtype) {
    (void)m, (void)n;
    if ((bits != 4 && bits != 8) || g != 128) return "the group-128 int8 tensor-core path is group size 128";
    if (a_dtype != RTNQ_BF16 && a_dtype != RTNQ_F16) return "activations must be bf16 or f16";
    if (k % 16 != 0) return "k must be a multiple of 16 for the int8 tensor-core path";
    return nullptr;
}

template <int PT, int BITS>
static cudaError_t launch_pt(const i4::Params& p, cudaStream_t st) {
    return p.peer.world ? i4::launch_nt<PT, BITS, true>(p, st) : i4::launch_nt<PT, BITS, false>(p, st);
}

cudaError_t launch_wgemm_i4(const WgemmArgs& A, cudaStream_t st) {
    imma::EncodeFn enc = imma::encoder();
    if (!enc) return cudaErrorNotSupported;
    const int64_t kblk = (A.k + i4::kKB - 1) / i4::kKB;
    char* ws = static_cast<char*>(A.workspace);
    i4::Params p{};
    p.counters = reinterpret_cast<int*>(ws);
    const size_t part = size_t(imma::sms()) * i4::kRows * 64 * sizeof(float);
    p.partials = reinterpret_cast<float*>(ws + kI4Counters);
    int8_t* planes_ws = reinterpret_cast<int8_t*>(ws + kI4Counters + align256_i4(part));
    int32_t* texp_ws = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(planes_ws) + align256_i4(size_t(3 * A.m * A.k)));
    // planes from the producer of the activations (fused into add+RMSNorm / SiLU*up), or ours
    const bool own_planes = A.planes == nullptr;
    int8_t* planes = own_planes ? planes_ws : const_cast<int8_t*>(A.planes);
    int32_t* texp = own_planes ? texp_ws : const_cast<int32_t*>(A.texp);
    const char* dbg_env = std::getenv("RTNQ_WGEMM_DEBUG");
    const int dbg = dbg_env ? std::atoi(dbg_env) : 0;
    unsigned long long* stamps = nullptr;
    if (dbg & 64) {
        void* base = nullptr;
        if (cudaGetSymbolAddress(&base, i4::g_i4_dbg) == cudaSuccess)
            stamps = static_cast<unsigned long long*>(base) + 1023 * 16;
    }
    // Optional (RTNQ_WEIGHT_PREFETCH=1): L2 prefetch of each GEMM CTA's first 64 KiB, issued by
    // the planes kernel (same partition rule as the launch below; a hint, so the occupancy clamp
    // of cluster sizes is ignored).  Measured 2x slower end to end on B200 (the prefetches hold
    // up the planes kernel), so it is off by default.
    imma::WeightPrefetch pf;
    if (std::getenv("RTNQ_WEIGHT_PREFETCH")) {
        const int nb = int((A.n + 127) / 128), kb = int((A.k + 127) / 128);
        int csize = 1;
        if (!std::getenv("RTNQ_WGEMM_CTAS") && int64_t(nb) * 2 <= imma::sms()) {
            const char* ce = std::getenv("RTNQ_WGEMM_CLUSTER");
            if (!ce || std::atoi(ce) != 0) {
                int S = imma::sms() / nb;
                S = S > 8 ? 8 : S;
                S = S > kb ? kb : S;
                csize = S < 2 ? 1 : S;
            }
        }
        pf.base = A.codes;
        pf.kind = 4;
        pf.KBLK = kb;
        pf.U = nb * kb;
        pf.csize = csize;
        pf.G = csize > 1 ? nb * csize : (pf.U < imma::sms() ? pf.U : imma::sms());
        pf.bytes = int64_t(nb) * kb * 8192;
        pf.head = 64 * 1024;
    }
    // planes inside the GEMM (default) or by the stand-alone planes kernel (RTNQ_PLANES_KERNEL=1,
    // or unaligned activations)
    static const bool planes_kernel = [] {
        const char* e = std::getenv("RTNQ_PLANES_KERNEL");
        return e && std::atoi(e) != 0;
    }();
    // (a handful of tokens: one producing CTA per token is a longer critical path than the
    // stand-alone kernel's token x slice grid; measured crossover between 1 and 16 tokens)
    // (and a small weight: its few stages per CTA cannot hide the producing CTAs' critical path;
    // scratch/shapes_seq.py, batch 16: qkv / o 10.3 / 9.1 us with the planes kernel, 11.8 / 10.4
    // in the GEMM; gate_up / down 23.7 / 19.4 vs 21.7 / 18.5)
    const int64_t units = ((A.n + i4::kRows - 1) / i4::kRows) * ((A.k + i4::kKB - 1) / i4::kKB);
    // W8 group-128 from 16 tokens too: with the sliced hand-off, gate_up / down at batch 16
    // 27.0 / 19.5 -> 24.9 / 17.2 us, batch 32 29.9 / 24.4 -> 27.7 / 21.7 us; at batch 8 the
    // stand-alone kernel stays (23.6 vs 24.5 us gate_up)
    static const int64_t min_units = [] {
        const char* e = std::getenv("RTNQ_OWN_PLANES_MIN_UNITS");
        return e ? int64_t(std::atoll(e)) : int64_t(2048);
    }();
    static const int min_m4 = [] {
        const char* e = std::getenv("RTNQ_OWN_PLANES_MIN_M");
        return e ? std::atoi(e) : imma::kOwnPlanesMinM;
    }();
    const bool in_gemm = own_planes && !planes_kernel && A.m >= (A.bits == 4 ? min_m4 : 16) &&
                         units >= min_units &&
                         (reinterpret_cast<uintptr_t>(A.a) & 15) == 0 && !(dbg & 64);
    if (in_gemm) {
        p.own.a = A.a;
        p.own.a_dtype = A.a_dtype;
        p.own.done = p.counters + (kI4Counters / sizeof(int) - 2);
        p.own.consumed = p.counters + (kI4Counters / sizeof(int) - 1);
        p.own.err = A.err;
        p.planes_w = planes;
    }
    if (own_planes && !in_gemm) {
        const bool vec = (reinterpret_cast<uintptr_t>(A.a) & 15) == 0;
        cudaError_t e = A.a_dtype == RTNQ_BF16
            ? (vec ? imma::launch_planes<RTNQ_BF16, true> : imma::launch_planes<RTNQ_BF16, false>)(
                  A.a, int(A.k), int(A.m), planes, texp, stamps, pf, A.err, st)
            : (vec ? imma::launch_planes<RTNQ_F16, true> : imma::launch_planes<RTNQ_F16, false>)(
                  A.a, int(A.k), int(A.m), planes, texp, stamps, pf, A.err, st);
        if (e != cudaSuccess) return e;
    }
    p.codes = A.codes;
    p.scales = A.scales;
    p.texp = texp;
    p.peer = A.peer;
    p.N = A.n;
    p.K = A.k;
    p.Mtot = int(A.m);
    p.NB = int((A.n + i4::kRows - 1) / i4::kRows);
    p.KBLK = int(kblk);
    p.U = p.NB * p.KBLK;
    p.out_dtype = A.out_dtype;
    p.debug = dbg;
    const int esz = A.out_dtype == RTNQ_F32 ? 4 : 2;
    // tokens per chunk: the smallest PT >= M (B operand N = 3 * PT rounded up to 16)
    const int pt = A.m <= 5 ? 5 : A.m <= 10 ? 10 : A.m <= 16 ? 16 : A.m <= 32 ? 32 : 64;
    // peer output: one launch = one allreduce round, so the tokens must fit one chunk and the
    // slot (int8_mma.cuh peer_*)
    if (A.peer.world && (A.m > pt || A.m * A.n > A.peer.cap || A.out_dtype != RTNQ_BF16))
        return cudaErrorInvalidValue;
    for (int64_t m0 = 0; m0 < A.m; m0 += pt) {
        p.M = int(A.m - m0 < pt ? A.m - m0 : pt);
        p.m0 = int(m0);
        p.out = static_cast<char*>(A.out) + m0 * A.n * esz;
        const int nt = pt;
        {
            const cuuint64_t dims[3] = {cuuint64_t(A.k), cuuint64_t(A.m), 3};
            const cuuint64_t strides[2] = {cuuint64_t(A.k), cuuint64_t(A.m * A.k)};
            const cuuint32_t box[3] = {128, cuuint32_t(nt), 3};
            const cuuint32_t es[3] = {1, 1, 1};
            if (enc(&p.tmap_p, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, planes, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return cudaErrorInvalidValue;
        }
        // partition: cluster split-K for few row-blocks, else stream-K over all SMs
        p.csize = 1;
        if (!std::getenv("RTNQ_WGEMM_CTAS") && int64_t(p.NB) * 2 <= imma::sms()) {
            const char* ce = std::getenv("RTNQ_WGEMM_CLUSTER");
            if (!ce || std::atoi(ce) != 0) {
                int S = imma::sms() / p.NB;
                S = S > 8 ? 8 : S;
                S = S > p.KBLK ? p.KBLK : S;
                p.csize = S < 2 ? 1 : S;
            }
        }
        int G = imma::sms();
        if (const char* e = std::getenv("RTNQ_WGEMM_CTAS")) G = std::atoi(e);
        G = G < 1 ? 1 : G;
        p.G = int(p.U < G ? p.U : G);
        cudaError_t e = A.bits == 8
            ? (nt == 5    ? launch_pt<5, 8>(p, st)
               : nt == 10 ? launch_pt<10, 8>(p, st)
               : nt == 16 ? launch_pt<16, 8>(p, st)
               : nt == 32 ? launch_pt<32, 8>(p, st)
                          : launch_pt<64, 8>(p, st))
            : (nt == 5    ? launch_pt<5, 4>(p, st)
               : nt == 10 ? launch_pt<10, 4>(p, st)
               : nt == 16 ? launch_pt<16, 4>(p, st)
               : nt == 32 ? launch_pt<32, 4>(p, st)
                          : launch_pt<64, 4>(p, st));
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace rtnq_b200
