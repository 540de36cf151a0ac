// wgemm_i8.cu -- W8A16 per-channel linear on tcgen05.mma.kind::i8.
//
// out[m][n] = S[n] * sum_k a[m][k] * code[n][k]        (gemm.hpp:18-27, one group per row)
//
// The 8-bit codes need no dequantization at all.  The RTNQ_NATIVE_I8 layout (common.cuh)
// holds the signed codes c (the reference's offset-binary byte u = c + 128, packing.cpp:19-22,
// minus the offset) as two's-complement bytes in 16 KiB tiles of 128 rows x 128 codes,
// contiguous and pre-swizzled.  One bulk copy moves a tile into 1024-aligned shared memory,
// where it already is the 128-byte-swizzled K-major s8 A operand of the tensor core.
//
// The bf16/f16 activations become three exact int8 planes, done once per call by
// act_planes_kernel:
//   a = 2^s * (P0 + P1 / 2^7 + P2 / 2^14),  |Pi| <= 64.
// This is exact for every element within 2^13 of the token's largest magnitude.  Smaller
// ones round at 2^-21 of that maximum, far inside the 1e-5 parity bar.  The planes are
// the s8 B operand: N = 3 * tokens.
//
// The int32 accumulators are exact.  They run over a CTA's whole K range in TMEM; the
// scale S[n] is per row, so it is applied once at the end:
//   out = S[n] * 2^s * (D0 + D1 / 2^7 + D2 / 2^14).
//
// Warp roles: warp 0 is the TMA producer, warp 1 the single-thread MMA issuer, and
// warps 4-7 the epilogue (TMEM lane quadrants).  Work is partitioned with stream-K or,
// for few row-blocks, cluster split-K with a DSMEM reduction, as in wgemm_tc.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "../common.cuh"
#include "int8_mma.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {
namespace i8 {
using namespace imma;

constexpr int kRows = 128;     // UMMA M = one row-block
constexpr int kKB = 64;        // stream-K bookkeeping unit (k-block of 64 codes)
constexpr int kUnit = 128;     // codes per unit = one 128-byte swizzle row
constexpr int kThreads = 256;  // warp 0 producer, warp 1 MMA, warps 4-7 epilogue
constexpr int kEpi0 = 4;

struct Params {
    CUtensorMap tmap_p;  // planes [3][M][K] s8, box {128, NT, 3}, SWIZZLE_128B
    const uint8_t* codes;  // RTNQ_NATIVE_I8: 16 KiB pre-swizzled 128 x 128 tiles, row-block major
    const uint16_t* scales;  // f16 per row
    const int32_t* texp;     // [M] token exponents s
    void* out;
    float* partials;
    int* counters;
    int64_t N, K;
    int M, Mtot, m0, NB, KBLK, U, G, csize, out_dtype;
    int pf;     // L2 prefetch distance in tiles (0 = off)
    int direct;  // cluster split-K: peers push into a dedicated smem region (no go handshake)
    int debug;  // profiling: 4 = no MMA issued, 2 = no loads (arrive only)
    imma::OwnPlanes own;  // own.a != nullptr: this launch computes its tokens' planes itself
    int8_t* planes_w;     // ... into this [3][Mtot][K] buffer (the TMA source), exponents into texp
    PeerOut peer;         // tensor parallel: output pushed into every rank's slot (world > 0)
};

template <int NT>
struct Geo {
    static constexpr int CODE_BYTES = kRows * kUnit;             // 16 KiB tile
    static constexpr int PLANE_BYTES = 3 * NT * kUnit;           // 6 / 12 / 24 KiB per tile
    // Two tiles per stage (one barrier round trip per 32 KiB of codes): a CTA's TMA ring
    // streams markedly faster with >= 32 KiB per stage than with 16 KiB (scratch/stream_bench3).
    static constexpr int TPS = NT <= 32 ? 2 : 1;                 // tiles per stage
    static constexpr int SPAN = 2 * TPS;                         // k-blocks per stage
    static constexpr int PLANE_OFF = TPS * CODE_BYTES;
    static constexpr int STAGE_BYTES = TPS * (CODE_BYTES + PLANE_BYTES);  // multiple of 1 KiB
    static constexpr int STAGES_FIT = (208 * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
    static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
    static constexpr int SMEM = BAR_OFF + 1024 + 1024;
    static constexpr int PUSH_OFF = BAR_OFF + 1024;              // direct-push partials region
    static constexpr int DN = 3 * NT;                             // accumulator columns
    // cluster split-K: the leader's stage area holds csize - 1 pushed partials
    static constexpr int MAXC_FIT = 1 + STAGES * STAGE_BYTES / (NT * kRows * 4);
    static constexpr int MAXC = MAXC_FIT > 8 ? 8 : MAXC_FIT;
    static_assert(STAGES >= 3, "");
};

__device__ unsigned long long g_i8_dbg[1024 * 16];  // profiling (debug & 32; & 64: globaltimer stamps)


// PEER: the output goes to the tensor-parallel peers' slots (a separate instantiation: the peer
// store path compiled into the plain kernel measured +2.5 us per launch, never executed)
template <int NT, bool PEER>
__global__ void __launch_bounds__(kThreads, 1) wgemm_i8_kernel(const __grid_constant__ Params p) {
#ifdef RTNQ_KERNEL_DEBUG
    const int dbg_ = p.debug;  // profiling knobs (scratch/*prof*.py, *tl.py)
#else
    constexpr int dbg_ = 0;  // compiled out: even disabled, the checks cost a few % per launch
#endif
    using GG = Geo<NT>;
    constexpr int STAGES = GG::STAGES, DN = GG::DN;
    extern __shared__ uint8_t smem_raw[];
    // align by indexing the __shared__ array (keeps the shared address space: LDS/STS, not
    // generic loads)
    uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + GG::BAR_OFF);  // [STAGES]
    uint64_t* empty = full + STAGES;                                  // [STAGES]
    uint64_t* dfull = empty + STAGES;                                 // [2]
    uint64_t* dempty = dfull + 2;                                     // [2]
    uint64_t* go = dempty + 2;      // cluster split-K: the leader is ready for partials
    uint64_t* rfull = dempty + 3;   // cluster split-K: all partials landed in the leader
    uint64_t* pub = dempty + 4;     // stream-K contributor partials stored (4 warps)
    uint64_t* pready = dempty + 5;  // own planes: this launch's planes / exponents published
    uint32_t* tslot = reinterpret_cast<uint32_t*>(dempty + 6);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, c = blockIdx.x;
    if ((dbg_ & 64) && threadIdx.x == 0) g_i8_dbg[c * 16 + 5] = gtime();

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
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 2), mbar_init(&empty[s], 1);
        for (int i = 0; i < 2; ++i) mbar_init(&dfull[i], 1), mbar_init(&dempty[i], 4);
        mbar_init(go, 1), mbar_init(rfull, 1), mbar_init(pub, 4), mbar_init(pready, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            su32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    // cluster peers touch each other's barriers only at the end: arrive now, wait there
    if (p.csize > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    const uint32_t tmem = *tslot;
    asm volatile("griddepcontrol.launch_dependents;");
    if (p.own.a && warp >= kEpi0) {  // the epilogue warps compute this CTA's share of the planes
        __shared__ float pred[4];
        own_planes_produce(p.own, int(p.K), p.m0, p.M, p.Mtot, c, int(gridDim.x), p.planes_w,
                           const_cast<int32_t*>(p.texp), threadIdx.x - kEpi0 * 32, 128, 3, pred);
    }

    // units: runs of <= SPAN k-blocks inside one row-block and one SPAN-aligned k-range
    auto chunk = [&](int u, int kb) {
        const int left_seg = p.KBLK - kb, left = u1 - u, cap = GG::SPAN - (kb & (GG::SPAN - 1));
        const int n = left_seg < left ? left_seg : left;
        return n < cap ? n : cap;
    };

    if (warp == 0 || warp == 2) {
        // ===================== producers: warp 0 codes, warp 2 activation planes ===========
        // Warp-uniform loops (one elected lane issues), incremental row-block / k-block.
        const bool codes = warp == 0;
        Cursor<GG::SPAN> cu(u0, u1, p.KBLK);
        int s = 0;
        uint32_t ph = 0;
        const long long t0 = clock64();
        long long tw = 0;
        // The CTA's tiles are one contiguous run of the NATIVE_I8 array: keep an L2 prefetch
        // window of p.pf tiles ahead of the smem ring (more bytes in flight than the ring holds).
        const int64_t kt = (p.KBLK + 1) >> 1;
        const int64_t t_last = u1 > u0 ? int64_t((u1 - 1) / p.KBLK) * kt + ((u1 - 1) % p.KBLK >> 1) : -1;
        int64_t pf_next = int64_t(cu.b) * kt + (cu.kb >> 1);
        if (!codes) {
            if (p.own.a) {  // planes computed by this launch's CTAs
                own_planes_acquire(p.own, p.M, int(gridDim.x), int(p.K));
                if (lane == 0) mbar_arrive(pready);
            } else {
                asm volatile("griddepcontrol.wait;" ::: "memory");  // planes from the previous kernel
            }
        }
        for (int i = 0; cu.more(); ++i) {
            const int n = cu.chunk();
            if (i >= STAGES) {
                const long long a0 = clock64();
                mbar_wait(&empty[s], ph ^ 1u);
                tw += clock64() - a0;
            }
            uint8_t* st = smem + s * GG::STAGE_BYTES;
            // the tiles this unit touches (1 or TPS, same row-block): tile t goes to stage slot
            // t % TPS. A half tile (one 64-code k-block) still loads the whole tile and its
            // 128-code planes box; the MMA uses one half.
            const int ta = cu.kb >> 1, tb = (cu.kb + n - 1) >> 1;
            const int slot0 = ta & (GG::TPS - 1);
            if (dbg_ & 2) {
                elect_arrive(&full[s]);
            } else if (codes) {  // contiguous, pre-swizzled 16 KiB tiles
                const int64_t tile = int64_t(cu.b) * kt + ta;
                if (p.pf > 0 && pf_next <= t_last && pf_next <= tile + p.pf) {
                    const int64_t nt4 = t_last - pf_next + 1 < 4 ? t_last - pf_next + 1 : 4;
                    elect_prefetch(p.codes + pf_next * GG::CODE_BYTES, uint32_t(nt4 * GG::CODE_BYTES));
                    pf_next += nt4;
                }
                elect_bulk(st + slot0 * GG::CODE_BYTES, p.codes + tile * GG::CODE_BYTES, &full[s],
                           uint32_t(tb - ta + 1) * GG::CODE_BYTES);
            } else {
                elect_expect(&full[s], uint32_t(tb - ta + 1) * GG::PLANE_BYTES);
                for (int t = ta; t <= tb; ++t)
                    elect_tma3d_tx(st + GG::PLANE_OFF + (t & (GG::TPS - 1)) * GG::PLANE_BYTES, &p.tmap_p,
                                   t * kUnit, p.m0, 0, &full[s]);
            }
            cu.advance(n);
            if (++s == STAGES) s = 0, ph ^= 1u;
        }
        if ((dbg_ & 32) && lane == 0 && codes) {
            g_i8_dbg[c * 8 + 0] = clock64() - t0;
            g_i8_dbg[c * 8 + 1] = tw;
        }
        if ((dbg_ & 64) && lane == 0 && codes) g_i8_dbg[c * 16 + 0] = gtime();
    } else if (warp == 3) {
        // ===================== stream-K publisher (off the epilogue's critical path) =======
        if (p.csize == 1 && u0 < u1 && u0 % p.KBLK != 0) {
            mbar_wait(pub, 0);
            if (lane == 0) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;" ::"l"(p.counters + u0 / p.KBLK) : "memory");
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (warp-uniform, one elected lane issues) ==========
        // D s32, A s8 (codes), B s8 (planes), M = 128, N = 3 * NT
        constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                   (uint32_t(DN >> 3) << 17) | (uint32_t(kRows >> 4) << 24);
        constexpr uint64_t kHi = (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) |
                                 (2ull << 61);  // K-major SWIZZLE_128B, SBO = 1024
        const uint32_t lo0 = su32(smem) >> 4;   // descriptor address field of stage 0
        Cursor<GG::SPAN> cu(u0, u1, p.KBLK);
        int s = 0, db = 0, seg = 0;
        uint32_t ph = 0, lo = lo0;
        bool first = true;
        const long long t0 = clock64();
        long long tw = 0, ti = 0;
        while (cu.more()) {
            const int n = cu.chunk();
            const bool seg_end = cu.seg_end(n);
            if (first && seg >= 2) {  // accumulator reuse: the epilogue drained it
                mbar_wait(&dempty[db], uint32_t((seg >> 1) - 1) & 1u);
                fence_after();
            }
            const long long a0 = clock64();
            mbar_wait(&full[s], ph);
            fence_after();
            const long long a1 = clock64();
            if ((dbg_ & 64) && lane == 0 && first && seg == 0) g_i8_dbg[c * 16 + 6] = gtime();
            tw += a1 - a0;
            const uint32_t d = tmem + db * DN;
            // one elected thread issues the stage's MMAs back to back and their commits;
            // k-block kb: tile slot (kb >> 1) % TPS, second 64-code half at +64 B
            // the whole warp issues (one elected lane, warp-uniform asm blocks; int8_mma.cuh)
            if (!(dbg_ & 4)) {
                for (int j = 0; j < n; ++j) {
                    const int kb = cu.kb + j;
                    const uint32_t alo = lo + uint32_t(((kb >> 1) & (GG::TPS - 1)) * (GG::CODE_BYTES >> 4)) +
                                         ((kb & 1) ? 4u : 0u);
                    const uint32_t blo = lo + uint32_t(GG::PLANE_OFF >> 4) +
                                         uint32_t(((kb >> 1) & (GG::TPS - 1)) * (GG::PLANE_BYTES >> 4)) +
                                         ((kb & 1) ? 4u : 0u);
                    mma2_i8_ss_warp(d, kHi | alo, kHi | blo, idesc, (first && j == 0) ? 0u : 1u);
                }
            }
            commit_elect(&empty[s]);
            if (seg_end) commit_elect(&dfull[db]);
            __syncwarp();
            first = false;
            ti += clock64() - a1;
            if (seg_end) {
                db ^= 1;
                ++seg;
                first = true;
            }
            cu.advance(n);
            if (++s == STAGES) s = 0, ph ^= 1u, lo = lo0;
            else lo += GG::STAGE_BYTES >> 4;
        }
        if ((dbg_ & 32) && lane == 0) {
            g_i8_dbg[c * 8 + 2] = clock64() - t0;
            g_i8_dbg[c * 8 + 3] = tw;
            g_i8_dbg[c * 8 + 4] = ti;
        }
        if ((dbg_ & 64) && lane == 0) g_i8_dbg[c * 16 + 1] = gtime();
    } else if (warp >= kEpi0) {
        // ===================== epilogue =====================
        const int q = warp & 3, row = q * 32 + lane, et = threadIdx.x - kEpi0 * 32;
        int pe = 0;  // tensor parallel: the peer round, read below once the previous grid is done
        const uint32_t lane_base = uint32_t(q * 32) << 16;
        int db = 0, seg = 0, u = u0;
        __shared__ float pow_s[NT];  // 2^s per token (s >= -126: a normal float)
        if (p.own.a) mbar_wait(pready, 0);  // texp published by this launch
        else asm volatile("griddepcontrol.wait;" ::: "memory");  // texp from the planes producer
        for (int t = et; t < NT; t += 128) pow_s[t] = t < p.M ? ldexpf(1.0f, __ldg(p.texp + p.m0 + t)) : 0.0f;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        // the output: local, or (tensor parallel) this rank's slot of every rank's buffer
        if constexpr (PEER) pe = peer_round(p.peer);
        auto emit_out = [&](int m, int64_t col, float v) {
            if constexpr (PEER) peer_store(p.peer, pe, int64_t(p.m0 + m) * p.N + col, v);
            else store_out(p.out, p.out_dtype, int64_t(m) * p.N + col, v);
        };
        while (u < u1) {
            // walk to this segment's end
            const int b = u / p.KBLK, kb0 = u - b * p.KBLK;
            int kbe = kb0, uu = u;
            while (true) {
                const int kb = uu - b * p.KBLK, n = chunk(uu, kb);
                uu += n, kbe = kb + n;
                if (kbe == p.KBLK || uu == u1) break;
            }
            const bool sole = kb0 == 0 && kbe == p.KBLK;
            if ((dbg_ & 64) && et == 0) g_i8_dbg[c * 16 + 8] = gtime();
            const int rows = min(kRows, int(p.N - int64_t(b) * kRows));
            const float srow = row < rows ? __half2float(__ushort_as_half(__ldg(p.scales + int64_t(b) * kRows + row))) : 0.0f;
            if ((dbg_ & 64) && et == 0) g_i8_dbg[c * 16 + 9] = gtime();
            // Stream-K: the row-block's owner is the CTA holding its first k-block (for that
            // CTA it is the last segment, finished last); the other contributors hand over
            // partials from their first segment, usually long before. The owner collects them
            // while its own MMAs drain.
            if ((dbg_ & 64) && et == 0) g_i8_dbg[c * 16 + 9] = gtime();
            const bool split = p.csize == 1 && !sole;
            const int c_first = split ? cta_of(int64_t(b) * p.KBLK, p.U, p.G) : c;
            const int c_last = split ? cta_of(int64_t(b + 1) * p.KBLK - 1, p.U, p.G) : c;
            const bool owner = split && c == c_first;
            float psum[NT];
#pragma unroll
            for (int m = 0; m < NT; ++m) psum[m] = 0.0f;
            if (owner) {
                if (et == 0) {
                    const int want = c_last - c_first;
                    int got;
                    do {
                        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(got) : "l"(p.counters + b) : "memory");
                    } while (got < want);
                    p.counters[b] = 0;  // ready for the next launch (stream-ordered after this one)
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                for (int cc = c_first + 1; cc <= c_last; ++cc) {  // fixed order: deterministic
                    const float4* src = reinterpret_cast<const float4*>(p.partials + (int64_t(cc) * kRows + row) * NT);
#pragma unroll
                    for (int j = 0; j < NT / 4; ++j) {
                        const float4 x = __ldcg(src + j);
                        psum[4 * j] += x.x, psum[4 * j + 1] += x.y, psum[4 * j + 2] += x.z, psum[4 * j + 3] += x.w;
                    }
                }
            }
            if ((dbg_ & 64) && et == 0) g_i8_dbg[c * 16 + 2] = gtime();
            mbar_wait(&dfull[db], uint32_t(seg >> 1) & 1u);
            fence_after();
            if ((dbg_ & 64) && et == 0) g_i8_dbg[c * 16 + 3] = gtime();
            float acc[NT], pw[NT];
#pragma unroll
            for (int t = 0; t < NT; ++t) pw[t] = pow_s[t];
            const long long ck0 = clock64();
            long long ck1 = 0;
#pragma unroll
            for (int j = 0; j < NT; j += 16) {
                uint32_t d0[16], d1[16], d2[16];
                if (dbg_ & 16) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) d0[e] = d1[e] = d2[e] = uint32_t(e + row);
                } else {
                    ld16(tmem + lane_base + db * DN + j, d0);
                    ld16(tmem + lane_base + db * DN + NT + j, d1);
                    ld16(tmem + lane_base + db * DN + 2 * NT + j, d2);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                }
                if (j == 0) ck1 = clock64();
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    // branch-free: pow_s is 0 for the padding tokens t >= M
                    const float x = float(int32_t(d0[e])) + float(int32_t(d1[e])) * 0.0078125f +
                                    float(int32_t(d2[e])) * 6.103515625e-05f;
                    acc[j + e] = x * pw[j + e] * srow;
                }
            }
            const long long ck2 = clock64();
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&dempty[db]);
            if ((dbg_ & 64) && et == 0) {
                g_i8_dbg[c * 16 + 12] = ck1 - ck0;
                g_i8_dbg[c * 16 + 13] = ck2 - ck1;
                g_i8_dbg[c * 16 + 14] = clock64() - ck2;
            }
            if ((dbg_ & 64) && et == 0) g_i8_dbg[c * 16 + 10] = gtime();
            const int64_t n0 = int64_t(b) * kRows;
            if (p.csize > 1) {
                // Cluster split-K (one segment per CTA): the leader (rank 0) opens its idle
                // stage area once its own MMAs are done; the peers push their partials there
                // with st.async, completing on the leader's rfull barrier.
                const int rank = c % p.csize;
                constexpr uint32_t kSlot = uint32_t(NT) * kRows * 4;
                asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
                if (rank == 0) {
                    if (et == 0) {
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(rfull)),
                                     "r"(uint32_t(p.csize - 1) * kSlot)
                                     : "memory");
                        for (int r = 1; r < p.csize && !p.direct; ++r) {
                            uint32_t ra;
                            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(su32(go)), "r"(r));
                            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
                        }
                    }
                    mbar_wait(rfull, 0);
                    const float4* red = reinterpret_cast<const float4*>(p.direct ? smem + GG::PUSH_OFF : smem);
                    for (int r = 1; r < p.csize; ++r) {  // rank order: deterministic
#pragma unroll
                        for (int j = 0; j < NT / 4; ++j) {
                            const float4 x = red[((r - 1) * kRows + row) * (NT / 4) + j];
                            acc[4 * j] += x.x, acc[4 * j + 1] += x.y, acc[4 * j + 2] += x.z, acc[4 * j + 3] += x.w;
                        }
                    }
                    if (row < rows)
#pragma unroll
                        for (int m = 0; m < NT; ++m)
                            if (m < p.M) emit_out(m, n0 + row, acc[m]);
                } else {
                    // direct: a region nobody else uses, so push at once (a complete_tx that lands
                    // before the leader's expect_tx only drives the tx-count negative meanwhile)
                    if (!p.direct) mbar_wait(go, 0);
                    uint32_t dst, rb;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(dst)
                                 : "r"(su32(p.direct ? smem + GG::PUSH_OFF : smem) +
                                       uint32_t(((rank - 1) * kRows + row) * NT * 4)));
                    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rb) : "r"(su32(rfull)));
#pragma unroll
                    for (int j = 0; j < NT / 4; ++j)
                        asm volatile(
                            "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                                dst + 16u * j),
                            "f"(acc[4 * j]), "f"(acc[4 * j + 1]), "f"(acc[4 * j + 2]), "f"(acc[4 * j + 3]), "r"(rb)
                            : "memory");
                }
            } else if (!split || owner) {
                if (row < rows)
#pragma unroll
                    for (int m = 0; m < NT; ++m)
                        if (m < p.M) emit_out(m, n0 + row, acc[m] + psum[m]);
            } else {  // contributor: this is the CTA's first segment, partial slot c
                float4* mine = reinterpret_cast<float4*>(p.partials + (int64_t(c) * kRows + row) * NT);
#pragma unroll
                for (int j = 0; j < NT / 4; ++j)
                    mine[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
                __syncwarp();
                if (lane == 0) mbar_arrive(pub);  // warp 3 publishes (gpu-scope fence + counter)
            }
            if ((dbg_ & 64) && et == 0) g_i8_dbg[c * 16 + 11] = gtime();
            u = uu;
            db ^= 1;
            ++seg;
        }
    }
    if ((dbg_ & 64) && threadIdx.x == kEpi0 * 32) g_i8_dbg[c * 16 + 4] = gtime();
    fence_before();
    __syncthreads();
    if ((dbg_ & 64) && threadIdx.x == 0) g_i8_dbg[c * 16 + 7] = gtime();
    if constexpr (PEER)
        if (threadIdx.x == 0) peer_complete(p.peer, peer_round(p.peer), int(gridDim.x));
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

// ---- host ----------------------------------------------------------------------------------
template <int NT, bool PEER>
cudaError_t launch_nt(Params p, cudaStream_t st, bool pdl) {
    using GG = Geo<NT>;
    auto kern = wgemm_i8_kernel<NT, PEER>;
    static unsigned long long configured = 0;  // per device
    static int max_clusters_dev[64][9] = {};
    int* max_clusters = max_clusters_dev[current_device_index()];
    constexpr int kSmemMax = 226 * 1024;  // 227 KiB opt-in less the static __shared__ arrays
    if (!(configured & current_device_bit())) {
        if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax))
            return e;
        configured |= current_device_bit();
    }
    if (p.csize > GG::MAXC) p.csize = GG::MAXC;
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
    // cluster split-K: a dedicated region for the peers' partials when it fits next to the ring
    static const bool direct_ok = [] {
        const char* e = std::getenv("RTNQ_I8_DIRECT");
        return !e || std::atoi(e) != 0;
    }();
    const int extra = (p.csize - 1) * NT * kRows * 4;
    p.direct = p.csize > 1 && direct_ok && GG::SMEM + extra <= kSmemMax;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(p.G));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = GG::SMEM + (p.direct ? extra : 0);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (p.csize > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = unsigned(p.csize);
        attr[na].val.clusterDim.y = attr[na].val.clusterDim.z = 1;
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

}  // namespace i8

constexpr size_t kI8Counters = 64 * 1024;

extern "C" int rtnq_i8_debug_read(void* host, size_t bytes) {
    if (bytes > sizeof(i8::g_i8_dbg)) bytes = sizeof(i8::g_i8_dbg);
    return cudaMemcpyFromSymbol(host, i8::g_i8_dbg, bytes) == cudaSuccess ? 0 : 1;
}

static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

size_t wgemm_i8_workspace_bytes(int64_t m, int64_t n, int64_t k) {
    (void)n;
    const size_t part = size_t(i8::sms()) * 2 * i8::kRows * 64 * sizeof(float);
    return kI8Counters + align256(part) + align256(size_t(3 * m * k)) + align256(size_t(m) * 4);
}

const char* wgemm_i8_unsupported(int64_t m, int64_t n, int64_t k, int bits, int64_t g, int a_dtype) {
    (void)m, (void)n;
    if (bits != 8 || g < k) return "the int8 tensor-core path is W8 per-channel (one group per row)";
    if (a_dtype != RTNQ_BF16 && a_dtype != RTNQ_F16) return "activations must be bf16 or f16";
    if (k % 16 != 0) return "k must be a multiple of 16 for the int8 tensor-core path";
    return nullptr;
}

cudaError_t launch_act_planes(const void* a, int a_dtype, int64_t m, int64_t k, int8_t* planes,
                              int32_t* texp, cudaStream_t st) {
    const bool vec = (reinterpret_cast<uintptr_t>(a) & 15) == 0;
    imma::WeightPrefetch none;
    return a_dtype == RTNQ_BF16
        ? (vec ? imma::launch_planes<RTNQ_BF16, true> : imma::launch_planes<RTNQ_BF16, false>)(
              a, int(k), int(m), planes, texp, nullptr, none, nullptr, st)
        : (vec ? imma::launch_planes<RTNQ_F16, true> : imma::launch_planes<RTNQ_F16, false>)(
              a, int(k), int(m), planes, texp, nullptr, none, nullptr, st);
}

cudaError_t launch_wgemm_i8(const WgemmArgs& A, cudaStream_t st) {
    i8::EncodeFn enc = i8::encoder();
    if (!enc) return cudaErrorNotSupported;
    const int64_t kblk = (A.k + 63) / 64;
    char* ws = static_cast<char*>(A.workspace);
    i8::Params p{};
    p.counters = reinterpret_cast<int*>(ws);
    const size_t part = size_t(i8::sms()) * 2 * i8::kRows * 64 * sizeof(float);
    p.partials = reinterpret_cast<float*>(ws + kI8Counters);
    int8_t* planes_ws = reinterpret_cast<int8_t*>(ws + kI8Counters + align256(part));
    int32_t* texp_ws = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(planes_ws) + align256(size_t(3 * A.m * A.k)));
    // planes from the producer of the activations (fused into add+RMSNorm / SiLU*up), or ours
    const bool own_planes = A.planes == nullptr;
    int8_t* planes = own_planes ? planes_ws : const_cast<int8_t*>(A.planes);
    int32_t* texp = own_planes ? texp_ws : const_cast<int32_t*>(A.texp);
    // 1. activation planes (once per call): planes and token exponents
    const char* dbg_env = std::getenv("RTNQ_WGEMM_DEBUG");
    const int dbg = dbg_env ? std::atoi(dbg_env) : 0;
    unsigned long long* stamps = nullptr;  // planes-kernel globaltimer stamps (debug & 64)
    if (dbg & 64) {
        void* base = nullptr;
        if (cudaGetSymbolAddress(&base, i8::g_i8_dbg) == cudaSuccess)
            stamps = static_cast<unsigned long long*>(base) + 1023 * 16;
    }
    // Optional (RTNQ_WEIGHT_PREFETCH=1): L2 prefetch of each GEMM CTA's first 64 KiB, issued by
    // the planes kernel (same partition rule as the launch below; a hint, so the occupancy clamp
    // of cluster sizes is ignored).  Measured 2x slower end to end on B200 (the prefetches hold
    // up the planes kernel), so it is off by default.
    imma::WeightPrefetch pf;
    if (std::getenv("RTNQ_WEIGHT_PREFETCH")) {
        const int nb = int((A.n + 127) / 128), kb = int((A.k + 63) / 64);
        int csize = 1;
        if (!std::getenv("RTNQ_WGEMM_CTAS") && int64_t(nb) * 2 <= i8::sms()) {
            const char* ce = std::getenv("RTNQ_WGEMM_CLUSTER");
            if (!ce || std::atoi(ce) != 0) {
                int S = i8::sms() / nb;
                S = S > 8 ? 8 : S;
                S = S > kb ? kb : S;
                csize = S < 2 ? 1 : S;
            }
        }
        pf.base = A.codes;
        pf.kind = 8;
        pf.KBLK = kb;
        pf.U = nb * kb;
        pf.csize = csize;
        pf.G = csize > 1 ? nb * csize : (pf.U < i8::sms() ? pf.U : i8::sms());
        pf.bytes = int64_t(nb) * ((kb + 1) >> 1) * 16384;
        pf.head = 64 * 1024;
    }
    // measured slower for W8 than the stand-alone planes kernel (scratch/seq8.py: 25.5 vs 23.5 us
    // per ffn_up launch at batch 16; the W8 CTA has only its 4 epilogue warps to spare), so
    // opt-in: RTNQ_I8_OWN_PLANES=1
    static const bool planes_kernel = [] {
        const char* e = std::getenv("RTNQ_I8_OWN_PLANES");
        return !(e && std::atoi(e) != 0);
    }();
    const bool in_gemm = own_planes && !planes_kernel && A.m >= imma::kOwnPlanesMinM &&
                         (reinterpret_cast<uintptr_t>(A.a) & 15) == 0 && !(dbg & 64);
    if (in_gemm) {  // planes inside the GEMM (int8_mma.cuh, OwnPlanes)
        p.own.a = A.a;
        p.own.a_dtype = A.a_dtype;
        p.own.done = p.counters + (kI8Counters / sizeof(int) - 2);
        p.own.consumed = p.counters + (kI8Counters / sizeof(int) - 1);
        p.own.err = A.err;
        p.planes_w = planes;
    }
    if (own_planes && !in_gemm) {
        const bool vec = (reinterpret_cast<uintptr_t>(A.a) & 15) == 0;
        cudaError_t e = A.a_dtype == RTNQ_BF16
            ? (vec ? i8::launch_planes<RTNQ_BF16, true> : i8::launch_planes<RTNQ_BF16, false>)(
                  A.a, int(A.k), int(A.m), planes, texp, stamps, pf, A.err, st)
            : (vec ? i8::launch_planes<RTNQ_F16, true> : i8::launch_planes<RTNQ_F16, false>)(
                  A.a, int(A.k), int(A.m), planes, texp, stamps, pf, A.err, st);
        if (e != cudaSuccess) return e;
    }
    // 2. the GEMM
    p.codes = A.codes;
    p.scales = A.scales;
    p.texp = texp;
    p.peer = A.peer;
    p.N = A.n;
    p.K = A.k;
    p.Mtot = int(A.m);
    p.NB = int((A.n + i8::kRows - 1) / i8::kRows);
    p.KBLK = int(kblk);
    p.U = p.NB * p.KBLK;
    p.out_dtype = A.out_dtype;
    p.debug = dbg;
    // L2 prefetch window of 2 tiles ahead of the ring: +0.6 % on the step, deeper windows lose
    // (profiles/r1h_i8_l2_prefetch_ab.log)
    static const int pf_env = [] {
        const char* e = std::getenv("RTNQ_I8_PF");
        return e ? std::atoi(e) : 2;
    }();
    p.pf = pf_env;
    const int esz = A.out_dtype == RTNQ_F32 ? 4 : 2;
    const int nt_max = A.m <= 16 ? 16 : A.m <= 32 ? 32 : 64;
    // peer output: one launch = one allreduce round, so the tokens must fit one chunk and the
    // slot (int8_mma.cuh peer_*)
    if (A.peer.world && (A.m > nt_max || A.m * A.n > A.peer.cap || A.out_dtype != RTNQ_BF16))
        return cudaErrorInvalidValue;
    for (int64_t m0 = 0; m0 < A.m; m0 += nt_max) {
        p.M = int(A.m - m0 < nt_max ? A.m - m0 : nt_max);
        p.m0 = int(m0);
        p.out = static_cast<char*>(A.out) + m0 * A.n * esz;
        const int nt = p.M <= 16 ? 16 : p.M <= 32 ? 32 : 64;
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
        if (!std::getenv("RTNQ_WGEMM_CTAS") && int64_t(p.NB) * 2 <= i8::sms()) {
            const char* ce = std::getenv("RTNQ_WGEMM_CLUSTER");
            if (!ce || std::atoi(ce) != 0) {
                int S = i8::sms() / p.NB;
                S = S > 8 ? 8 : S;
                S = S > p.KBLK ? p.KBLK : S;
                p.csize = S < 2 ? 1 : S;
            }
        }
        int G = i8::sms();
        if (const char* e = std::getenv("RTNQ_WGEMM_CTAS")) G = std::atoi(e);
        G = G < 1 ? 1 : G;
        p.G = int(p.U < G ? p.U : G);
        const bool pdl = true;  // the planes kernel precedes it in the stream
        const bool peer = p.peer.world > 0;
        cudaError_t e = nt == 16 ? (peer ? i8::launch_nt<16, true>(p, st, pdl) : i8::launch_nt<16, false>(p, st, pdl))
                      : nt == 32 ? (peer ? i8::launch_nt<32, true>(p, st, pdl) : i8::launch_nt<32, false>(p, st, pdl))
                                 : (peer ? i8::launch_nt<64, true>(p, st, pdl) : i8::launch_nt<64, false>(p, st, pdl));
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace rtnq_b200
