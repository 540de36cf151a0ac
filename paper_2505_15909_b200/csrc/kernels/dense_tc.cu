// dense_tc.cu -- the dequant-first contraction on tcgen05 (gemm_dequant,
// gemm.cpp:94-98, and the m >= threshold branch of gemm_auto, :100-109).
//
// dequant_first.cu splits the exactly dequantized weights W = S * code into two 16-bit terms,
// W = hi + lo.  This kernel computes
//     out[m][n] = sum_k a[m][k] * (hi[n][k] + lo[n][k])
// in ONE accumulation: every 64-wide k-block of a 128 x 128 output tile issues the 4 K16 steps of
// a . hi^T and the 4 of a . lo^T into the same f32 TMEM accumulator (tcgen05.mma kind::f16,
// bf16 or f16 operands, both K-major from 128B-swizzled TMA tiles), and the epilogue writes the
// output type directly (no f32 C round trip, no cast kernel).
//
// Warp roles (192 threads, one tile per CTA):
//   warp 0      TMA producer: per k-block one box of a (128 x 64) and one each of hi and lo
//               (128 x 64), 48 KiB per stage, 4 stages
//   warp 1      TMEM allocation + the MMA issuer (warp-uniform asm, one elected lane)
//   warps 2-5   epilogue: tcgen05.ld of the 128 x 128 f32 accumulator (warp w reads TMEM lanes
//               32 (w % 4) ..), staged through shared memory so that each output row is written
//               by one warp with coalesced stores
//
// Roofline: 2 x 2 m n k flops (the hi and lo terms) against 2 (m + 2 n) k + m n * |out| bytes;
// tensor-bound for m >= 1024 (the only sizes gemm_auto sends here).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "int8_mma.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {
namespace dtc {
using namespace imma;

constexpr int BM = 128, BN = 128, BK = 64, STAGES = 4, THREADS = 192;
constexpr int TILE_BYTES = BM * BK * 2;  // 16 KiB: one 128 x 64 16-bit box (BM == BN)
constexpr int STAGE_BYTES = 3 * TILE_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 1024;  // ring + barriers + alignment
constexpr int OUT_LD = BN + 4;                            // staging row stride (floats)
static_assert(4 * 32 * OUT_LD * 4 <= STAGES * STAGE_BYTES, "epilogue staging fits the ring");

struct Params {
    CUtensorMap ta, th, tl;  // a [M][K], hi / lo [N][K]; 16-bit, box {64, 128}, SWIZZLE_128B
    void* out;               // [M][N] row-major, odtype
    int odtype;
    int M, N, KB;            // KB = k-blocks of 64
    int MT;                  // m-tiles
};

__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}

template <bool BF16>
__global__ void __launch_bounds__(THREADS, 1) dense_tc_kernel(const __grid_constant__ Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* accf = empty + STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(accf + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // tile order: all m-tiles of an n-tile back to back, so a wave of CTAs shares a few n-tiles
    // of hi / lo (the large operand) in L2 while the activations stay L2-resident
    const int mt = int(blockIdx.x % unsigned(p.MT)), nt = int(blockIdx.x / unsigned(p.MT));
    const int n0 = nt * BN, m0 = mt * BM;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
        mbar_init(accf, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tslot;
    if (warp == 0) {
        // ---- producer ----
        for (int kb = 0; kb < p.KB; ++kb) {
            const int s = kb % STAGES;
            if (kb >= STAGES) mbar_wait(&empty[s], uint32_t(kb / STAGES - 1) & 1u);
            uint8_t* st = smem + s * STAGE_BYTES;
            if (lane == 0) {
                mbar_expect_tx(&full[s], STAGE_BYTES);
                tma2d(st, &p.ta, kb * BK, m0, &full[s]);
                tma2d(st + TILE_BYTES, &p.th, kb * BK, n0, &full[s]);
                tma2d(st + 2 * TILE_BYTES, &p.tl, kb * BK, n0, &full[s]);
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ---- MMA issuer: D f32, A = activations (M = 128), B = hi / lo (N = 128), K16 steps ----
        constexpr uint32_t fmt = BF16 ? 1u : 0u;
        constexpr uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (uint32_t(BN >> 3) << 17) |
                                   (uint32_t(BM >> 4) << 24);
        for (int kb = 0; kb < p.KB; ++kb) {
            const int s = kb % STAGES;
            mbar_wait(&full[s], uint32_t(kb / STAGES) & 1u);
            fence_after();
            const uint32_t st = su32(smem + s * STAGE_BYTES);
            const uint64_t ad = sw128_desc(st), hd = sw128_desc(st + TILE_BYTES), ld = sw128_desc(st + 2 * TILE_BYTES);
            if (lane == 0) {
#pragma unroll
                for (int ks = 0; ks < BK / 16; ++ks) {  // 32 bytes of K per step inside the 128B atom
                    mma_f16(tmem, ad + 2 * ks, hd + 2 * ks, idesc, (kb | ks) != 0);
                    mma_f16(tmem, ad + 2 * ks, ld + 2 * ks, idesc, 1u);
                }
                commit(&empty[s]);
            }
            __syncwarp();
        }
        if (lane == 0) commit(accf);
        __syncwarp();
    } else {
        // ---- epilogue (warps 2-5): TMEM lane quadrant q = warp % 4 ----
        const int q = warp & 3;
        mbar_wait(accf, 0);
        fence_after();
        // the ring is idle now (every MMA, hence every TMA, completed): stage the tile there
        float* stage = reinterpret_cast<float*>(smem) + q * 32 * OUT_LD;
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 32) {
            uint32_t v[32];
            ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(c0), v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            float4* dst = reinterpret_cast<float4*>(stage + lane * OUT_LD + c0);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                dst[j] = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                     __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        }
        __syncwarp();
        const int col = n0 + lane * 4;
        for (int r = 0; r < 32; ++r) {
            const int m = m0 + q * 32 + r;
            if (m >= p.M) break;
            const float4 x = *reinterpret_cast<const float4*>(stage + r * OUT_LD + lane * 4);
            const float xs[4] = {x.x, x.y, x.z, x.w};
            const int64_t o = int64_t(m) * p.N + col;
            if (col + 3 < p.N && (p.N & 3) == 0) {
                if (p.odtype == RTNQ_F32) {
                    *reinterpret_cast<float4*>(static_cast<float*>(p.out) + o) = x;
                } else if (p.odtype == RTNQ_BF16) {
                    const __nv_bfloat162 a = __floats2bfloat162_rn(x.x, x.y), b = __floats2bfloat162_rn(x.z, x.w);
                    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p.out) + o) =
                        make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
                } else {
                    const __half2 a = __floats2half2_rn(x.x, x.y), b = __floats2half2_rn(x.z, x.w);
                    *reinterpret_cast<uint2*>(static_cast<__half*>(p.out) + o) =
                        make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
                }
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (col + e < p.N) store_out(p.out, p.odtype, o + e, xs[e]);
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
    }
}

static bool encode(CUtensorMap* m, const void* base, int64_t rows, int64_t k, int64_t ld_elems) {
    EncodeFn enc = encoder();
    if (!enc) return false;
    const cuuint64_t dims[2] = {cuuint64_t(k), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(ld_elems * 2)};
    const cuuint32_t box[2] = {BK, 128};
    const cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace dtc

// out[m][n] = a . (hi + lo)^T; a [m][k] (row stride lda elements), hi / lo [n][k] (stride ldw),
// 16-bit (bf16 or f16, the same type), strides multiples of 8 elements, 16-byte-aligned bases.
const char* launch_dense_hilo(const void* a, int64_t lda, const void* hi, const void* lo, int64_t ldw, int a_dtype,
                              int64_t m, int64_t n, int64_t k, void* out, int odtype, cudaStream_t st) {
    using namespace dtc;
    if (lda % 8 || ldw % 8) return "dense tensor-core GEMM: row strides must be multiples of 8 elements";
    if (m > (int64_t(1) << 31) - BM || n > (int64_t(1) << 31) - BN) return "dense tensor-core GEMM: too large";
    Params p{};
    if (!encode(&p.ta, a, m, k, lda) || !encode(&p.th, hi, n, k, ldw) || !encode(&p.tl, lo, n, k, ldw))
        return "cuTensorMapEncodeTiled failed";
    p.out = out;
    p.odtype = odtype;
    p.M = int(m), p.N = int(n), p.KB = int((k + BK - 1) / BK);
    auto kern = a_dtype == RTNQ_BF16 ? dense_tc_kernel<true> : dense_tc_kernel<false>;
    static unsigned long long configured[2] = {0, 0};  // per device
    unsigned long long& cf = configured[a_dtype == RTNQ_BF16 ? 1 : 0];
    if (!(cf & current_device_bit())) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
            return "cudaFuncSetAttribute failed";
        cf |= current_device_bit();
    }
    p.MT = int((m + BM - 1) / BM);
    const dim3 grid(unsigned(((n + BN - 1) / BN) * p.MT));
    kern<<<grid, THREADS, SMEM, st>>>(p);
    return cudaGetLastError() == cudaSuccess ? nullptr : "dense tensor-core GEMM launch failed";
}

}  // namespace rtnq_b200
