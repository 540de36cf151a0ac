// quant_native.cu -- one-pass RTN quantize-and-pack straight into the int8-MMA operand layouts
// (the model-load kernels of the two default linears):
//
//   quant_i4_kernel      W4 group 128 -> RTNQ_NATIVE_I4 (+ row-major bytes, f32 / f16 / native
//                        f16 scales), the operand of wgemm_i4.cu
//   quant_rowwise_kernel W8 per-channel (one group per row) -> RTNQ_NATIVE_I8 (+ row-major
//                        bytes and scales), the operand of wgemm_i8.cu
//
// Both read each weight once (16-byte loads, several in flight per thread), reduce the group
// absmax with warp shuffles (per row across the CTA for per-channel), compute the reference
// scale (scale_from_absmax: the f64 quotient rounded up, quant.cpp:49-68) and write whole 8- or
// 16-byte pieces of the destination tiles.  Padding rows and columns of the 128 x 128 tiles are
// written as code 0 by the same launch.
//
// Codes (round half away from zero of v / S, clamped; quant.cpp:24-29) take a fast path of a
// few FP32 operations per weight: y = v * (1/S), b = clamp(y) + 1.5 * 2^23 (so the low bits of
// b are rint(y) in two's complement), and the distance of y from rint(y).  y is within 2^-16 of
// the exact quotient, so rint(y) is the reference's code unless the quotient lies within 2^-15
// (8-bit) / 2^-18 (4-bit) of a half-integer (codes_fast8 explains the clamp at the ends of the
// range, where the group's absmax element sits).  A warp with any such weight -- or a non-finite
// one, or a scale below 2^-64 -- redoes its weights with quantize_fast (exact FMA tie tests),
// which also raises *err |= 1 for non-finite weights (InvalidInputError, quant.cpp:50-55).
#include <float.h>

#include "../common.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {

namespace {

// 8 consecutive elements of dtype DT: one 16-byte load (bf16/f16) or two (f32)
template <int DT>
struct Raw8 {
    uint4 a, b;
    __device__ __forceinline__ void load(const void* w, int64_t idx) {
        if constexpr (DT == RTNQ_F32) {
            const uint4* p = reinterpret_cast<const uint4*>(static_cast<const float*>(w) + idx);
            a = __ldg(p), b = __ldg(p + 1);
        } else {
            a = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(w) + idx));
        }
    }
    __device__ __forceinline__ void zero() { a = b = make_uint4(0, 0, 0, 0); }
    __device__ __forceinline__ void get(float (&v)[8]) const {
        if constexpr (DT == RTNQ_F32) {
            v[0] = __uint_as_float(a.x), v[1] = __uint_as_float(a.y), v[2] = __uint_as_float(a.z);
            v[3] = __uint_as_float(a.w), v[4] = __uint_as_float(b.x), v[5] = __uint_as_float(b.y);
            v[6] = __uint_as_float(b.z), v[7] = __uint_as_float(b.w);
        } else {
            const uint32_t u[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if constexpr (DT == RTNQ_BF16) {
                    v[2 * i] = __uint_as_float(u[i] << 16);
                    v[2 * i + 1] = __uint_as_float(u[i] & 0xFFFF0000u);
                } else {
                    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&u[i]));
                    v[2 * i] = f.x, v[2 * i + 1] = f.y;
                }
            }
        }
    }
};

// Largest magnitude of a Raw8 as an order-preserving integer key (the |value| bits: 16-bit for
// bf16 / f16, two lanes per word reduced with __vmaxu2; 32-bit for f32).  NaN keys sort above
// inf, so one compare of the reduced key detects any non-finite weight of a group.
template <int DT>
__device__ __forceinline__ uint32_t mag_key(const Raw8<DT>& r) {
    if constexpr (DT == RTNQ_F32) {
        const uint32_t m = 0x7FFFFFFFu;
        return max(max(max(r.a.x & m, r.a.y & m), max(r.a.z & m, r.a.w & m)),
                   max(max(r.b.x & m, r.b.y & m), max(r.b.z & m, r.b.w & m)));
    } else {
        const uint32_t m = 0x7FFF7FFFu;
        const uint32_t x = __vmaxu2(__vmaxu2(r.a.x & m, r.a.y & m), __vmaxu2(r.a.z & m, r.a.w & m));
        return max(x & 0xFFFFu, x >> 16);
    }
}
template <int DT>
__device__ __forceinline__ bool key_nonfinite(uint32_t k) {
    return DT == RTNQ_F32 ? k >= 0x7F800000u : DT == RTNQ_BF16 ? k >= 0x7F80u : k >= 0x7C00u;
}
template <int DT>
__device__ __forceinline__ float key_value(uint32_t k) {  // finite keys only
    if constexpr (DT == RTNQ_F32) return __uint_as_float(k);
    else if constexpr (DT == RTNQ_BF16) return __uint_as_float(k << 16);
    else return __half2float(__ushort_as_half(static_cast<unsigned short>(k)));
}

// Fast path: q[i] low bits = the code of v[i] (two's complement, from the packed-FP32 rint of
// y = v / S); returns max(dmax, |y - rint(y)|) over the 8 weights -- the caller takes the exact
// path for the warp if any lane's maximum comes within the margin of 0.5 (a near-tie).  y is
// clamped to [kLo, qmax] first: above qmax - 0.5 + margin the code is qmax whatever the
// rounding, and below -(qmax + 0.5) + 2 margin it is -qmax unless the quotient is exactly
// -(qmax + 0.5), which only v == -absmax can reach when absmax == (qmax + 0.5) S exactly
// (neg_top; fixed up by the caller).  So a group's absmax element never forces the exact path.
template <int BITS>
struct FastQ {
    static constexpr float kMax = float((1 << (BITS - 1)) - 1);
    static constexpr float kMargin = BITS == 4 ? 1.0f / 262144.0f : 1.0f / 32768.0f;
    static constexpr float kThr = 0.5f - kMargin, kLo = -kMax - 0.5f + 2.0f * kMargin;
    static constexpr uint32_t kMinBits = 0x4B400000u - (1u << (BITS - 1));  // bits of b for qmin
};
// element pair i of a Raw8 as a float2 (built in place: the packed FP32 ops read register pairs)
template <int DT>
__device__ __forceinline__ float2 pair(const Raw8<DT>& r, int i) {
    if constexpr (DT == RTNQ_F32) {
        const uint32_t w[8] = {r.a.x, r.a.y, r.a.z, r.a.w, r.b.x, r.b.y, r.b.z, r.b.w};
        return make_float2(__uint_as_float(w[2 * i]), __uint_as_float(w[2 * i + 1]));
    } else {
        const uint32_t w[4] = {r.a.x, r.a.y, r.a.z, r.a.w};
        if constexpr (DT == RTNQ_BF16)
            return make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xFFFF0000u));
        else
            return __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
    }
}
template <int BITS, int DT>
__device__ __forceinline__ float codes_fast8(const Raw8<DT>& r, float inv, uint32_t (&q)[8], float dmax) {
    using F = FastQ<BITS>;
    const float2 inv2 = make_float2(inv, inv), mg = make_float2(12582912.0f, 12582912.0f);
    const float2 m1 = make_float2(-1.0f, -1.0f);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 y = __fmul2_rn(pair(r, i), inv2);
        const float2 yc = make_float2(fminf(fmaxf(y.x, F::kLo), F::kMax), fminf(fmaxf(y.y, F::kLo), F::kMax));
        const float2 b = __fadd2_rn(yc, mg);           // 1.5 * 2^23 + rint(yc)
        const float2 d = __fadd2_rn(yc, __ffma2_rn(b, m1, mg));  // yc - rint(yc), exact
        dmax = fmaxf(dmax, fmaxf(fabsf(d.x), fabsf(d.y)));
        q[2 * i] = __float_as_uint(b.x), q[2 * i + 1] = __float_as_uint(b.y);
    }
    return dmax;
}

// -absmax if the group's quotient range reaches exactly -(qmax + 0.5), else NaN (see above)
template <int BITS>
__device__ __forceinline__ float neg_top(float amax, float s) {
    constexpr float kTop = float(1 << (BITS - 1)) - 0.5f;
    return __fmaf_rn(-kTop, s, amax) == 0.0f ? -amax : __int_as_float(0x7fc00000);
}

// Exact path: the reference's codes via the FMA tie tests; flags non-finite weights.
template <int BITS>
__device__ __forceinline__ bool codes_exact8(const float (&v)[8], const QuantScale& qs, uint32_t (&q)[8]) {
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        bad |= !(fabsf(v[i]) <= FLT_MAX);
        q[i] = uint32_t(quantize_fast<BITS>(v[i] * qs.pre, qs.s, qs.inv));
    }
    return bad;
}

// low bytes of four words -> one word
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

constexpr int kI4Threads = 256;  // 8 lanes per row (16 codes each), 32 rows per pass
#ifndef RTNQ_QI4_PASS
#define RTNQ_QI4_PASS 2
#endif
#ifndef RTNQ_QI4_LPR
#define RTNQ_QI4_LPR 8  // 4 (32 codes per lane) measured 6 % slower: more near-tie passes redone
#endif
#ifndef RTNQ_QI4_MINB  // CTAs per SM the register budget must allow
#define RTNQ_QI4_MINB (RTNQ_QI4_LPR == 4 ? 4 : 6)
#endif
constexpr int kI4Lpr = RTNQ_QI4_LPR;   // lanes per row (4: 32 codes per lane, 8: 16)
constexpr int kI4Pass = RTNQ_QI4_PASS;  // passes per CTA: (256 / kI4Lpr) * kI4Pass rows of one group
static_assert(kI4Lpr == 4 || kI4Lpr == 8, "");
static_assert(128 % (256 / kI4Lpr * kI4Pass) == 0, "a CTA covers a whole divisor of a 128-row tile");

}  // namespace

// grid (cols / 128, ceil(rows / 128) * 128 / (32 kI4Pass)): CTA (x, y) quantizes group x of 32 kI4Pass rows;
// rows >= `rows` (inside the last 128-row tile) only get their zero padding written.
// Lane j of a row holds codes p..p+7 and p+64..p+71 (p = 8j): exactly the 8 NATIVE_I4 bytes
// p..p+7 of the row (high nibble code p+i, low nibble code p+64+i).
#ifdef RTNQ_QI4_COUNT
__device__ unsigned long long g_qi4_count[4];  // warp passes, passes with a near-tie, near-tie lanes
extern "C" int rtnq_qi4_count_read(void* host) {
    return cudaMemcpyFromSymbol(host, g_qi4_count, sizeof(g_qi4_count)) == cudaSuccess ? 0 : 1;
}
#endif
template <int DT>
__global__ void __launch_bounds__(kI4Threads, RTNQ_QI4_MINB)
quant_i4_kernel(const void* __restrict__ w, int64_t rows, int64_t cols, uint8_t* __restrict__ ni4,
                uint8_t* __restrict__ rm, float* __restrict__ s32, uint16_t* __restrict__ s16,
                uint16_t* __restrict__ s16n, int32_t* __restrict__ err) {
    // LPR lanes per row; lane j holds V 8-code vectors of each half: codes p .. p + 8V - 1 and
    // 64 + p .. (p = 8 V j), i.e. exactly the 8V NATIVE_I4 bytes p .. p + 8V - 1 of the row
    constexpr int LPR = kI4Lpr, V = 8 / LPR, RPP = kI4Threads / LPR;  // rows per pass
    const int t = threadIdx.x, lane = t & 31, j = t & (LPR - 1), p = 8 * V * j;
    const int64_t grp = blockIdx.x, gpr = cols / 128;
    const int64_t row0 = int64_t(blockIdx.y) * (kI4Pass * RPP) + t / LPR;
    Raw8<DT> lo[kI4Pass][V], hi[kI4Pass][V];
#pragma unroll
    for (int s = 0; s < kI4Pass; ++s) {  // all loads first
        const int64_t r = row0 + s * RPP;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            if (r < rows) {
                const int64_t base = r * cols + grp * 128 + p + 8 * v;
                lo[s][v].load(w, base);
                hi[s][v].load(w, base + 64);
            } else {
                lo[s][v].zero(), hi[s][v].zero();
            }
        }
    }
    // group absmax keys of every pass (LPR lanes per row); then lane j computes the scale of pass
    // j % kI4Pass once -- the f64 division runs once per lane group for all its passes -- and the
    // row's lanes fetch theirs
    uint32_t keys[kI4Pass];
#pragma unroll
    for (int s = 0; s < kI4Pass; ++s) {
        uint32_t key = 0;
#pragma unroll
        for (int v = 0; v < V; ++v) key = max(key, max(mag_key(lo[s][v]), mag_key(hi[s][v])));
#pragma unroll
        for (int o = 1; o < LPR; o <<= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
        keys[s] = key;
    }
    uint32_t mykey = keys[0];
#pragma unroll
    for (int s = 1; s < kI4Pass; ++s) mykey = (j % kI4Pass) == s ? keys[s] : mykey;
    const float mym = key_nonfinite<DT>(mykey) ? 0.0f : key_value<DT>(mykey);
    const float mysc = scale_from_absmax(mym, 4);
    const QuantScale myqs = quant_scale_prep(mysc);
    bool bad = false;
#pragma unroll
    for (int s = 0; s < kI4Pass; ++s) {
        const int64_t r = row0 + s * RPP;
        const int src = (lane & ~(LPR - 1)) | (s % LPR);
        const bool nonfinite = key_nonfinite<DT>(keys[s]);
        const float m = nonfinite ? 0.0f : key_value<DT>(keys[s]);
        const float sc = __shfl_sync(0xffffffffu, mysc, src);
        QuantScale qs;
        qs.s = __shfl_sync(0xffffffffu, myqs.s, src);
        qs.inv = __shfl_sync(0xffffffffu, myqs.inv, src);
        qs.pre = __shfl_sync(0xffffffffu, myqs.pre, src);
        uint32_t ql[V][8], qh[V][8];
        float dm = 0.0f;
#pragma unroll
        for (int v = 0; v < V; ++v) dm = codes_fast8<4>(hi[s][v], qs.inv, qh[v], codes_fast8<4>(lo[s][v], qs.inv, ql[v], dm));
        // a warp holding any near-tie, a non-finite weight or a tiny scale redoes its weights
        // exactly.  Near-ties are common for bf16 weights: an absmax mantissa of 1.25, 1.5, ...
        // puts v / S within 2^-23 of half-integers (S = RU(absmax / 7.5)), ~2e-3 of the weights
        // and 57 % of the warp passes of random bf16 weights (scratch/qi4_count.py, build with
        // -DRTNQ_QI4_COUNT); the exact redo costs ~25 % of the kernel.  Measured slower: redoing
        // only the flagged weights (code size), a one-sided midpoint test on flagged passes or on
        // every weight (register spills / per-weight integer work), a non-inlined exact path.
#ifdef RTNQ_QI4_COUNT
        if (lane == 0) atomicAdd(&g_qi4_count[0], 1ull);
        {
            const unsigned tie = __ballot_sync(0xffffffffu, !(dm < FastQ<4>::kThr));
            if (lane == 0 && tie) atomicAdd(&g_qi4_count[1], 1ull);
            if (lane == 0) atomicAdd(&g_qi4_count[2], static_cast<unsigned long long>(__popc(tie)));
        }
#endif
        if (__any_sync(0xffffffffu, !(dm < FastQ<4>::kThr) || nonfinite || qs.pre != 1.0f)) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                float vl[8], vh[8];
                lo[s][v].get(vl), hi[s][v].get(vh);
                bad |= codes_exact8<4>(vl, qs, ql[v]);
                bad |= codes_exact8<4>(vh, qs, qh[v]);
            }
        } else {
            const float nt = neg_top<4>(m, sc);
            if (__any_sync(0xffffffffu, nt == nt)) {  // absmax == 7.5 S exactly: -absmax -> -8
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    float vl[8], vh[8];
                    lo[s][v].get(vl), hi[s][v].get(vh);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        ql[v][i] = vl[i] == nt ? FastQ<4>::kMinBits : ql[v][i];
                        qh[v][i] = vh[i] == nt ? FastQ<4>::kMinBits : qh[v][i];
                    }
                }
            }
        }
        uint32_t L[V][2], H[V][2];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            L[v][0] = pack4(ql[v][0], ql[v][1], ql[v][2], ql[v][3]), L[v][1] = pack4(ql[v][4], ql[v][5], ql[v][6], ql[v][7]);
            H[v][0] = pack4(qh[v][0], qh[v][1], qh[v][2], qh[v][3]), H[v][1] = pack4(qh[v][4], qh[v][5], qh[v][6], qh[v][7]);
        }
        if (ni4) {  // byte i = code(p + i) << 4 | code(p + 64 + i) & 15
            uint32_t b[2 * V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                b[2 * v] = ((L[v][0] << 4) & 0xF0F0F0F0u) | (H[v][0] & 0x0F0F0F0Fu);
                b[2 * v + 1] = ((L[v][1] << 4) & 0xF0F0F0F0u) | (H[v][1] & 0x0F0F0F0Fu);
            }
            const int64_t rr = r & 127, tile = (r >> 7) * gpr + grp;
            uint8_t* dst = ni4 + tile * 8192 + rr * 64;
            if constexpr (V == 2) {  // one whole 16-byte chunk: chunk j
                *reinterpret_cast<uint4*>(dst + ((j ^ ((rr >> 1) & 3)) << 4)) = make_uint4(b[0], b[1], b[2], b[3]);
            } else {                 // half a chunk: chunk j / 2, half j % 2
                *reinterpret_cast<uint2*>(dst + (((j >> 1) ^ ((rr >> 1) & 3)) << 4) + ((j & 1) << 3)) =
                    make_uint2(b[0], b[1]);
            }
        }
        if (r < rows) {
            if (rm) {  // offset binary (packing.cpp:24-30): element 2i low nibble, 2i+1 high
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const uint32_t e0 = __byte_perm(L[v][0], L[v][1], 0x6420), o0 = __byte_perm(L[v][0], L[v][1], 0x7531);
                    const uint32_t e1 = __byte_perm(H[v][0], H[v][1], 0x6420), o1 = __byte_perm(H[v][0], H[v][1], 0x7531);
                    uint8_t* dst = rm + ((r * cols + grp * 128 + p + 8 * v) >> 1);
                    *reinterpret_cast<uint32_t*>(dst) = ((e0 & 0x0F0F0F0Fu) | ((o0 << 4) & 0xF0F0F0F0u)) ^ 0x88888888u;
                    *reinterpret_cast<uint32_t*>(dst + 32) = ((e1 & 0x0F0F0F0Fu) | ((o1 << 4) & 0xF0F0F0F0u)) ^ 0x88888888u;
                }
            }
            if (j == 0) {
                if (s32) s32[r * gpr + grp] = sc;
                const uint16_t h = __half_as_ushort(__float2half_rn(sc));
                if (s16) s16[r * gpr + grp] = h;
                if (s16n) s16n[native_scale_index(rows, gpr, r, grp)] = h;
            }
        }
    }
    if (err && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 1);
}

constexpr int kRwThreads = 256;
constexpr int kRwHold = 4;  // 16-code chunks per thread kept in registers

// T threads per row, 256 / T rows per CTA; grid covers the rows padded to whole 128-row tiles
// (rows >= `rows` write the zero padding).  Thread lt of a row owns chunks lt, lt + T, ... of
// 16 codes; the first kRwHold stay in registers between the max and the quantize pass, the rest
// (K > 64 T) are read again.
template <int DT, int T>
__global__ void __launch_bounds__(kRwThreads)
quant_rowwise_kernel(const void* __restrict__ w, int64_t rows, int64_t cols, uint8_t* __restrict__ ni8,
                     uint8_t* __restrict__ rm, float* __restrict__ s32, uint16_t* __restrict__ s16,
                     uint16_t* __restrict__ s16n, int32_t* __restrict__ err) {
    constexpr int R = kRwThreads / T, WPR = T / 32;
    __shared__ uint32_t wkey[kRwThreads / 32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, lt = t % T, rw = t / T;
    const int64_t r = int64_t(blockIdx.x) * R + rw;
    const int64_t nch = cols / 16, kt = (cols + 127) / 128, nchp = kt * 8;  // chunks, padded
    const bool live = r < rows;
    const int64_t rbase = r * cols;
    Raw8<DT> v[kRwHold][2];
    uint32_t key = 0;
#pragma unroll
    for (int jj = 0; jj < kRwHold; ++jj) {
        const int64_t ch = lt + int64_t(jj) * T;
        if (live && ch < nch) {
            v[jj][0].load(w, rbase + ch * 16);
            v[jj][1].load(w, rbase + ch * 16 + 8);
        } else {
            v[jj][0].zero(), v[jj][1].zero();
        }
    }
#pragma unroll
    for (int jj = 0; jj < kRwHold; ++jj) key = max(key, max(mag_key(v[jj][0]), mag_key(v[jj][1])));
    for (int64_t ch = lt + int64_t(kRwHold) * T; live && ch < nch; ch += T) {
        Raw8<DT> x0, x1;  // past the register window: max-reduce now, read again below
        x0.load(w, rbase + ch * 16);
        x1.load(w, rbase + ch * 16 + 8);
        key = max(key, max(mag_key(x0), mag_key(x1)));
    }
    for (int o = 16; o; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
    if (lane == 0) wkey[warp] = key;
    __syncthreads();
    uint32_t rkey = 0;
#pragma unroll
    for (int i = 0; i < WPR; ++i) rkey = max(rkey, wkey[rw * WPR + i]);
    const bool nonfinite = key_nonfinite<DT>(rkey);
    const float amax = nonfinite ? 0.0f : key_value<DT>(rkey);
    const float sc = scale_from_absmax(amax, 8);
    const QuantScale qs = quant_scale_prep(sc);
    const float nt = neg_top<8>(amax, sc);
    if (live && lt == 0) {
        if (s32) s32[r] = sc;
        const uint16_t h = __half_as_ushort(__float2half_rn(sc));
        if (s16) s16[r] = h;
        if (s16n) s16n[native_scale_index(rows, 1, r, 0)] = h;
    }
    const int64_t rr = r & 127, tile0 = (r >> 7) * kt;
    bool bad = false;
    // every lane of a warp runs the same number of chunks (warp-uniform slow-path vote)
    auto emit = [&](int64_t ch, const Raw8<DT>& x0, const Raw8<DT>& x1) {
        uint32_t qa[8], qb[8];
        const float dm = codes_fast8<8>(x1, qs.inv, qb, codes_fast8<8>(x0, qs.inv, qa, 0.0f));
        if (__any_sync(0xffffffffu, !(dm < FastQ<8>::kThr) || nonfinite || qs.pre != 1.0f)) {
            float a[8], b[8];
            x0.get(a), x1.get(b);
            bad |= codes_exact8<8>(a, qs, qa);
            bad |= codes_exact8<8>(b, qs, qb);
        } else if (__any_sync(0xffffffffu, nt == nt)) {  // absmax == 127.5 S exactly: -absmax -> -128
            float a[8], b[8];
            x0.get(a), x1.get(b);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                qa[i] = a[i] == nt ? FastQ<8>::kMinBits : qa[i];
                qb[i] = b[i] == nt ? FastQ<8>::kMinBits : qb[i];
            }
        }
        const bool real = live && ch < nch;
        uint4 q = make_uint4(pack4(qa[0], qa[1], qa[2], qa[3]), pack4(qa[4], qa[5], qa[6], qa[7]),
                             pack4(qb[0], qb[1], qb[2], qb[3]), pack4(qb[4], qb[5], qb[6], qb[7]));
        if (!real) q = make_uint4(0, 0, 0, 0);
        if (ch < nchp && ni8)
            *reinterpret_cast<uint4*>(ni8 + (tile0 + (ch >> 3)) * 16384 + rr * 128 + (((ch & 7) ^ (rr & 7)) << 4)) = q;
        if (rm && real)  // offset binary (packing.cpp:19-22): two's complement ^ 0x80
            *reinterpret_cast<uint4*>(rm + rbase + ch * 16) =
                make_uint4(q.x ^ 0x80808080u, q.y ^ 0x80808080u, q.z ^ 0x80808080u, q.w ^ 0x80808080u);
    };
#pragma unroll
    for (int jj = 0; jj < kRwHold; ++jj) emit(lt + int64_t(jj) * T, v[jj][0], v[jj][1]);
    const int64_t rounds = (nchp + T - 1) / T;  // the same for every lane
    for (int64_t jj = kRwHold; jj < rounds; ++jj) {
        const int64_t ch = lt + jj * T;
        Raw8<DT> x0, x1;
        if (live && ch < nch) {
            x0.load(w, rbase + ch * 16);
            x1.load(w, rbase + ch * 16 + 8);
        } else {
            x0.zero(), x1.zero();
        }
        emit(ch, x0, x1);
    }
    if (err && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 1);
}

bool quant_i4_supported(int64_t rows, int64_t cols, int bits, int64_t g) {
    return bits == 4 && g == 128 && rows > 0 && cols > 0 && cols % 128 == 0 && (rows + 127) / 128 * 4 <= 65535;
}

bool quant_rowwise_supported(int64_t rows, int64_t cols, int bits, int64_t g) {
    return bits == 8 && g >= cols && rows > 0 && cols > 0 && cols % 16 == 0 && (rows + 127) / 128 * 128 <= INT32_MAX;
}

void launch_quant_i4(const void* w, int dtype, int64_t rows, int64_t cols, uint8_t* ni4, uint8_t* rm, float* s32,
                     uint16_t* s16, uint16_t* s16n, int32_t* err, cudaStream_t st) {
    const dim3 grid(unsigned(cols / 128), unsigned((rows + 127) / 128 * (128 / (kI4Threads / kI4Lpr * kI4Pass))));
    if (dtype == RTNQ_F32) quant_i4_kernel<RTNQ_F32><<<grid, kI4Threads, 0, st>>>(w, rows, cols, ni4, rm, s32, s16, s16n, err);
    else if (dtype == RTNQ_F16) quant_i4_kernel<RTNQ_F16><<<grid, kI4Threads, 0, st>>>(w, rows, cols, ni4, rm, s32, s16, s16n, err);
    else quant_i4_kernel<RTNQ_BF16><<<grid, kI4Threads, 0, st>>>(w, rows, cols, ni4, rm, s32, s16, s16n, err);
}

template <int DT>
static void launch_rowwise_dt(const void* w, int64_t rows, int64_t cols, uint8_t* ni8, uint8_t* rm, float* s32,
                              uint16_t* s16, uint16_t* s16n, int32_t* err, cudaStream_t st) {
    const int64_t prow = (rows + 127) / 128 * 128, nch = cols / 16;
    // threads per row: the fewest that keep the row in the register window, else 256
    if (nch <= 64 * kRwHold)
        quant_rowwise_kernel<DT, 64><<<unsigned(prow / 4), kRwThreads, 0, st>>>(w, rows, cols, ni8, rm, s32, s16, s16n, err);
    else if (nch <= 128 * kRwHold)
        quant_rowwise_kernel<DT, 128><<<unsigned(prow / 2), kRwThreads, 0, st>>>(w, rows, cols, ni8, rm, s32, s16, s16n, err);
    else
        quant_rowwise_kernel<DT, 256><<<unsigned(prow), kRwThreads, 0, st>>>(w, rows, cols, ni8, rm, s32, s16, s16n, err);
}

void launch_quant_rowwise(const void* w, int dtype, int64_t rows, int64_t cols, uint8_t* ni8, uint8_t* rm,
                          float* s32, uint16_t* s16, uint16_t* s16n, int32_t* err, cudaStream_t st) {
    if (dtype == RTNQ_F32) launch_rowwise_dt<RTNQ_F32>(w, rows, cols, ni8, rm, s32, s16, s16n, err, st);
    else if (dtype == RTNQ_F16) launch_rowwise_dt<RTNQ_F16>(w, rows, cols, ni8, rm, s32, s16, s16n, err, st);
    else launch_rowwise_dt<RTNQ_BF16>(w, rows, cols, ni8, rm, s32, s16, s16n, err, st);
}

}  // namespace rtnq_b200
