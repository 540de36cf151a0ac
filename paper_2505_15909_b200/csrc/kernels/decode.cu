// decode.cu -- the non-GEMM kernels of one decode layer (toy.cpp:91-117,
// generalized to Llama-3.1: GQA, RoPE, a KV cache): fused residual-add + RMSNorm,
// decode attention over the cache, SiLU-gated FFN activation.  All bf16 in HBM, f32
// math.  These are small next to the weight stream and are written for
// HBM efficiency: 16-byte loads, one pass over the data.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cstdlib>
#include <mutex>

#include "int8_mma.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {
namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Ready to run as a PDL secondary: lets its successor launch right away (every successor waits
// for this grid's completion before it reads what this grid writes), then waits for its
// predecessor before touching memory.  A no-op when launched stream-ordered (launch_pdl).
__device__ __forceinline__ void pdl_prologue() {
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// x <- x + delta (if delta), out <- rmsnorm(x) * w.  One CTA per token row (toy.cpp:19-30:
// mean of squares, 1/sqrt(ms + eps), times the norm weight).
__global__ void add_rmsnorm_kernel(__nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ delta,
                                   const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ out,
                                   int h, float eps, int8_t* __restrict__ planes, int32_t* __restrict__ texp) {
    pdl_prologue();
    extern __shared__ float red[];
    const int row = blockIdx.x;
    __nv_bfloat16* xr = x + int64_t(row) * h;
    const __nv_bfloat16* dr = delta ? delta + int64_t(row) * h : nullptr;
    float ss = 0.0f;
    for (int i = threadIdx.x * 8; i < h; i += blockDim.x * 8) {
        uint4 xv = *reinterpret_cast<const uint4*>(xr + i);
        __nv_bfloat162* xp = reinterpret_cast<__nv_bfloat162*>(&xv);
        if (dr) {
            const uint4 dv = *reinterpret_cast<const uint4*>(dr + i);
            const __nv_bfloat162* dp = reinterpret_cast<const __nv_bfloat162*>(&dv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 a = __bfloat1622float2(xp[j]), b = __bfloat1622float2(dp[j]);
                xp[j] = __floats2bfloat162_rn(a.x + b.x, a.y + b.y);
            }
            *reinterpret_cast<uint4*>(xr + i) = xv;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 a = __bfloat1622float2(xp[j]);
            ss += a.x * a.x + a.y * a.y;
        }
    }
    ss = warp_sum(ss);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    if (warp == 0) {
        float v = lane < nw ? red[lane] : 0.0f;
        v = warp_sum(v);
        if (lane == 0) red[0] = rsqrtf(v / float(h) + eps);
    }
    __syncthreads();
    const float inv = red[0];
    for (int i = threadIdx.x * 8; i < h; i += blockDim.x * 8) {
        const uint4 xv = *reinterpret_cast<const uint4*>(xr + i);
        const uint4 wv = *reinterpret_cast<const uint4*>(w + i);
        const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&xv);
        const __nv_bfloat162* wp = reinterpret_cast<const __nv_bfloat162*>(&wv);
        uint4 ov;
        __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&ov);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 a = __bfloat1622float2(xp[j]), b = __bfloat1622float2(wp[j]);
            op[j] = __floats2bfloat162_rn(a.x * inv * b.x, a.y * inv * b.y);
        }
        *reinterpret_cast<uint4*>(out + int64_t(row) * h + i) = ov;
    }
    if (planes) {  // the int8 GEMMs' activation planes of this output row, straight away
        __syncthreads();
        imma::row_to_planes(reinterpret_cast<const uint16_t*>(out + int64_t(row) * h), h, row, gridDim.x,
                            planes, texp);
    }
}

// ---- register-resident row kernels (one CTA per token row; every element loaded once) -------
// The row stays in registers (VPT 16-byte vectors per thread) across the passes: sum of squares
// (or max) -> scale -> output -> activation planes of the output, so a row costs one DRAM round
// trip plus two block reductions instead of a load per pass.
constexpr int kRowThreads = 256;

// Sum (or max) over the CL CTAs of a row's thread-block cluster: block reduction, then every CTA
// reads the CL partials over DSMEM in rank order (deterministic, identical in every CTA).
template <int CL>
__device__ __forceinline__ float row_reduce(float v, float* red, float* cpart, bool is_max) {
    v = is_max ? warp_max(v) : warp_sum(v);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();  // red / cpart are reused across calls
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = 0.0f;
#pragma unroll
    for (int i = 0; i < kRowThreads / 32; ++i) r = is_max ? fmaxf(r, red[i]) : r + red[i];
    if constexpr (CL == 1) return r;
    if (threadIdx.x == 0) *cpart = r;
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const uint32_t my = static_cast<uint32_t>(__cvta_generic_to_shared(cpart));
    float t = 0.0f;
#pragma unroll
    for (int q = 0; q < CL; ++q) {
        uint32_t ra;
        float x;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(my), "r"(q));
        asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x) : "r"(ra));
        t = is_max ? fmaxf(t, x) : t + x;
    }
    // the peers' cpart may be rewritten by the next reduction only after every CTA has read it
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    return t;
}

// vector v of this thread: CTA `rank` of the row's CL takes vectors rank * 256 + tid + v * 256 * CL
template <int CL>
__device__ __forceinline__ int row_vec(int rank, int v) { return rank * kRowThreads + threadIdx.x + v * kRowThreads * CL; }

// planes of a bf16 row held as VPT vectors per thread (row_to_planes' arithmetic, bit-identical)
template <int VPT, int CL>
__device__ __forceinline__ void planes_from_regs(const uint4 (&ov)[VPT], int n8, int rank, int t, int M, int K,
                                                 int8_t* __restrict__ planes, int32_t* __restrict__ texp,
                                                 float* red, float* cpart) {
    auto cvt = [](uint32_t h) -> float { return __uint_as_float(h << 16); };
    float mx = 0.0f;
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
        if (row_vec<CL>(rank, v) >= n8) break;
        const uint32_t w[4] = {ov[v].x, ov[v].y, ov[v].z, ov[v].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) mx = fmaxf(mx, fmaxf(fabsf(cvt(w[i] & 0xffffu)), fabsf(cvt(w[i] >> 16))));
    }
    const float amax = row_reduce<CL>(mx, red, cpart, true);
    int e = 0;
    if (amax > 0.0f) frexpf(amax, &e);
    const int s = max(e - 6, -126);
    if (threadIdx.x == 0 && rank == 0) texp[t] = s;
    const float inv = __int_as_float((127 - s) << 23);
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
        const int vi = row_vec<CL>(rank, v);
        if (vi >= n8) break;
        const uint32_t w[4] = {ov[v].x, ov[v].y, ov[v].z, ov[v].w};
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
            *reinterpret_cast<uint2*>(planes + (int64_t(pl) * M + t) * K + int64_t(vi) * 8) =
                make_uint2(pk[pl][0], pk[pl][1]);
    }
}

// grid (m * CL): a thread-block cluster of CL CTAs per token row
template <int VPT, int CL>
__global__ void __launch_bounds__(kRowThreads) add_rmsnorm_rows_kernel(
    __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ delta, const __nv_bfloat16* __restrict__ w,
    __nv_bfloat16* __restrict__ out, int h, float eps, int8_t* __restrict__ planes, int32_t* __restrict__ texp,
    PeerIn pin) {
    pdl_prologue();
    __shared__ float red[kRowThreads / 32];
    __shared__ float cpart;
    const int row = blockIdx.x / CL, rank = blockIdx.x % CL, n8 = h / 8;
    __nv_bfloat16* xr = x + int64_t(row) * h;
    const __nv_bfloat16* dr = delta ? delta + int64_t(row) * h : nullptr;
    uint4 xv[VPT], dv[VPT];
    if (pin.buf) {  // tensor parallel: delta = sum of every rank's partial of this round
        const int e = *reinterpret_cast<volatile int*>(imma::peer_epoch(pin.buf)) + 1;
        if (threadIdx.x == 0) imma::peer_wait(pin.buf, pin.world, e);
        __syncthreads();
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            const int vi = row_vec<CL>(rank, v);
            if (vi < n8) {
                xv[v] = *reinterpret_cast<const uint4*>(xr + vi * 8);
                float acc[8] = {};
                for (int q = 0; q < pin.world; ++q) {
                    const uint4 sv = imma::peer_ld16(imma::peer_slot(pin.buf, pin.cap, e & 1, q) + int64_t(row) * h + vi * 8);
                    const __nv_bfloat162* sp = reinterpret_cast<const __nv_bfloat162*>(&sv);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float2 f = __bfloat1622float2(sp[j]);
                        acc[2 * j] += f.x, acc[2 * j + 1] += f.y;
                    }
                }
                __nv_bfloat162* dp = reinterpret_cast<__nv_bfloat162*>(&dv[v]);
#pragma unroll
                for (int j = 0; j < 4; ++j) dp[j] = __floats2bfloat162_rn(acc[2 * j], acc[2 * j + 1]);
            }
        }
    } else {
#pragma unroll
        for (int v = 0; v < VPT; ++v) {  // every load of the row in flight at once
            const int vi = row_vec<CL>(rank, v);
            if (vi < n8) {
                xv[v] = *reinterpret_cast<const uint4*>(xr + vi * 8);
                if (dr) dv[v] = *reinterpret_cast<const uint4*>(dr + vi * 8);
            }
        }
    }
    const bool has_d = dr || pin.buf;
    float ss = 0.0f;
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
        const int vi = row_vec<CL>(rank, v);
        if (vi >= n8) break;
        __nv_bfloat162* xp = reinterpret_cast<__nv_bfloat162*>(&xv[v]);
        if (has_d) {
            const __nv_bfloat162* dp = reinterpret_cast<const __nv_bfloat162*>(&dv[v]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 a = __bfloat1622float2(xp[j]), b = __bfloat1622float2(dp[j]);
                xp[j] = __floats2bfloat162_rn(a.x + b.x, a.y + b.y);
            }
            *reinterpret_cast<uint4*>(xr + vi * 8) = xv[v];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 a = __bfloat1622float2(xp[j]);
            ss += a.x * a.x + a.y * a.y;
        }
    }
    const float inv = rsqrtf(row_reduce<CL>(ss, red, &cpart, false) / float(h) + eps);
    uint4 ov[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
        const int vi = row_vec<CL>(rank, v);
        if (vi >= n8) break;
        const uint4 wv = __ldg(reinterpret_cast<const uint4*>(w + vi * 8));
        const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&xv[v]);
        const __nv_bfloat162* wp = reinterpret_cast<const __nv_bfloat162*>(&wv);
        __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&ov[v]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 a = __bfloat1622float2(xp[j]), b = __bfloat1622float2(wp[j]);
            op[j] = __floats2bfloat162_rn(a.x * inv * b.x, a.y * inv * b.y);
        }
        *reinterpret_cast<uint4*>(out + int64_t(row) * h + vi * 8) = ov[v];
    }
    if (planes) planes_from_regs<VPT, CL>(ov, n8, rank, row, gridDim.x / CL, h, planes, texp, red, &cpart);
    if (pin.buf) {  // this CTA's reads of the round are done
        __syncthreads();
        if (threadIdx.x == 0) imma::peer_consumed_by(pin.buf, int(gridDim.x));
    }
}

template <int VPT, int CL>
__global__ void __launch_bounds__(kRowThreads) silu_mul_rows_kernel(const __nv_bfloat16* __restrict__ gu,
                                                                    __nv_bfloat16* __restrict__ act, int f,
                                                                    int8_t* __restrict__ planes,
                                                                    int32_t* __restrict__ texp) {
    pdl_prologue();
    __shared__ float red[kRowThreads / 32];
    __shared__ float cpart;
    const int t = blockIdx.x / CL, rank = blockIdx.x % CL, n8 = f / 8;
    const __nv_bfloat16* gr = gu + int64_t(t) * 2 * f;
    uint4 gv[VPT], uv[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
        const int vi = row_vec<CL>(rank, v);
        if (vi < n8) {
            gv[v] = *reinterpret_cast<const uint4*>(gr + vi * 8);
            uv[v] = *reinterpret_cast<const uint4*>(gr + f + vi * 8);
        }
    }
    uint4 ov[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
        const int vi = row_vec<CL>(rank, v);
        if (vi >= n8) break;
        const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&gv[v]);
        const __nv_bfloat162* up = reinterpret_cast<const __nv_bfloat162*>(&uv[v]);
        __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&ov[v]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 g = __bfloat1622float2(gp[q]), u = __bfloat1622float2(up[q]);
            op[q] = __floats2bfloat162_rn(g.x / (1.0f + __expf(-g.x)) * u.x, g.y / (1.0f + __expf(-g.y)) * u.y);
        }
        *reinterpret_cast<uint4*>(act + int64_t(t) * f + vi * 8) = ov[v];
    }
    if (planes) planes_from_regs<VPT, CL>(ov, n8, rank, t, gridDim.x / CL, f, planes, texp, red, &cpart);
}

// cluster-launched row kernel: cluster of CL CTAs per row, VPT vectors per thread
template <typename... KArgs, typename... Args>
cudaError_t launch_rows(void (*kern)(KArgs...), int64_t m, int cl, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(m * cl));
    cfg.blockDim = dim3(kRowThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = unsigned(cl);
    attr.val.clusterDim.y = attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = cl > 1 ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// CTAs per row (cluster size): enough that ~all SMs share the rows, at most 8 (portable)
static int row_cluster(int64_t m, int64_t n8) {
    int cl = 1;
    while (cl < 8 && m * cl * 2 <= 148 && n8 > 2 * int64_t(cl) * kRowThreads) cl *= 2;
    return cl;
}

// One CTA per token: the SiLU*up row, then its activation planes (row_to_planes).
__global__ void silu_mul_planes_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ act,
                                       int f, int8_t* __restrict__ planes, int32_t* __restrict__ texp) {
    pdl_prologue();
    const int t = blockIdx.x;
    for (int j = threadIdx.x * 8; j < f; j += blockDim.x * 8) {
        const uint4 gv = *reinterpret_cast<const uint4*>(gu + int64_t(t) * 2 * f + j);
        const uint4 uv = *reinterpret_cast<const uint4*>(gu + int64_t(t) * 2 * f + f + j);
        const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&gv);
        const __nv_bfloat162* up = reinterpret_cast<const __nv_bfloat162*>(&uv);
        uint4 ov;
        __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&ov);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 g = __bfloat1622float2(gp[q]), u = __bfloat1622float2(up[q]);
            op[q] = __floats2bfloat162_rn(g.x / (1.0f + __expf(-g.x)) * u.x,
                                          g.y / (1.0f + __expf(-g.y)) * u.y);
        }
        *reinterpret_cast<uint4*>(act + int64_t(t) * f + j) = ov;
    }
    __syncthreads();
    imma::row_to_planes(reinterpret_cast<const uint16_t*>(act + int64_t(t) * f), f, t, gridDim.x, planes, texp);
}

// act[t][j] = silu(gu[t][j]) * gu[t][f + j]: gate in columns [0, f), up in [f, 2f)
// (toy.cpp:108-112 keeps the same fused [gate | up] output).
__global__ void silu_mul_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ act,
                                int64_t m, int f) {
    pdl_prologue();
    const int64_t n8 = m * f / 8;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t e = i * 8, t = e / f, j = e % f;
        const uint4 gv = *reinterpret_cast<const uint4*>(gu + t * 2 * f + j);
        const uint4 uv = *reinterpret_cast<const uint4*>(gu + t * 2 * f + f + j);
        const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&gv);
        const __nv_bfloat162* up = reinterpret_cast<const __nv_bfloat162*>(&uv);
        uint4 ov;
        __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&ov);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 g = __bfloat1622float2(gp[q]), u = __bfloat1622float2(up[q]);
            op[q] = __floats2bfloat162_rn(g.x / (1.0f + __expf(-g.x)) * u.x,
                                          g.y / (1.0f + __expf(-g.y)) * u.y);
        }
        *reinterpret_cast<uint4*>(act + e) = ov;
    }
}


// Decode attention for one (token b, kv head): the group's query heads attend over cache
// positions [0, pos] after the new k/v (rotated k) are appended at `pos`.
// qkv row layout: [Hq*D | Hkv*D | Hkv*D] (the column-split QKV output of one rank).
// cache layout: [B][Lmax][Hkv][D] for K and for V.  One CTA = G warps (G = Hq/Hkv <= 32);
// warp w owns query head kvh * G + w; head_dim D = 128.
// Flash-decoding split across CTAs: grid (Hkv, B, nsp), nsp chosen so the grid is ~2 waves of the
// SMs and the context splits evenly (launch_decode_attention).  A CTA stages its chunk's K and V
// rows in shared memory with cp.async (every 16-byte load in flight at once; 256-byte rows whose
// 16-byte chunks are XOR-swizzled by the row, so a lane-per-row walk of 16-byte chunks and a
// row-per-warp walk are both bank-conflict free); each warp scores its positions lane-parallel,
// exponentiates against the chunk max and accumulates P*V (lanes own 4 head dims, 4 chains),
// writing a (max, sum, P*V) partial; the splits merge over DSMEM inside a thread-block cluster
// (nsp <= 8) or through the caller's workspace (the last CTA to arrive):
// out = sum_s e^(m_s - M) acc_s / sum_s e^(m_s - M) l_s.
constexpr int kD = 128;
constexpr int kMaxChunk = 256;  // positions per CTA at most (smem)
constexpr int kPart = kD + 4;   // floats per split partial: max, sum, 2 pad, P*V (16-B aligned)

__device__ __forceinline__ uint32_t swz(int t, int c) { return uint32_t(t * 16 + (c ^ (t & 15))); }  // 16-B chunk

// The end of a split CTA, per warp = query head qh (lane: head dims 4 lane .. 4 lane + 3): its
// (max, sum, unnormalised P.V) partial -> the output (one split), or the DSMEM merge inside the
// cluster (scratch: kPart floats per warp of idle shared memory), or the last-CTA global merge.
__device__ __forceinline__ bool attn_finish(float cmax, float csum, float4 a4, float* scratch, float* __restrict__ part,
                                            int* __restrict__ arrivals, __nv_bfloat16* __restrict__ out, int b,
                                            int kvh, int qh, int hq, int hkv, int sp, int nsp, int cluster_merge) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (nsp == 1) {  // the whole context in this CTA: normalise and write, no merge
        float o[4];
        o[0] = a4.x / csum, o[1] = a4.y / csum, o[2] = a4.z / csum, o[3] = a4.w / csum;
        __nv_bfloat16* op = out + (int64_t(b) * hq + qh) * kD + 4 * lane;
        *reinterpret_cast<__nv_bfloat162*>(op) = __floats2bfloat162_rn(o[0], o[1]);
        *reinterpret_cast<__nv_bfloat162*>(op + 2) = __floats2bfloat162_rn(o[2], o[3]);
        return true;
    }
    if (cluster_merge) {
        // the splits of this (token, KV head) are one thread-block cluster: partials stay in
        // each CTA's shared memory (idle scratch) and rank 0 merges them over DSMEM
        __syncthreads();  // every warp is done reading the staging buffers
        float* mine = scratch + warp * kPart;
        if (lane == 0) mine[0] = cmax, mine[1] = csum;
        *reinterpret_cast<float4*>(mine + 4 + 4 * lane) =
            a4;
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (sp == 0) {
            const uint32_t my = static_cast<uint32_t>(__cvta_generic_to_shared(mine));
            float mq[8], lq[8];
            float M = -INFINITY;
#pragma unroll
            for (int q = 0; q < 8; ++q) {  // nsp <= 8: fixed trip count keeps mq/lq in registers
                if (q >= nsp) break;
                uint32_t ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(my), "r"(q));
                asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(mq[q]) : "r"(ra));
                asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(lq[q]) : "r"(ra + 4));
                M = fmaxf(M, mq[q]);
            }
            float L = 0.0f, a[4] = {0, 0, 0, 0};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q >= nsp) break;
                uint32_t ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(my + uint32_t(16 + 16 * lane)), "r"(q));
                float4 x;
                asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(ra));
                const float w = __expf(mq[q] - M);
                L = fmaf(w, lq[q], L);
                a[0] = fmaf(w, x.x, a[0]), a[1] = fmaf(w, x.y, a[1]), a[2] = fmaf(w, x.z, a[2]), a[3] = fmaf(w, x.w, a[3]);
            }
            const float inv = 1.0f / L;
            __nv_bfloat16* op = out + (int64_t(b) * hq + qh) * kD + 4 * lane;
            *reinterpret_cast<__nv_bfloat162*>(op) = __floats2bfloat162_rn(a[0] * inv, a[1] * inv);
            *reinterpret_cast<__nv_bfloat162*>(op + 2) = __floats2bfloat162_rn(a[2] * inv, a[3] * inv);
        }
        // peers keep their shared memory alive until rank 0 has read it
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        return sp == 0;
    }
    // partial: [b][qh][split] -> {max, sum, acc[kD]}
    float* pr = part + ((int64_t(b) * hq + qh) * nsp + sp) * kPart;
    if (lane == 0) pr[0] = cmax, pr[1] = csum;
    *reinterpret_cast<float4*>(pr + 4 + 4 * lane) =
        a4;
    // the last split CTA of this (token, KV head) merges the partials (self-resetting counter)
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int prev = atomicAdd(arrivals + b * hkv + kvh, 1);
        last = prev == nsp - 1;
        if (last) arrivals[b * hkv + kvh] = 0;
    }
    __syncthreads();
    if (!last) return false;
    __threadfence();
    const float* ph = part + (int64_t(b) * hq + qh) * nsp * kPart;
    float M = -INFINITY;
    for (int q = 0; q < nsp; ++q) M = fmaxf(M, __ldcg(ph + q * kPart));
    float L = 0.0f, a[4] = {0, 0, 0, 0};
    for (int q = 0; q < nsp; ++q) {
        const float w = __expf(__ldcg(ph + q * kPart) - M);
        L = fmaf(w, __ldcg(ph + q * kPart + 1), L);
        const float4 x = __ldcg(reinterpret_cast<const float4*>(ph + q * kPart + 4 + 4 * lane));
        a[0] = fmaf(w, x.x, a[0]), a[1] = fmaf(w, x.y, a[1]), a[2] = fmaf(w, x.z, a[2]), a[3] = fmaf(w, x.w, a[3]);
    }
    const float inv = 1.0f / L;
    __nv_bfloat16* op = out + (int64_t(b) * hq + qh) * kD + 4 * lane;
    *reinterpret_cast<__nv_bfloat162*>(op) = __floats2bfloat162_rn(a[0] * inv, a[1] * inv);
    *reinterpret_cast<__nv_bfloat162*>(op + 2) = __floats2bfloat162_rn(a[2] * inv, a[3] * inv);
    return true;
}

// The o-projection's activation planes from the attention output, in the attention kernel: the
// CTA that wrote the last of a token's hkv head groups (a self-resetting per-token counter)
// computes the token's planes from its whole output row (token_planes: the planes kernel's
// arithmetic), so the o-projection needs no planes kernel of its own.
__device__ __forceinline__ void attn_token_planes(bool wrote, const __nv_bfloat16* __restrict__ out, int b, int hq,
                                                  int hkv, int batch, int* __restrict__ tok_arrivals,
                                                  int8_t* __restrict__ planes, int32_t* __restrict__ texp) {
    __shared__ int tlast;
    __shared__ float red[32];
    if (wrote) __threadfence();  // every writing thread: its rows visible device-wide first
    __syncthreads();             // every warp wrote its head rows
    if (threadIdx.x == 0) {
        tlast = 0;
        if (wrote) {
            const int prev = atomicAdd(tok_arrivals + b, 1);
            tlast = prev == hkv - 1;
            if (tlast) tok_arrivals[b] = 0;
        }
    }
    __syncthreads();
    if (!tlast) return;
    __threadfence();
    imma::token_planes<RTNQ_BF16>(reinterpret_cast<const uint16_t*>(out) + int64_t(b) * hq * kD, hq * kD, b, batch,
                                  planes, texp, nullptr, int(threadIdx.x), int(blockDim.x), 1, red);
}

__global__ void decode_attention_kernel(const __nv_bfloat16* __restrict__ qkv,
                                        __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc,
                                        float* __restrict__ part, int hq, int hkv, int lmax,
                                        int pos, float theta, __nv_bfloat16* __restrict__ out,
                                        int* __restrict__ arrivals, int cluster_merge, int chunk,
                                        int8_t* __restrict__ planes, int32_t* __restrict__ texp,
                                        int* __restrict__ tok_arrivals) {
    // grid (hkv, batch, split): this CTA covers positions [t0, t0 + n) of one KV head and its
    // G query heads (a warp each) and writes the split's (max, sum, unnormalised P.V) partial
    pdl_prologue();
    extern __shared__ uint4 smq[];
    uint4* ks = smq;                          // [chunk][16] swizzled 16-byte chunks
    uint4* vs = ks + chunk * 16;              // [chunk][16]
    float* qs = reinterpret_cast<float*>(vs + chunk * 16);  // [G][kD] rotated, scaled queries
    float* ps = qs + (blockDim.x / 32) * kD;                // [G][chunk] probabilities
    const int b = blockIdx.y, kvh = blockIdx.x, sp = blockIdx.z, nsp = gridDim.z, G = hq / hkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nthr = blockDim.x;
    const int64_t row = int64_t(b) * (hq + 2 * hkv) * kD;
    const __nv_bfloat16* kn = qkv + row + int64_t(hq) * kD + int64_t(kvh) * kD;
    const __nv_bfloat16* vn = kn + int64_t(hkv) * kD;
    const int64_t cstride = int64_t(hkv) * kD;  // between positions
    __nv_bfloat16* kcb = kc + (int64_t(b) * lmax) * cstride + int64_t(kvh) * kD;
    __nv_bfloat16* vcb = vc + (int64_t(b) * lmax) * cstride + int64_t(kvh) * kD;
    const int t0 = sp * chunk, n = min(chunk, pos + 1 - t0);
    // RoPE angles of position `pos`, computed once per CTA (accurate sincosf: the angles reach
    // thousands of radians at the low frequencies) and shared by the key and every query head
    __shared__ float2 cs_s[kD / 2];
    if (threadIdx.x < kD / 2) {
        const float inv = powf(theta, -2.0f * float(threadIdx.x) / float(kD));
        float sn, cn;
        sincosf(float(pos) * inv, &sn, &cn);
        cs_s[threadIdx.x] = make_float2(cn, sn);
    }
    __syncthreads();
    auto rot = [&](float a, float bb, int d) {
        const float2 c = cs_s[d];
        return make_float2(a * c.x - bb * c.y, bb * c.x + a * c.y);
    };
    // the split holding `pos` appends the new (rotated) key and the value there
    if (sp == nsp - 1 && warp == 0) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            const int d = lane + 32 * h2;
            const float2 r = rot(__bfloat162float(kn[d]), __bfloat162float(kn[d + kD / 2]), d);
            kcb[int64_t(pos) * cstride + d] = __float2bfloat16_rn(r.x);
            kcb[int64_t(pos) * cstride + d + kD / 2] = __float2bfloat16_rn(r.y);
            vcb[int64_t(pos) * cstride + d] = vn[d];
            vcb[int64_t(pos) * cstride + d + kD / 2] = vn[d + kD / 2];
        }
    }
    // rotated, pre-scaled query of this warp's head
    const int qh = kvh * G + warp;
    const __nv_bfloat16* qp = qkv + row + int64_t(qh) * kD;
    const float scale = rsqrtf(float(kD));
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
        const int d = lane + 32 * h2;
        const float2 r = rot(__bfloat162float(qp[d]), __bfloat162float(qp[d + kD / 2]), d);
        qs[warp * kD + d] = r.x * scale;
        qs[warp * kD + d + kD / 2] = r.y * scale;
    }
    __threadfence_block();
    __syncthreads();  // the appended row is written before the staging copies below read it
    // stage K and V rows [t0, t0 + n): cp.async.cg (L2, coherent with the row appended above),
    // every copy in flight before one wait
    for (int i = threadIdx.x; i < n * 16; i += nthr) {
        const int t = i >> 4, c = i & 15;
        const uint32_t kd = static_cast<uint32_t>(__cvta_generic_to_shared(ks + swz(t, c)));
        const uint32_t vd = static_cast<uint32_t>(__cvta_generic_to_shared(vs + swz(t, c)));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(kd), "l"(kcb + int64_t(t0 + t) * cstride + c * 8)
                     : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(vd), "l"(vcb + int64_t(t0 + t) * cstride + c * 8)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const float* qw = qs + warp * kD;
    float* pw = ps + warp * chunk;
    // scores: lane owns positions t = lane + 32 j, reads its row 16 bytes (8 dims) at a time
    float cmax = -INFINITY;
    for (int t = lane; t < n; t += 32) {
        float sa[4] = {0.0f, 0.0f, 0.0f, 0.0f};  // four independent FMA chains
#pragma unroll 4
        for (int c = 0; c < 16; ++c) {
            const uint4 kv = ks[swz(t, c)];
            const float4 q0 = *reinterpret_cast<const float4*>(qw + 8 * c);
            const float4 q1 = *reinterpret_cast<const float4*>(qw + 8 * c + 4);
            const float2 k0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&kv.x));
            const float2 k1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&kv.y));
            const float2 k2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&kv.z));
            const float2 k3 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&kv.w));
            sa[0] = fmaf(q0.x, k0.x, sa[0]);
            sa[1] = fmaf(q0.y, k0.y, sa[1]);
            sa[2] = fmaf(q0.z, k1.x, sa[2]);
            sa[3] = fmaf(q0.w, k1.y, sa[3]);
            sa[0] = fmaf(q1.x, k2.x, sa[0]);
            sa[1] = fmaf(q1.y, k2.y, sa[1]);
            sa[2] = fmaf(q1.z, k3.x, sa[2]);
            sa[3] = fmaf(q1.w, k3.y, sa[3]);
        }
        const float sacc = (sa[0] + sa[1]) + (sa[2] + sa[3]);
        pw[t] = sacc;
        cmax = fmaxf(cmax, sacc);
    }
    cmax = warp_max(cmax);
    float csum = 0.0f;
    for (int t = lane; t < n; t += 32) {
        const float e = __expf(pw[t] - cmax);
        pw[t] = e;
        csum += e;
    }
    csum = warp_sum(csum);
    __syncwarp();
    // P * V: lane owns head dims 4*lane .. 4*lane+3 (8 bytes of 16-byte chunk lane/2); four
    // independent accumulator chains
    float acc[4][4] = {};
    const int vc8 = lane >> 1, vh = (lane & 1) * 2;  // chunk, 32-bit word within it
    auto vrow = [&](int t) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(vs + swz(t, vc8)) + vh;
        return make_float4(__bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w)).x,
                           __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w)).y,
                           __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w + 1)).x,
                           __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w + 1)).y);
    };
    int t = 0;
    for (; t + 4 <= n; t += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float pt = pw[t + u];
            const float4 v = vrow(t + u);
            acc[u][0] = fmaf(pt, v.x, acc[u][0]);
            acc[u][1] = fmaf(pt, v.y, acc[u][1]);
            acc[u][2] = fmaf(pt, v.z, acc[u][2]);
            acc[u][3] = fmaf(pt, v.w, acc[u][3]);
        }
    }
    for (; t < n; ++t) {
        const float pt = pw[t];
        const float4 v = vrow(t);
        acc[0][0] = fmaf(pt, v.x, acc[0][0]);
        acc[0][1] = fmaf(pt, v.y, acc[0][1]);
        acc[0][2] = fmaf(pt, v.z, acc[0][2]);
        acc[0][3] = fmaf(pt, v.w, acc[0][3]);
    }
    const bool wrote = attn_finish(
        cmax, csum,
        make_float4(acc[0][0] + acc[1][0] + acc[2][0] + acc[3][0], acc[0][1] + acc[1][1] + acc[2][1] + acc[3][1],
                    acc[0][2] + acc[1][2] + acc[2][2] + acc[3][2], acc[0][3] + acc[1][3] + acc[2][3] + acc[3][3]),
        reinterpret_cast<float*>(ks), part, arrivals, out, b, kvh, qh, hq, hkv, sp, nsp, cluster_merge);
    if (planes) attn_token_planes(wrote, out, b, hq, hkv, int(gridDim.y), tok_arrivals, planes, texp);
}

// Tensor-core variant (G <= 8 query heads per KV head): Q K^T and P V on mma.sync m16n8k16
// (bf16 x bf16 -> f32).  Queries and probabilities are split into bf16 hi + lo parts stacked in
// the 16 rows of the A tile (row h: hi part of head h, row 8 + h: lo part), so the products keep
// ~16 significant bits of q and p; keys and values are bf16 already.  Same staging, splits and
// merge as decode_attention_kernel (a split loaded at once); its CUDA-core score and P V loops
// become ~8 + 16 MMAs per 16 positions per warp.  Splits of more than 128 positions run
// decode_attention_mma_warp_kernel below.
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void decode_attention_mma_kernel(const __nv_bfloat16* __restrict__ qkv,
                                            __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc,
                                            float* __restrict__ part, int hq, int hkv, int lmax,
                                            int pos, float theta, __nv_bfloat16* __restrict__ out,
                                            int* __restrict__ arrivals, int cluster_merge, int chunk,
                                            int8_t* __restrict__ planes, int32_t* __restrict__ texp,
                                            int* __restrict__ tok_arrivals) {
    constexpr int kQS = kD + 8;                     // bf16 per A-tile row of the queries (padded)
    const int chunkp = (chunk + 15) / 16 * 16, kPS = chunkp + 8;
    extern __shared__ uint4 smq[];
    uint4* ks = smq;                                 // [chunkp][16] swizzled 16-byte chunks
    uint4* vs = ks + chunkp * 16;                    // [chunkp][16]
    __nv_bfloat16* qa = reinterpret_cast<__nv_bfloat16*>(vs + chunkp * 16);  // [16][kQS] q hi / lo
    __nv_bfloat16* pa = qa + 16 * kQS;               // [16][kPS] p hi / lo
    float* sc = reinterpret_cast<float*>(pa + 16 * kPS);  // [G][chunkp] scores
    float* fin = sc + 8 * chunkp;                    // [G][kPart] per-head results
    const int b = blockIdx.y, kvh = blockIdx.x, sp = blockIdx.z, nsp = gridDim.z, G = hq / hkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nthr = blockDim.x, W = nthr >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int64_t row = int64_t(b) * (hq + 2 * hkv) * kD;
    const __nv_bfloat16* kn = qkv + row + int64_t(hq) * kD + int64_t(kvh) * kD;
    const __nv_bfloat16* vn = kn + int64_t(hkv) * kD;
    const int64_t cstride = int64_t(hkv) * kD;
    __nv_bfloat16* kcb = kc + (int64_t(b) * lmax) * cstride + int64_t(kvh) * kD;
    __nv_bfloat16* vcb = vc + (int64_t(b) * lmax) * cstride + int64_t(kvh) * kD;
    const int t0 = sp * chunk, n = min(chunk, pos + 1 - t0);
    // the cached rows (every position but pos, written by earlier steps) first: their DRAM
    // latency overlaps the RoPE table, the query rotation and the append below
    for (int i = threadIdx.x; i < n * 16; i += nthr) {
        const int t = i >> 4, c = i & 15;
        if (t0 + t == pos) continue;
        const uint32_t kd = static_cast<uint32_t>(__cvta_generic_to_shared(ks + swz(t, c)));
        const uint32_t vd = static_cast<uint32_t>(__cvta_generic_to_shared(vs + swz(t, c)));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(kd), "l"(kcb + int64_t(t0 + t) * cstride + c * 8)
                     : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(vd), "l"(vcb + int64_t(t0 + t) * cstride + c * 8)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // only now the dependency on the previous kernel (the qkv linear): with programmatic
    // dependent launch the cached rows above stream in under its tail
    pdl_prologue();
    __shared__ float2 cs_s[kD / 2];
    if (threadIdx.x < kD / 2) {
        const float inv = powf(theta, -2.0f * float(threadIdx.x) / float(kD));
        float sn, cn;
        sincosf(float(pos) * inv, &sn, &cn);
        cs_s[threadIdx.x] = make_float2(cn, sn);
    }
    // zero the probability tile (rows of absent heads, positions past n) and the absent query rows
    for (int i = threadIdx.x; i < 16 * kPS / 2; i += nthr) reinterpret_cast<uint32_t*>(pa)[i] = 0u;
    for (int i = threadIdx.x; i < 16 * kQS / 2; i += nthr) {
        const int r = i / (kQS / 2);
        if ((r & 7) >= G) reinterpret_cast<uint32_t*>(qa)[i] = 0u;
    }
    for (int i = n * 16 + threadIdx.x; i < chunkp * 16; i += nthr)  // rows past n: finite zeros
        ks[swz(i >> 4, i & 15)] = vs[swz(i >> 4, i & 15)] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    auto rot = [&](float a, float bb, int d) {
        const float2 c = cs_s[d];
        return make_float2(a * c.x - bb * c.y, bb * c.x + a * c.y);
    };
    if (sp == nsp - 1 && warp == 0) {  // append the rotated key and the value at pos (cache + tile)
        const int tp = pos - t0;
        __nv_bfloat16* ksh = reinterpret_cast<__nv_bfloat16*>(ks);
        __nv_bfloat16* vsh = reinterpret_cast<__nv_bfloat16*>(vs);
        auto sidx = [&](int d) { return int(swz(tp, d >> 3)) * 8 + (d & 7); };
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            const int d = lane + 32 * h2;
            const float2 r = rot(__bfloat162float(kn[d]), __bfloat162float(kn[d + kD / 2]), d);
            const __nv_bfloat16 k0 = __float2bfloat16_rn(r.x), k1 = __float2bfloat16_rn(r.y);
            const __nv_bfloat16 v0 = vn[d], v1 = vn[d + kD / 2];
            kcb[int64_t(pos) * cstride + d] = k0;
            kcb[int64_t(pos) * cstride + d + kD / 2] = k1;
            vcb[int64_t(pos) * cstride + d] = v0;
            vcb[int64_t(pos) * cstride + d + kD / 2] = v1;
            ksh[sidx(d)] = k0, ksh[sidx(d + kD / 2)] = k1;
            vsh[sidx(d)] = v0, vsh[sidx(d + kD / 2)] = v1;
        }
    }
    {  // rotated, pre-scaled query of head `warp`, as bf16 hi (row warp) + lo (row 8 + warp)
        const __nv_bfloat16* qp = qkv + row + int64_t(kvh * G + warp) * kD;
        const float scale = rsqrtf(float(kD));
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            const int d = lane + 32 * h2;
            const float2 r = rot(__bfloat162float(qp[d]), __bfloat162float(qp[d + kD / 2]), d);
            const float q0 = r.x * scale, q1 = r.y * scale;
            const __nv_bfloat16 h0 = __float2bfloat16_rn(q0), h1 = __float2bfloat16_rn(q1);
            qa[warp * kQS + d] = h0;
            qa[warp * kQS + d + kD / 2] = h1;
            qa[(8 + warp) * kQS + d] = __float2bfloat16_rn(q0 - __bfloat162float(h0));
            qa[(8 + warp) * kQS + d + kD / 2] = __float2bfloat16_rn(q1 - __bfloat162float(h1));
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    // S = Q K^T: warp w takes the 8-position tiles w, w + W, ...
    {
        uint32_t af[8][4];
        const uint32_t* q32 = reinterpret_cast<const uint32_t*>(qa);
#pragma unroll
        for (int k16 = 0; k16 < 8; ++k16) {
            af[k16][0] = q32[(g * kQS + 16 * k16 + 2 * t4) >> 1];
            af[k16][1] = q32[((g + 8) * kQS + 16 * k16 + 2 * t4) >> 1];
            af[k16][2] = q32[(g * kQS + 16 * k16 + 8 + 2 * t4) >> 1];
            af[k16][3] = q32[((g + 8) * kQS + 16 * k16 + 8 + 2 * t4) >> 1];
        }
        for (int j = warp; j < chunkp / 8; j += W) {
            float c[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            const int r = 8 * j + g;  // this lane's key row (B column)
#pragma unroll
            for (int k16 = 0; k16 < 8; ++k16) {
                const uint32_t b0 = reinterpret_cast<const uint32_t*>(ks + swz(r, 2 * k16))[t4];
                const uint32_t b1 = reinterpret_cast<const uint32_t*>(ks + swz(r, 2 * k16 + 1))[t4];
                mma_bf16(c, af[k16][0], af[k16][1], af[k16][2], af[k16][3], b0, b1);
            }
            if (g < G) {  // rows g (hi) + g + 8 (lo) of head g, positions 8j + 2t4, + 1
                const int p0 = 8 * j + 2 * t4;
                sc[g * chunkp + p0] = c[0] + c[2];
                sc[g * chunkp + p0 + 1] = c[1] + c[3];
            }
        }
    }
    __syncthreads();
    // softmax of head `warp` over its n positions; probabilities as bf16 hi (row h) + lo (8 + h)
    float cmax = -INFINITY, csum = 0.0f;
    {
        const float* sw = sc + warp * chunkp;
        for (int t = lane; t < n; t += 32) cmax = fmaxf(cmax, sw[t]);
        cmax = warp_max(cmax);
        for (int t = lane; t < n; t += 32) {
            const float e = __expf(sw[t] - cmax);
            csum += e;
            const __nv_bfloat16 hi = __float2bfloat16_rn(e);
            pa[warp * kPS + t] = hi;
            pa[(8 + warp) * kPS + t] = __float2bfloat16_rn(e - __bfloat162float(hi));
        }
        csum = warp_sum(csum);
    }
    __syncthreads();
    // O = P V: warp w takes the 8-dim tiles w, w + W, ... over all 16-position k-steps
    {
        const uint32_t* p32 = reinterpret_cast<const uint32_t*>(pa);
        for (int nt = warp; nt < kD / 8; nt += W) {
            float c[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            for (int k16 = 0; k16 < chunkp / 16; ++k16) {
                const uint32_t a0 = p32[(g * kPS + 16 * k16 + 2 * t4) >> 1];
                const uint32_t a1 = p32[((g + 8) * kPS + 16 * k16 + 2 * t4) >> 1];
                const uint32_t a2 = p32[(g * kPS + 16 * k16 + 8 + 2 * t4) >> 1];
                const uint32_t a3 = p32[((g + 8) * kPS + 16 * k16 + 8 + 2 * t4) >> 1];
                // B = V[16 positions][8 dims] (row-major k x n): two 8x8 matrices, transposed load
                const uint32_t va = static_cast<uint32_t>(
                    __cvta_generic_to_shared(vs + swz(16 * k16 + (lane & 15), nt)));
                uint32_t b0, b1;
                asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                             : "=r"(b0), "=r"(b1) : "r"(va));
                mma_bf16(c, a0, a1, a2, a3, b0, b1);
            }
            if (g < G) {
                fin[g * kPart + 4 + 8 * nt + 2 * t4] = c[0] + c[2];
                fin[g * kPart + 4 + 8 * nt + 2 * t4 + 1] = c[1] + c[3];
            }
        }
    }
    __syncthreads();
    const float4 a4 = *reinterpret_cast<const float4*>(fin + warp * kPart + 4 + 4 * lane);
    const bool wrote = attn_finish(cmax, csum, a4, reinterpret_cast<float*>(ks), part, arrivals, out, b, kvh,
                                   kvh * G + warp, hq, hkv, sp, nsp, cluster_merge);
    if (planes) attn_token_planes(wrote, out, b, hq, hkv, int(gridDim.y), tok_arrivals, planes, texp);
}

// Long splits (> 128 positions): the same arithmetic, streamed.  A split's positions pass through
// kStages cp.async stages of kSub positions (the next loads while this one is scored), so a split
// can be any length and three CTAs share an SM (68 KiB of shared memory each).  Each warp owns 16
// positions of a stage: its scores stay in registers and become the P operand of its P V MMAs
// (the m16n8 C fragments of two 8-position tiles are the m16n8k16 A fragment; rows g / g + 8 =
// bf16 hi / lo of head g), it keeps its own online softmax, and the warps merge once at the end:
// one barrier per stage.  B16 ctx 4096: 144 us (one-shot kernel) -> 74 (a block-wide softmax
// per stage, 4 barriers) -> 55 us, 4.9 TB/s on the KV bytes (profiles/r2_attention_long_ctx.md).
template <int kSub, int kStages>
__global__ void __launch_bounds__(256) decode_attention_mma_warp_kernel(
    const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc,
    float* __restrict__ part, int hq, int hkv, int lmax, int pos, float theta, __nv_bfloat16* __restrict__ out,
    int* __restrict__ arrivals, int cluster_merge, int chunk, int8_t* __restrict__ planes,
    int32_t* __restrict__ texp, int* __restrict__ tok_arrivals) {
    constexpr int kQS = kD + 8;  // bf16 per A-tile row of the queries (padded)
    extern __shared__ uint4 smq[];
    uint4* ks = smq;                                                                 // [kStages][kSub][16] swizzled
    uint4* vs = ks + kStages * kSub * 16;                                            // [kStages][kSub][16]
    __nv_bfloat16* qa = reinterpret_cast<__nv_bfloat16*>(vs + kStages * kSub * 16);  // [16][kQS] q hi / lo
    float* wacc = reinterpret_cast<float*>(ks);  // after the last stage: [warp][head][kD] P V partials
    __shared__ float wm[8][8], wl[8][8];        // [warp][head]: running max, sum
    const int b = blockIdx.y, kvh = blockIdx.x, sp = blockIdx.z, nsp = gridDim.z, G = hq / hkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nthr = blockDim.x, W = nthr >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int64_t row = int64_t(b) * (hq + 2 * hkv) * kD;
    const __nv_bfloat16* kn = qkv + row + int64_t(hq) * kD + int64_t(kvh) * kD;
    const __nv_bfloat16* vn = kn + int64_t(hkv) * kD;
    const int64_t cstride = int64_t(hkv) * kD;
    __nv_bfloat16* kcb = kc + (int64_t(b) * lmax) * cstride + int64_t(kvh) * kD;
    __nv_bfloat16* vcb = vc + (int64_t(b) * lmax) * cstride + int64_t(kvh) * kD;
    const int t0 = sp * chunk, n = min(chunk, pos + 1 - t0), nsub = (n + kSub - 1) / kSub;
    auto issue = [&](int s) {
        // sub-chunk s -> stage s % kStages: rows past its end zeroed (finite for the MMAs), the
        // appended row (pos, not in the cache yet) skipped -- warp 0 writes it before that stage's use
        const int base = t0 + s * kSub, ns = min(kSub, n - s * kSub);
        uint4* kst = ks + (s % kStages) * kSub * 16;
        uint4* vst = vs + (s % kStages) * kSub * 16;
        for (int i = threadIdx.x; i < kSub * 16; i += nthr) {
            const int t = i >> 4, c = i & 15;
            if (t >= ns) {
                kst[swz(t, c)] = vst[swz(t, c)] = make_uint4(0, 0, 0, 0);
                continue;
            }
            if (base + t == pos) continue;
            const uint32_t kd = static_cast<uint32_t>(__cvta_generic_to_shared(kst + swz(t, c)));
            const uint32_t vd = static_cast<uint32_t>(__cvta_generic_to_shared(vst + swz(t, c)));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(kd),
                         "l"(kcb + int64_t(base + t) * cstride + c * 8)
                         : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(vd),
                         "l"(vcb + int64_t(base + t) * cstride + c * 8)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int i = 0; i < kStages - 1 && i < nsub; ++i) issue(i);
    pdl_prologue();
    __shared__ float2 cs_s[kD / 2];
    if (threadIdx.x < kD / 2) {
        const float inv = powf(theta, -2.0f * float(threadIdx.x) / float(kD));
        float sn, cn;
        sincosf(float(pos) * inv, &sn, &cn);
        cs_s[threadIdx.x] = make_float2(cn, sn);
    }
    for (int i = threadIdx.x; i < 16 * kQS / 2; i += nthr) {  // the absent heads' query rows
        const int r = i / (kQS / 2);
        if ((r & 7) >= G) reinterpret_cast<uint32_t*>(qa)[i] = 0u;
    }
    __syncthreads();
    auto rot = [&](float a, float bb, int d) {
        const float2 c = cs_s[d];
        return make_float2(a * c.x - bb * c.y, bb * c.x + a * c.y);
    };
    const bool appender = sp == nsp - 1 && warp == 0;
    __nv_bfloat16 ak[4], av[4];
    if (appender) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            const int d = lane + 32 * h2;
            const float2 r = rot(__bfloat162float(kn[d]), __bfloat162float(kn[d + kD / 2]), d);
            ak[h2] = __float2bfloat16_rn(r.x), ak[2 + h2] = __float2bfloat16_rn(r.y);
            av[h2] = vn[d], av[2 + h2] = vn[d + kD / 2];
            kcb[int64_t(pos) * cstride + d] = ak[h2];
            kcb[int64_t(pos) * cstride + d + kD / 2] = ak[2 + h2];
            vcb[int64_t(pos) * cstride + d] = av[h2];
            vcb[int64_t(pos) * cstride + d + kD / 2] = av[2 + h2];
        }
    }
    {
        const __nv_bfloat16* qp = qkv + row + int64_t(kvh * G + warp) * kD;
        const float scale = rsqrtf(float(kD));
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
            const int d = lane + 32 * h2;
            const float2 r = rot(__bfloat162float(qp[d]), __bfloat162float(qp[d + kD / 2]), d);
            const float q0 = r.x * scale, q1 = r.y * scale;
            const __nv_bfloat16 h0 = __float2bfloat16_rn(q0), h1 = __float2bfloat16_rn(q1);
            qa[warp * kQS + d] = h0;
            qa[warp * kQS + d + kD / 2] = h1;
            qa[(8 + warp) * kQS + d] = __float2bfloat16_rn(q0 - __bfloat162float(h0));
            qa[(8 + warp) * kQS + d + kD / 2] = __float2bfloat16_rn(q1 - __bfloat162float(h1));
        }
    }
    __syncthreads();
    uint32_t af[8][4];
    {
        const uint32_t* q32 = reinterpret_cast<const uint32_t*>(qa);
#pragma unroll
        for (int k16 = 0; k16 < 8; ++k16) {
            af[k16][0] = q32[(g * kQS + 16 * k16 + 2 * t4) >> 1];
            af[k16][1] = q32[((g + 8) * kQS + 16 * k16 + 2 * t4) >> 1];
            af[k16][2] = q32[(g * kQS + 16 * k16 + 8 + 2 * t4) >> 1];
            af[k16][3] = q32[((g + 8) * kQS + 16 * k16 + 8 + 2 * t4) >> 1];
        }
    }
    float m_run = -INFINITY, l_part = 0.0f;  // head g's running max (quad-uniform), this lane's sum
    float acc[kD / 8][4];
#pragma unroll
    for (int i = 0; i < kD / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0f;
    for (int s = 0; s < nsub; ++s) {
        // committed so far: sub-chunks up to s + kStages - 2 (this iteration's issue comes after
        // the barrier below); those after s may stay in flight
        const int pend = min(kStages - 2, nsub - 1 - s);
        if (pend >= 2)
            asm volatile("cp.async.wait_group 2;" ::: "memory");
        else if (pend == 1)
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        else
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        const int ns = min(kSub, n - s * kSub);
        uint4* kst = ks + (s % kStages) * kSub * 16;
        uint4* vst = vs + (s % kStages) * kSub * 16;
        if (appender && s == nsub - 1) {
            const int tp = pos - t0 - s * kSub;
            __nv_bfloat16* ksh = reinterpret_cast<__nv_bfloat16*>(kst);
            __nv_bfloat16* vsh = reinterpret_cast<__nv_bfloat16*>(vst);
            auto sidx = [&](int d) { return int(swz(tp, d >> 3)) * 8 + (d & 7); };
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                const int d = lane + 32 * h2;
                ksh[sidx(d)] = ak[h2], ksh[sidx(d + kD / 2)] = ak[2 + h2];
                vsh[sidx(d)] = av[h2], vsh[sidx(d + kD / 2)] = av[2 + h2];
            }
        }
        // stage s is visible to every warp, and every warp is done with stage s - 1: its buffer
        // takes the sub-chunk kStages - 1 ahead
        __syncthreads();
        if (s + kStages - 1 < nsub) issue(s + kStages - 1);
        for (int sl = warp; sl < kSub / 16; sl += W) {
            const int p0 = 16 * sl;
            if (p0 >= ns) break;
            float c0[4] = {0.0f, 0.0f, 0.0f, 0.0f}, c1[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
            for (int k16 = 0; k16 < 8; ++k16) {
                const uint32_t* k0 = reinterpret_cast<const uint32_t*>(kst + swz(p0 + g, 2 * k16));
                const uint32_t* k1 = reinterpret_cast<const uint32_t*>(kst + swz(p0 + g, 2 * k16 + 1));
                const uint32_t* k2 = reinterpret_cast<const uint32_t*>(kst + swz(p0 + 8 + g, 2 * k16));
                const uint32_t* k3 = reinterpret_cast<const uint32_t*>(kst + swz(p0 + 8 + g, 2 * k16 + 1));
                mma_bf16(c0, af[k16][0], af[k16][1], af[k16][2], af[k16][3], k0[t4], k1[t4]);
                mma_bf16(c1, af[k16][0], af[k16][1], af[k16][2], af[k16][3], k2[t4], k3[t4]);
            }
            // head g's scores at positions p0 + 2 t4, +1, p0 + 8 + 2 t4, +1 (rows g + g + 8)
            float sv[4] = {c0[0] + c0[2], c0[1] + c0[3], c1[0] + c1[2], c1[1] + c1[3]};
            const int q0 = p0 + 2 * t4;
            if (q0 >= ns) sv[0] = -INFINITY;
            if (q0 + 1 >= ns) sv[1] = -INFINITY;
            if (q0 + 8 >= ns) sv[2] = -INFINITY;
            if (q0 + 9 >= ns) sv[3] = -INFINITY;
            float mloc = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
            mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 1));
            mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, 2));
            const float mnew = fmaxf(m_run, mloc), mref = mnew == -INFINITY ? 0.0f : mnew;
            const float al = __expf(m_run - mref);
            m_run = mnew;
            float pr[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) pr[j] = __expf(sv[j] - mref);
            l_part = fmaf(l_part, al, (pr[0] + pr[1]) + (pr[2] + pr[3]));
            const __nv_bfloat162 h01 = __floats2bfloat162_rn(pr[0], pr[1]), h23 = __floats2bfloat162_rn(pr[2], pr[3]);
            const __nv_bfloat162 l01 = __floats2bfloat162_rn(pr[0] - __low2float(h01), pr[1] - __high2float(h01));
            const __nv_bfloat162 l23 = __floats2bfloat162_rn(pr[2] - __low2float(h23), pr[3] - __high2float(h23));
            const uint32_t a0 = *reinterpret_cast<const uint32_t*>(&h01), a1 = *reinterpret_cast<const uint32_t*>(&l01);
            const uint32_t a2 = *reinterpret_cast<const uint32_t*>(&h23), a3 = *reinterpret_cast<const uint32_t*>(&l23);
            const uint32_t vrow = static_cast<uint32_t>(__cvta_generic_to_shared(vst)) + uint32_t(p0 + (lane & 15)) * 256u;
            const int vsw = (p0 + (lane & 15)) & 15;
#pragma unroll
            for (int nt = 0; nt < kD / 8; ++nt) {
                float* c = acc[nt];
                c[0] *= al, c[1] *= al, c[2] *= al, c[3] *= al;
                uint32_t b0, b1;
                asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                             : "=r"(b0), "=r"(b1)
                             : "r"(vrow + uint32_t((nt ^ vsw) * 16)));
                mma_bf16(acc[nt], a0, a1, a2, a3, b0, b1);
            }
        }
    }
    __syncthreads();  // every warp is done with the stages: the partials reuse them
    float l = l_part + __shfl_xor_sync(0xffffffffu, l_part, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    if (t4 == 0) wm[warp][g] = m_run, wl[warp][g] = l;
    if (g < G) {
        float* wa = wacc + (warp * 8 + g) * kD;
#pragma unroll
        for (int nt = 0; nt < kD / 8; ++nt)
            *reinterpret_cast<float2*>(wa + 8 * nt + 2 * t4) = make_float2(acc[nt][0] + acc[nt][2], acc[nt][1] + acc[nt][3]);
    }
    __syncthreads();
    // warp h = head h: merge the warps' partials of this split
    float M = -INFINITY;
    for (int w = 0; w < W; ++w) M = fmaxf(M, wm[w][warp]);
    float L = 0.0f;
    float4 a4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    for (int w = 0; w < W; ++w) {
        const float mw = wm[w][warp];
        const float wt = mw == -INFINITY ? 0.0f : __expf(mw - M);
        L = fmaf(wt, wl[w][warp], L);
        const float4 x = *reinterpret_cast<const float4*>(wacc + (w * 8 + warp) * kD + 4 * lane);
        a4.x = fmaf(wt, x.x, a4.x), a4.y = fmaf(wt, x.y, a4.y), a4.z = fmaf(wt, x.z, a4.z), a4.w = fmaf(wt, x.w, a4.w);
    }
    // (attn_finish's cluster scratch reuses these bytes after its first barrier)
    const bool wrote = attn_finish(M, L, a4, reinterpret_cast<float*>(ks), part, arrivals, out, b, kvh,
                                   kvh * G + warp, hq, hkv, sp, nsp, cluster_merge);
    if (planes) attn_token_planes(wrote, out, b, hq, hkv, int(gridDim.y), tok_arrivals, planes, texp);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    // RTNQ_DECODE_PDL=1 launches these as PDL secondaries; by default they are stream-ordered
    // (griddepcontrol is then a no-op).
    static const int pdl = [] {
        const char* e = std::getenv("RTNQ_DECODE_PDL");
        return e ? std::atoi(e) : 0;
    }();
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

}  // namespace

#define RTNQ_ROWS_VPT(KERN, CL, vpt, m, st, ...)                                                    \
    ((vpt) <= 1    ? launch_rows(KERN<1, CL>, m, CL, st, __VA_ARGS__)                                 \
     : (vpt) <= 2  ? launch_rows(KERN<2, CL>, m, CL, st, __VA_ARGS__)                                 \
     : (vpt) <= 4  ? launch_rows(KERN<4, CL>, m, CL, st, __VA_ARGS__)                                 \
     : (vpt) <= 8  ? launch_rows(KERN<8, CL>, m, CL, st, __VA_ARGS__)                                 \
     : (vpt) <= 16 ? launch_rows(KERN<16, CL>, m, CL, st, __VA_ARGS__)                                \
                   : launch_rows(KERN<32, CL>, m, CL, st, __VA_ARGS__))
#define RTNQ_ROWS_DISPATCH(KERN, m, n8, st, ...)                                                    \
    [&]() {                                                                                         \
        const int cl_ = row_cluster(m, n8);                                                         \
        const int64_t vpt_ = ((n8) + int64_t(cl_) * kRowThreads - 1) / (int64_t(cl_) * kRowThreads); \
        return cl_ == 8   ? RTNQ_ROWS_VPT(KERN, 8, vpt_, m, st, __VA_ARGS__)                        \
               : cl_ == 4 ? RTNQ_ROWS_VPT(KERN, 4, vpt_, m, st, __VA_ARGS__)                        \
               : cl_ == 2 ? RTNQ_ROWS_VPT(KERN, 2, vpt_, m, st, __VA_ARGS__)                        \
                          : RTNQ_ROWS_VPT(KERN, 1, vpt_, m, st, __VA_ARGS__);                       \
    }()

cudaError_t launch_add_rmsnorm(void* x, const void* delta, const void* w, void* out, int64_t m,
                               int64_t h, float eps, cudaStream_t st, int8_t* planes, int32_t* texp,
                               PeerIn pin) {
    if (h % 8) return cudaErrorInvalidValue;
    if (h / 8 <= 32 * kRowThreads)  // the row in registers (of a cluster of CTAs)
        return RTNQ_ROWS_DISPATCH(add_rmsnorm_rows_kernel, m, h / 8, st, static_cast<__nv_bfloat16*>(x),
                                  static_cast<const __nv_bfloat16*>(delta), static_cast<const __nv_bfloat16*>(w),
                                  static_cast<__nv_bfloat16*>(out), int(h), eps, planes, texp, pin);
    if (pin.buf) return cudaErrorInvalidValue;
    return launch_pdl(add_rmsnorm_kernel, dim3(unsigned(m)), dim3(256), 8 * sizeof(float), st,
                      static_cast<__nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(delta),
                      static_cast<const __nv_bfloat16*>(w), static_cast<__nv_bfloat16*>(out), int(h), eps,
                      planes, texp);
}

cudaError_t launch_silu_mul(const void* gu, void* act, int64_t m, int64_t f, cudaStream_t st, int8_t* planes,
                            int32_t* texp) {
    if (f % 8) return cudaErrorInvalidValue;
    if (planes && f / 8 <= 32 * kRowThreads)  // the row in registers (of a cluster of CTAs)
        return RTNQ_ROWS_DISPATCH(silu_mul_rows_kernel, m, f / 8, st, static_cast<const __nv_bfloat16*>(gu),
                                  static_cast<__nv_bfloat16*>(act), int(f), planes, texp);
    if (planes)
        return launch_pdl(silu_mul_planes_kernel, dim3(unsigned(m)), dim3(256), 0, st,
                          static_cast<const __nv_bfloat16*>(gu), static_cast<__nv_bfloat16*>(act), int(f), planes,
                          texp);
    const int64_t n8 = m * f / 8;
    const unsigned blocks = unsigned(n8 / 256 + 1 < 1184 ? n8 / 256 + 1 : 1184);
    return launch_pdl(silu_mul_kernel, dim3(blocks), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(gu),
                      static_cast<__nv_bfloat16*>(act), m, int(f));
}

// The tensor-core kernels (up to 8 query heads per KV head) take any chunk (the streaming kernel
// beyond kMaxChunk positions); the CUDA-core kernel stages a whole chunk of <= kMaxChunk.
static bool attention_uses_mma(int64_t hq, int64_t hkv) {
    static const bool no_mma = std::getenv("RTNQ_ATTN_NO_MMA") != nullptr;
    return hq / hkv <= 8 && !no_mma;
}

// splits of the context: ~`waves` waves of CTAs over the SMs, chunks of >= 32 positions (and at
// most kMaxChunk for the CUDA-core kernel)
constexpr int kStreamExtraSplits = 8;
static void attention_split(int64_t batch, int64_t hkv, int64_t pos, bool mma, int* nsp_out, int* chunk_out,
                            bool* stream_out = nullptr) {
    static const int64_t waves = [] {
        const char* e = std::getenv("RTNQ_ATTN_WAVES");
        return e ? int64_t(std::atoi(e)) : int64_t(2);
    }();
    static const int64_t max_chunk_env = [] {
        const char* e = std::getenv("RTNQ_ATTN_MAX_CHUNK");
        return e ? int64_t(std::atoi(e)) : int64_t(0);
    }();
    int64_t max_chunk = mma ? int64_t(1) << 30 : int64_t(kMaxChunk);
    if (max_chunk_env > 0 && max_chunk_env < max_chunk) max_chunk = max_chunk_env < 32 ? 32 : max_chunk_env;
    const int64_t ctx = pos + 1, pairs = batch * hkv;
    int64_t nsp = (waves * 148 + pairs - 1) / pairs;
    nsp = nsp < 1 ? 1 : nsp;
    const int64_t max_sp = (ctx + 31) / 32, min_sp = (ctx + max_chunk - 1) / max_chunk;
    nsp = nsp > max_sp ? max_sp : nsp;
    nsp = nsp < min_sp ? min_sp : nsp;
    int64_t chunk = (ctx + nsp - 1) / nsp;
    chunk = (chunk + 7) / 8 * 8;
    if (stream_out) *stream_out = false;
    static const int64_t stream_min = [] {
        const char* e = std::getenv("RTNQ_ATTN_STREAM_MIN");
        return e ? int64_t(std::atoi(e)) : int64_t(128);
    }();
    if (mma && chunk > stream_min) {
        // the streaming kernel (3 CTAs per SM, long-running CTAs): the smallest split count from
        // here whose grid fills its last wave of 3 x 148 CTAs to >= 1/1.2 -- a grid just past a
        // whole wave runs a long tail (B32 ctx 4096: 2 splits, 1.15 waves, 196 us; 3 splits, 145 us)
        const int64_t n0 = nsp;
        int64_t best = n0;
        double best_eff = 1e30;
        for (int64_t n = n0; n <= n0 + kStreamExtraSplits && n <= max_sp; ++n) {
            const double w = double(pairs * n) / (3.0 * 148.0);
            const double eff = ceil(w) / w;
            if (eff < best_eff) best = n, best_eff = eff;
            if (eff <= 1.2) {
                best = n;
                break;
            }
        }
        chunk = (ctx + best - 1) / best;
        chunk = (chunk + 7) / 8 * 8;
        if (stream_out) *stream_out = true;
    }
    *nsp_out = int((ctx + chunk - 1) / chunk);
    *chunk_out = int(chunk);
}

// Workspace: [self-resetting counters: a fixed 64 KiB][partials].  The counters (split merges
// [batch][hkv], then the o-planes tokens [batch]) sit at the same offsets whatever the call's
// batch, so calls of different batch sizes can share one workspace: a batch-dependent offset of
// the partials once put one call's partials over another call's counters.
constexpr size_t kAttnCounterBytes = 64 * 1024;
size_t decode_attention_workspace_bytes(int64_t batch, int64_t hq, int64_t hkv, int64_t max_len) {
    int nsp, chunk;
    // the largest context of this cache; the streaming kernel's split count may exceed the
    // default rule's by up to kStreamExtraSplits, whatever the context
    attention_split(batch, hkv, max_len - 1, hkv > 0 && attention_uses_mma(hq, hkv), &nsp, &chunk);
    nsp += kStreamExtraSplits;
    return kAttnCounterBytes + size_t(batch) * size_t(hq) * size_t(nsp) * kPart * sizeof(float) + 256;
}

cudaError_t launch_decode_attention(const void* qkv, void* kcache, void* vcache, void* out,
                                    int64_t batch, int64_t hq, int64_t hkv, int64_t head_dim,
                                    int64_t lmax, int64_t pos, float theta, cudaStream_t st,
                                    void* ws, size_t ws_bytes, int8_t* planes, int32_t* texp) {
    if (head_dim != kD || hkv <= 0 || hq % hkv || hq / hkv > 32 || pos < 0 || pos >= lmax ||
        size_t(batch * hkv + batch) * sizeof(int) > kAttnCounterBytes)
        return cudaErrorInvalidValue;
    const int G = int(hq / hkv);
    int nsp, chunk;
    const bool mma = attention_uses_mma(hq, hkv);
    bool stream = false;
    attention_split(batch, hkv, pos, mma, &nsp, &chunk, &stream);
    auto mma_smem = [](int ch) {
        const int chp = (ch + 15) / 16 * 16;
        return size_t(2 * chp * 16) * 16 + size_t(16) * (kD + 8) * 2 + size_t(16) * (chp + 8) * 2 +
               size_t(8) * chp * 4 + size_t(8) * kPart * 4;
    };
    constexpr int kStreamSub = 64, kStreamStages = 2;
    const size_t stream_smem = size_t(2 * kStreamStages * kStreamSub * 16) * 16 + size_t(16) * (kD + 8) * 2;
    auto stream_kern = decode_attention_mma_warp_kernel<kStreamSub, kStreamStages>;
    const size_t smem = stream ? stream_smem
                        : mma  ? mma_smem(chunk)
                               : size_t(2 * chunk * 16) * 16 + size_t(G) * (kD + chunk) * 4;
    static unsigned long long configured = 0;  // per device
    if (!(configured & current_device_bit())) {
        cudaFuncSetAttribute(decode_attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(2 * kMaxChunk * 16 * 16 + 32 * (kD + kMaxChunk) * 4));
        cudaFuncSetAttribute(decode_attention_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(mma_smem(kMaxChunk)));
        cudaFuncSetAttribute(stream_kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(stream_smem));
        configured |= current_device_bit();
    }
    // split-merge scratch: the counters (zero-initialized, self-resetting) and the partials, from
    // the caller's workspace; without one, a per-device buffer (single stream only)
    int* arrivals;
    float* part;
    const size_t need_part = size_t(batch) * size_t(hq) * size_t(nsp) * kPart * sizeof(float);
    if (ws) {
        if (ws_bytes < decode_attention_workspace_bytes(batch, hq, hkv, pos + 1)) return cudaErrorInvalidValue;
        arrivals = static_cast<int*>(ws);
        part = reinterpret_cast<float*>(static_cast<char*>(ws) + kAttnCounterBytes);
    } else {
        static std::mutex mu;
        std::lock_guard<std::mutex> lock(mu);
        static float* part_dev[64] = {};
        static size_t part_bytes_dev[64] = {};
        static int* arrivals_dev[64] = {};
        static size_t arrivals_n_dev[64] = {};
        float*& pd = part_dev[current_device_index()];
        size_t& pb = part_bytes_dev[current_device_index()];
        int*& ad = arrivals_dev[current_device_index()];
        size_t& an = arrivals_n_dev[current_device_index()];
        if (size_t(batch * hkv + batch) > an) {  // zeroed on this stream; an older buffer stays valid for graphs
            const size_t want = size_t(batch * hkv + batch) * 2;
            int* fresh = nullptr;
            if (cudaError_t e = cudaMalloc(&fresh, want * sizeof(int))) return e;
            if (cudaError_t e = cudaMemsetAsync(fresh, 0, want * sizeof(int), st)) return e;
            ad = fresh, an = want;
        }
        if (need_part > pb) {
            float* fresh = nullptr;
            if (cudaError_t e = cudaMalloc(&fresh, need_part * 2)) return e;
            pd = fresh, pb = need_part * 2;
        }
        arrivals = ad, part = pd;
    }
    // 2..8 splits: one thread-block cluster per (token, KV head), merged over DSMEM; more splits
    // merge through global memory (the last CTA to arrive)
    static const int max_cluster = [] {
        const char* e = std::getenv("RTNQ_ATTN_MAX_CLUSTER");
        return e ? std::atoi(e) : 8;
    }();
    const int cluster = nsp >= 2 && nsp <= max_cluster && !std::getenv("RTNQ_ATTN_NO_CLUSTER") ? 1 : 0;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(hkv), unsigned(batch), unsigned(nsp));
    cfg.blockDim = dim3(unsigned(32 * G));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    // programmatic dependent launch for the tensor-core kernel: its cached-row loads run before
    // its griddepcontrol.wait (RTNQ_ATTN_PDL=0: stream-ordered)
    static const bool attn_pdl = [] {
        const char* e = std::getenv("RTNQ_ATTN_PDL");
        return !(e && std::atoi(e) == 0);
    }();
    cudaLaunchAttribute attrs[2];
    int na = 0;
    if (cluster) {
        attrs[na].id = cudaLaunchAttributeClusterDimension;
        attrs[na].val.clusterDim.x = 1;
        attrs[na].val.clusterDim.y = 1;
        attrs[na].val.clusterDim.z = unsigned(nsp);
        ++na;
    }
    if (mma && attn_pdl) {
        attrs[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg,
                              stream ? stream_kern
                              : mma  ? decode_attention_mma_kernel
                                     : decode_attention_kernel,
                              static_cast<const __nv_bfloat16*>(qkv),
                              static_cast<__nv_bfloat16*>(kcache), static_cast<__nv_bfloat16*>(vcache), part,
                              int(hq), int(hkv), int(lmax), int(pos), theta, static_cast<__nv_bfloat16*>(out),
                              arrivals, cluster, chunk, planes, texp, arrivals + batch * hkv);
}

}  // namespace rtnq_b200
