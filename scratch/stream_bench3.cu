// Microbenchmark: HBM streaming through smem with cp.async.bulk + mbarrier vs plain LDG.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mb_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(d)), "l"(s), "r"(n), "r"(su32(b)) : "memory");
}

// Each CTA streams its contiguous share of `bytes` in chunks of STAGE bytes split into NCOPY copies.
template <int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32) tma_stream(const uint8_t* src, size_t bytes, int stage, int stages, int ncopy, unsigned* sink, size_t stride = 0, int extra = 0) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = (uint64_t*)(sm + (size_t)stage * stages);
    uint64_t* empty = full + stages;
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    size_t per = bytes / gridDim.x / stage * stage;
    const uint8_t* base = src + per * blockIdx.x;
    int n = (int)(per / stage);
    if (threadIdx.x == 0) { for (int s = 0; s < stages; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], NCW); } asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    if (warp == NCW) {
        int s = 0; uint32_t ph = 0;
        for (int i = 0; i < n; ++i) {
            if (i >= stages) mb_wait(&empty[s], ph ^ 1);
            if (lane == 0) mb_tx(&full[s], stage + (extra ? 512 : 0));
            __syncwarp();
            int cb = stage / ncopy;
            const uint8_t* chunk = stride ? src + ((size_t)i * gridDim.x + blockIdx.x) % (bytes / stage) * stage : base + (size_t)i * stage;
            if (stride) chunk = src + (((size_t)blockIdx.x * n + i) * stride) % (bytes - stage) / 512 * 512;
            if (extra && lane == 0) bulk(sm + (size_t)s * stage, chunk, 512, &full[s]);
            for (int c = lane; c < ncopy; c += 32) bulk(sm + (size_t)s * stage + c * cb, chunk + c * cb, cb, &full[s]);
            if (++s == stages) { s = 0; ph ^= 1; }
        }
        return;
    }
    unsigned acc = 0; int s = 0; uint32_t ph = 0;
    for (int i = 0; i < n; ++i) {
        mb_wait(&full[s], ph);
        const uint4* p = (const uint4*)(sm + (size_t)s * stage);
        for (int j = warp * 32 + lane; j < stage / 16; j += NCW * 32) { uint4 v = p[j]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
        __syncwarp();
        if (lane == 0) mb_arrive(&empty[s]);
        if (++s == stages) { s = 0; ph ^= 1; }
    }
    if (acc == 0x12345678) sink[0] = acc;
}

template <int UNROLL>
__global__ void ldg_stream(const uint4* src, size_t n16, unsigned* sink) {
    unsigned acc = 0;
    size_t stride = (size_t)gridDim.x * blockDim.x * UNROLL;
    for (size_t i = (size_t)blockIdx.x * blockDim.x * UNROLL + threadIdx.x; i < n16; i += stride) {
        uint4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) { size_t k = i + (size_t)u * blockDim.x; v[u] = k < n16 ? __ldcs(src + k) : make_uint4(0,0,0,0); }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    if (acc == 0x12345678) sink[0] = acc;
}

int main() {
    const size_t cap = (size_t)1 << 30;
    uint8_t* buf; unsigned* sink;
    cudaMalloc(&buf, cap); cudaMalloc(&sink, 4); cudaMemset(buf, 1, cap);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    struct V { int stage, stages, ncopy, ctas; };
    V vs[] = {{16384, 8, 1, 148}, {16384, 8, 2, 148}, {16384, 8, 4, 148}, {16384, 8, 8, 148},
              {32768, 6, 1, 148}, {32768, 6, 2, 148}, {32768, 6, 4, 148}, {32768, 6, 8, 148},
              {65536, 3, 1, 148}, {65536, 3, 4, 148}, {65536, 3, 16, 148},
              {16384, 6, 1, 296}, {16384, 6, 4, 296}, {32768, 3, 4, 296},
              {16384, 8, 4, 96}, {32768, 6, 4, 96}};
    for (size_t bytes : {(size_t)25165824, (size_t)117440512})
    for (V v : vs) {
        size_t smem = (size_t)v.stage * v.stages + 16 * v.stages;
        cudaFuncSetAttribute(tma_stream<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int nrot = int(cap / bytes);
        for (int r = 0; r < nrot; ++r) tma_stream<4><<<v.ctas, 160, smem>>>(buf + r * bytes, bytes, v.stage, v.stages, v.ncopy, sink);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 40; ++r) tma_stream<4><<<v.ctas, 160, smem>>>(buf + (r % nrot) * bytes, bytes, v.stage, v.stages, v.ncopy, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("bytes=%9zu ctas=%d stage=%6d stages=%2d ncopy=%2d %7.2f us/launch %8.1f GB/s %s\n", bytes, v.ctas, v.stage, v.stages, v.ncopy, ms * 1e3 / 40,
               bytes * 40 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
