// tmem_bw.cu -- TMEM read-port microbenchmark (round 2, verdict item 4: pin the W4 limiter).
//
//   A: tcgen05.ld.32x32b.x32 throughput with W warps (W/4 per TMEM lane quadrant), no MMA
//   B: tcgen05.mma kind::i8 M128 x N x K32 issue rate, A from TMEM (TS) or smem (SS), no loads
//   C: B and A at the same time (the W4 kernel's MMA + epilogue)
// One CTA per SM (grid = #SMs, every SM busy), clock64 per role, bytes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu && ./tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
                     su32(b)), "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void commit1(uint64_t* b) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ bool elect_one_lane() {
    uint32_t p;
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\nselp.u32 %0, 1, 0, e;\n}\n" : "=r"(p));
    return p != 0;
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bd, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                 "r"(a), "l"(bd), "r"(id), "r"(acc)
                 : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(ad), "l"(bd), "r"(id), "r"(acc)
                 : "memory");
}
#define LD32(taddr, r)                                                                                              \
    asm volatile(                                                                                                   \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19," \
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                                  \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),  \
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),       \
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),      \
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                   \
        : "r"(taddr))

struct Cfg {
    int ld_warps;   // warps doing tcgen05.ld (0 = none); warp w reads lane quadrant w % 4
    int mma;        // 0 none, 1 TS (A from TMEM), 2 SS (A from smem)
    int n;          // MMA N
    int iters;
    int nd;         // independent accumulators, round-robin (consecutive MMAs hit different D)
    int m = 128;    // MMA M (64 or 128)
    int issuers = 1;  // warps issuing MMAs concurrently (disjoint accumulators / A slots)
    int variant = 0;  // 0: lane 0 issues (compiler elect loop per MMA); 1: warp-uniform, 4 MMAs per asm
    int st_warps = 0; // warps 8.. doing tcgen05.st.32x32b.x32 + wait::st loops (the W4 expansion)
    int commits = 0;  // variant 1: tcgen05.commit's per 8 MMAs (to distinct mbarriers)
};
// 4 k-steps into one accumulator, one elect for the block: A from TMEM at a, a+8, a+16, a+24,
// B descriptors bd, bd+2, bd+4, bd+6 (32 B steps); the first overwrites D
__device__ __forceinline__ void mma4_ts(uint32_t d, uint32_t a, uint64_t bd, uint32_t id) {
    asm volatile(
        "{\n.reg .pred e, p0, p1;\n.reg .b32 a1, a2, a3;\n.reg .b64 b1, b2, b3;\n"
        "setp.ne.b32 p0, 0, 0;\nsetp.eq.b32 p1, 0, 0;\n"
        "add.u32 a1, %1, 8;\nadd.u32 a2, %1, 16;\nadd.u32 a3, %1, 24;\n"
        "add.u64 b1, %2, 2;\nadd.u64 b2, %2, 4;\nadd.u64 b3, %2, 6;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p0;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %3, p1;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a2], b2, %3, p1;\n"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a3], b3, %3, p1;\n}\n" ::"r"(d),
        "r"(a), "l"(bd), "r"(id)
        : "memory");
}

__global__ void __launch_bounds__(384, 1) bench(Cfg c, long long* out, unsigned* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bars[4];
    __shared__ uint64_t cbars[4];
    __shared__ uint32_t ts;
    __shared__ volatile int go;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
    for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) base[i] = (uint8_t)(i * 2654435761u >> 24);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1), mbar_init(&cbars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
        go = 0;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&ts)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = ts;
    long long t0 = clock64();
    if (warp < c.issuers && c.mma) {
        // D in columns [0, 256) (two accumulators), A (TS) in columns [384, 512)
        const uint32_t b0 = su32(base + 32 * 1024);
        const uint64_t sw = (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
        const uint32_t id = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(c.n >> 3) << 17) | (uint32_t(c.m >> 4) << 24);
        if (c.variant == 1) {
            const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
            const uint64_t bd0 = sw | ((b0 >> 4) & 0x3FFF);
            for (int i = 0; i < c.iters; i += 16) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    mma4_ts(tm + uint32_t(warp) * 32 + uint32_t(u & 1) * 16, tm + 384 + uint32_t(u) * 32, bd0, id);
                    if (u & 1)
                        for (int cc = 0; cc < c.commits; ++cc)
                            asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(&cbars[cc])) : "memory");
                }
            }
            if (elect_one_lane()) commit1(&bars[warp]);
        } else if (lane == 0) {
            // 16 MMAs per iteration, addresses from compile-time offsets (no per-MMA index math):
            // nd accumulators round-robin, each gets 4 k-steps
            const uint32_t abase = tmem + 384 + uint32_t(warp) * 0, bb = ((b0 >> 4) & 0x3FFF);
            const uint32_t tw = tmem + uint32_t(warp) * 32;  // this issuer's accumulators (N <= 16)
            const uint64_t bd0 = sw | bb;
            const uint64_t ad0 = sw | ((su32(base) >> 4) & 0x3FFF);
            for (int i = 0; i < c.iters; i += 16) {
                if (c.nd == 1) {
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        const int ks = u & 3;
                        const uint32_t d = c.issuers > 1 ? tw + uint32_t((u >> 2) & 1) * 16 : tmem + uint32_t((u >> 2) & 1) * 128;
                        if (c.mma == 1) mma_ts(d, abase + (u >> 2) * 32 + ks * 8, bd0 + 2 * ks, id, ks);
                        else mma_ss(d, ad0 + ((u >> 2) & 1) * 1024 + 2 * ks, bd0 + 2 * ks, id, ks);
                    }
                } else if (c.nd == 2) {
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        const int ks = (u >> 1) & 3;
                        const uint32_t d = tmem + uint32_t(u & 1) * 128;
                        if (c.mma == 1) mma_ts(d, abase + (u & 1) * 32 + ks * 8, bd0 + 2 * ks, id, ks);
                        else mma_ss(d, ad0 + (u & 1) * 1024 + 2 * ks, bd0 + 2 * ks, id, ks);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        const int ks = (u >> 2) & 3;
                        const uint32_t d = tmem + uint32_t(u & 3) * 64;
                        if (c.mma == 1) mma_ts(d, abase + (u & 3) * 32 + ks * 8, bd0 + 2 * ks, id, ks);
                        else mma_ss(d, ad0 + (u & 1) * 1024 + 2 * ks, bd0 + 2 * ks, id, ks);
                    }
                }
            }
            commit1(&bars[warp]);
        }
        __syncwarp();
        mbar_wait(&bars[warp], 0);
        const long long t1 = clock64();
        if (lane == 0 && warp == 0) out[blockIdx.x * 32 + 0] = t1 - t0;
    } else if (warp >= 4 && warp < 4 + c.ld_warps) {
        const int q = (warp - 4) & 3;
        const uint32_t ta = tmem + (uint32_t(q * 32) << 16) + 256;  // columns [256, 384): no overlap with D/A
        uint32_t r[32], acc = 0;
        const int n = c.mma ? 1 << 30 : c.iters;
        int i = 0;
        for (; i < n; ++i) {
            LD32(ta + uint32_t(i & 3) * 32, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 32; ++k) acc += r[k];
            if (c.mma && (i & 15) == 15 && go) break;
        }
        const long long t1 = clock64();
        if (lane == 0) {
            out[blockIdx.x * 32 + 1 + (warp - 4)] = t1 - t0;
            out[blockIdx.x * 32 + 9 + (warp - 4)] = i;
        }
        if (acc == 0x12345678u) sink[0] = acc;
    } else if (warp >= 8 && warp < 8 + c.st_warps) {
        const int q = warp & 3;
        const uint32_t ta = tmem + (uint32_t(q * 32) << 16) + 384 + 64;  // A slots 2-3 (the MMA reads 0-3)
        uint32_t v[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = lane * 77u + k;
        int i = 0;
        for (; i < (1 << 30); ++i) {
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
                "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta + uint32_t(i & 1) * 32),
                "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            if ((i & 15) == 15 && go) break;
        }
        const long long t1 = clock64();
        if (lane == 0) {
            out[blockIdx.x * 32 + 17 + (warp - 8)] = t1 - t0;
            out[blockIdx.x * 32 + 25 + (warp - 8)] = i;
        }
    }
    if (warp == 0 && c.mma && lane == 0) go = 1;  // (multi-issuer: warp 0's time is reported)
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* out;
    unsigned* sink;
    cudaMalloc(&out, sms * 32 * sizeof(long long));
    cudaMalloc(&sink, 64);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    long long h[32];
    auto run = [&](Cfg c, const char* name) {
        cudaMemset(out, 0, sms * 32 * sizeof(long long));
        bench<<<sms, 384, 80 * 1024>>>(c, out, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);  // CTA 0
        printf("%-34s", name);
        if (c.mma) {
            const double cyc = double(h[0]) / c.iters;
            printf(" mma %.1f cyc/MMA (A %s %.1f B/clk)", cyc, c.mma == 1 ? "TMEM" : "smem", 4096.0 / cyc);
        }
        double ldb = 0;
        for (int w = 0; w < c.ld_warps; ++w) {
            const double it = c.mma ? double(h[9 + w]) : double(c.iters);
            ldb += it * 4096.0 / double(h[1 + w]);
        }
        if (c.ld_warps) printf(" ld %.1f B/clk (%d warps)", ldb, c.ld_warps);
        double stb = 0;
        for (int w = 0; w < c.st_warps; ++w) stb += double(h[25 + w]) * 4096.0 / double(h[17 + w]);
        if (c.st_warps) printf(" st %.1f B/clk (%d warps)", stb, c.st_warps);
        printf("\n");
    };
    for (int w : {1, 2, 4, 8}) {
        char nm[64];
        snprintf(nm, sizeof nm, "ld only, %d warps", w);
        run(Cfg{w, 0, 48, 4096, 1}, nm);
    }
    for (int cm : {0, 1, 3}) {
        Cfg c{0, 1, 48, 4096, 1};
        c.variant = 1;
        c.commits = cm;
        char nm[64];
        snprintf(nm, sizeof nm, "v1 N=48, %d commits / 8 MMAs", cm);
        run(c, nm);
    }
    for (int n : {16, 48, 96}) {
        char nm[64];
        snprintf(nm, sizeof nm, "mma TS only, N=%d", n);
        run(Cfg{0, 1, n, 4096, 4}, nm);
        snprintf(nm, sizeof nm, "mma SS only, N=%d", n);
        run(Cfg{0, 2, n, 4096, 4}, nm);
        snprintf(nm, sizeof nm, "mma TS + ld 4 warps, N=%d", n);
        run(Cfg{4, 1, n, 4096, 4}, nm);
        snprintf(nm, sizeof nm, "mma SS + ld 4 warps, N=%d", n);
        run(Cfg{4, 2, n, 4096, 4}, nm);
    }
    return 0;
}
