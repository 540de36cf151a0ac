// Prototype: validate tcgen05 mechanics (TMEM alloc, tcgen05.st A operand, smem
// B descriptor, tcgen05.mma kind::f16 with A in TMEM, commit, tcgen05.ld of D).
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int N>
__global__ void proto(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int variant) {
    __shared__ __align__(1024) uint8_t sB[N * 16 * 2 * 4];  // up to K=64
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)), "n"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    // B: N tokens x 16 k, core-matrix K-major layout [n-group][k-chunk][8 rows][8 elems]
    for (int i = t; i < N * 16; i += blockDim.x) {
        int tok = i / 16, k = i % 16;
        int off = (((tok / 8) * 2 + (k / 8)) * 8 + (tok % 8)) * 8 + (k % 8);
        reinterpret_cast<__nv_bfloat16*>(sB)[off] = B[tok * 16 + k];
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tmem_base;
    // A: row r = t, 8 columns, column c = {A[r][2c], A[r][2c+1]}
    uint32_t r[8];
    for (int c = 0; c < 8; ++c) {
        __nv_bfloat16 lo = A[t * 16 + 2 * c], hi = A[t * 16 + 2 * c + 1];
        if (variant == 1) { lo = A[t * 16 + c]; hi = A[t * 16 + c + 8]; }
        r[c] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
    }
    const uint32_t a_addr = base + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a_addr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (t == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
        const uint32_t saddr = su32(sB);
        const uint64_t bdesc = (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
                               ((uint64_t)((2 * 128) >> 4) << 32) | (1ull << 46);
        const uint32_t d_addr = base + 32;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                     ::"r"(d_addr), "r"(base), "l"(bdesc), "r"(idesc), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
    // wait
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W_%=;\n}\n" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t d[16];
    const uint32_t dl = base + ((uint32_t)(warp * 32) << 16) + 32;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
                   "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
                 : "r"(dl));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16 && j < N; ++j) D[t * N + j] = __uint_as_float(d[j]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(64));
}

int main() {
    const int N = 16;
    __nv_bfloat16 hA[128 * 16], hB[N * 16];
    float fA[128 * 16], fB[N * 16];
    srand(1);
    for (int i = 0; i < 128 * 16; ++i) { fA[i] = (float)(rand() % 17 - 8); hA[i] = __float2bfloat16(fA[i]); }
    for (int i = 0; i < N * 16; ++i) { fB[i] = (float)(rand() % 9 - 4) * 0.5f; hB[i] = __float2bfloat16(fB[i]); }
    __nv_bfloat16 *dA, *dB; float* dD;
    cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, 128 * N * 4);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    for (int variant = 0; variant < 2; ++variant) {
        cudaMemset(dD, 0, 128 * N * 4);
        proto<N><<<1, 128>>>(dA, dB, dD, variant);
        cudaError_t e = cudaDeviceSynchronize();
        float hD[128 * N];
        cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
        int bad = 0; double maxe = 0;
        for (int r = 0; r < 128; ++r) for (int j = 0; j < N; ++j) {
            double ref = 0; for (int k = 0; k < 16; ++k) ref += fA[r * 16 + k] * fB[j * 16 + k];
            double err = fabs(ref - hD[r * N + j]); if (err > 1e-3) ++bad; if (err > maxe) maxe = err;
        }
        printf("variant %d (%s): err=%s bad=%d maxerr=%g  D[0][0..3]=%g %g %g %g\n", variant,
               variant == 0 ? "col c = k{2c,2c+1}" : "col c = k{c,c+8}", cudaGetErrorString(e), bad, maxe,
               hD[0], hD[1], hD[2], hD[3]);
    }
    return 0;
}
