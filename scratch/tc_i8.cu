// kind::i8 MMA throughput, A and B from shared memory (SS), M=128, N in {16,48,96}, K=32.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc) : "memory"); }
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(bd), "r"(id), "r"(acc) : "memory"); }
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc) : "memory"); }
template <int N>
__global__ void k(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar; __shared__ uint32_t ts;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 96 * 1024; i += blockDim.x) base[i] = (uint8_t)(i * 2654435761u >> 24);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&ts))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = ts;
  if (warp == 0) {
    // A: 128 rows x 32 B per MMA, K-major no swizzle: core matrix 8 rows x 16 B; LBO (k) = 2048, SBO (8 rows) = 128
    const uint32_t a0 = su32(base);
    const uint64_t ahi = (uint64_t(2048 >> 4) << 16) | (uint64_t(128 >> 4) << 32) | (1ull << 46);
    // B: N rows x 32 B: LBO = N*16, SBO = 128
    const uint32_t b0 = su32(base + 64 * 1024);
    const uint64_t bhi = (uint64_t((N * 16) >> 4) << 16) | (uint64_t(128 >> 4) << 32) | (1ull << 46);
    const uint32_t id_i8 = (2u << 4) | (0u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (8u << 24);
    const uint32_t id_f16 = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (8u << 24);
    // 128B-swizzled K-major A: atom = 8 rows x 128 B (1 KB); SBO = 1024 (next 8 rows), LBO unused (1),
    // layout type 2 (SWIZZLE_128B) in bits 61-63; a k32 step advances the start address by 32 B
    const uint64_t ahs = (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
    uint32_t ph = 0;
    {
      long long t0 = clock64();
      for (int i = 0; i < 256; ++i) {
        const int tile = (i >> 2) & 3, ks = i & 3;  // 16 KB tiles (128 rows x 128 B), 4 k32 steps each
        const uint64_t ad = ahs | (((a0 + tile * 16384 + ks * 32) >> 4) & 0x3FFF);
        const uint64_t bd = bhi | (((b0 + (i & 7) * N * 32) >> 4) & 0x3FFF);
        mma_i8(tmem, ad, bd, id_i8, i & 3);
      }
      commit(&bar); mbar_wait(&bar, ph); ph ^= 1;
      long long t1 = clock64();
      if (lane == 0) out[3] = (t1 - t0) / 256;
    }
    {
      // TS: A from TMEM (cols 256.. : 4 slots x 32 cols), B SW128 from smem
      const uint64_t bhs = (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
      long long t0 = clock64();
      for (int i = 0; i < 256; ++i) {
        const int slot = (i >> 2) & 3, ks = i & 3;
        const uint64_t bd = bhs | (((b0 + ks * 32) >> 4) & 0x3FFF);
        mma_i8_ts(tmem + ((i >> 2) & 1) * 128, tmem + 256 + slot * 32 + ks * 8, bd, id_i8, ks);
      }
      commit(&bar); mbar_wait(&bar, ph); ph ^= 1;
      long long t1 = clock64();
      if (lane == 0) out[4] = (t1 - t0) / 256;
    }
    {
      // 8 TS MMAs per asm block (one elect), precomputed operands
      const uint64_t bhs = (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
      const uint64_t bd0 = bhs | (((b0) >> 4) & 0x3FFF);
      long long t0 = clock64();
      for (int i = 0; i < 32; ++i) {
        const uint32_t d = tmem + (i & 1) * 128, a = tmem + 256 + (i & 3) * 32;
        asm volatile("{\n.reg .pred e;\n.reg .b64 b1, b2, b3;\nelect.sync _|e, 0xffffffff;\n"
                     "add.u64 b1, %2, 2;\nadd.u64 b2, %2, 4;\nadd.u64 b3, %2, 6;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 0;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%4], b1, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%5], b2, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%6], b3, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%4], b1, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%5], b2, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%6], b3, %3, 1;\n}\n"
                     :: "r"(d), "r"(a), "l"(bd0), "r"(id_i8), "r"(a + 8), "r"(a + 16), "r"(a + 24) : "memory");
      }
      commit(&bar); mbar_wait(&bar, ph); ph ^= 1;
      long long t1 = clock64();
      if (lane == 0) out[5] = (t1 - t0) / 256;
      // same with SS (A SW128 from smem)
      const uint64_t ad0 = ahs | (((a0) >> 4) & 0x3FFF);
      t0 = clock64();
      for (int i = 0; i < 32; ++i) {
        const uint32_t d = tmem + (i & 1) * 128;
        const uint64_t ad = ad0 + (i & 3) * (16384 >> 4);
        asm volatile("{\n.reg .pred e;\n.reg .b64 a1, a2, a3, b1, b2, b3;\nelect.sync _|e, 0xffffffff;\n"
                     "add.u64 a1, %1, 2;\nadd.u64 a2, %1, 4;\nadd.u64 a3, %1, 6;\n"
                     "add.u64 b1, %2, 2;\nadd.u64 b2, %2, 4;\nadd.u64 b3, %2, 6;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 0;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a2, b2, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a3, b3, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a2, b2, %3, 1;\n"
                     "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a3, b3, %3, 1;\n}\n"
                     :: "r"(d), "l"(ad), "l"(bd0), "r"(id_i8) : "memory");
      }
      commit(&bar); mbar_wait(&bar, ph); ph ^= 1;
      t1 = clock64();
      if (lane == 0) out[6] = (t1 - t0) / 256;
    }
    for (int pass = 0; pass < 3; ++pass) {
      long long t0 = clock64();
      for (int i = 0; i < 256; ++i) {
        const uint64_t ad = ahi | (((a0 + (i & 15) * 4096) >> 4) & 0x3FFF);   // fresh 4 KB A tiles
        const uint64_t bd = bhi | (((b0 + (i & 7) * N * 32) >> 4) & 0x3FFF);
        if (pass < 2) mma_i8(tmem, ad, bd, id_i8, i & 3);
        else mma_f16(tmem, ad, bd, id_f16, i & 3);
      }
      commit(&bar); mbar_wait(&bar, ph); ph ^= 1;
      long long t1 = clock64();
      if (lane == 0) out[pass] = (t1 - t0) / 256;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) { asm volatile("tcgen05.fence::after_thread_sync;"); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem)); }
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[7];
  auto run = [&](auto kern, int n) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    kern<<<1, 128, 100 * 1024>>>(d); cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("N=%d err %s\n", n, cudaGetErrorString(e)); return; }
    cudaMemcpy(h, d, 56, cudaMemcpyDeviceToHost);
    printf("N=%3d: i8 SS noswz %lld; f16 SS %lld; i8 SS SW128 %lld; i8 TS %lld | batched x8: TS %lld SS %lld cycles/MMA\n", n, h[0], h[2], h[3], h[4], h[5], h[6]);
  };
  run(k<16>, 16); run(k<48>, 48); run(k<96>, 96);
  return 0;
}
