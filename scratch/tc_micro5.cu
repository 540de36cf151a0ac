// Microbenchmark of tcgen05 / mbarrier primitive costs on one SM (cycles, clock64).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(bd), "r"(id), "r"(acc) : "memory"); }
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred e, p;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(acc) : "memory"); }

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


template <int NT>
__global__ void micro(long long* out, int iters, int fill) {
  __shared__ __align__(1024) uint8_t act[32 * 1024];
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32 * 1024; i += blockDim.x) act[i] = (fill ? uint8_t((i * 2654435761u) >> 24) & 0x3F : 0);
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (fill && warp < 4) {
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = 0x3F803F80u ^ ((threadIdx.x * 131 + i * 7) & 0x007F007F);
    for (int c = 0; c < 256; c += 32)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + (uint32_t(warp * 32) << 16) + c),
        "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),"r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]),
        "r"(v[16]),"r"(v[17]),"r"(v[18]),"r"(v[19]),"r"(v[20]),"r"(v[21]),"r"(v[22]),"r"(v[23]),"r"(v[24]),"r"(v[25]),"r"(v[26]),"r"(v[27]),"r"(v[28]),"r"(v[29]),"r"(v[30]),"r"(v[31]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(NT >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t bdesc = uint64_t((su32(act) >> 4) & 0x3FFF) | (uint64_t((NT * 16) >> 4) << 16) | (uint64_t(128 >> 4) << 32) | (1ull << 46);
    const uint64_t adesc = uint64_t((su32(act) >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (1ull << 46);
    uint32_t ph = 0, ph1 = 0;
    long long t0, t1;
    // (13) sweep: B tiles cycled (512 B each) x A tiles cycled, D alternating every 8
    {
      const int bcyc[5] = {1, 2, 8, 32, 64};
      for (int bi = 0; bi < 5; ++bi)
        for (int aa = 0; aa < 2; ++aa) {
          t0 = clock64();
#pragma unroll 16
          for (int k = 0; k < 1024; ++k)
            mma(tmem + 384 + ((k >> 3) & 1) * NT, tmem + (aa ? (k & 15) * 8 : 0),
                bdesc + (k & (bcyc[bi] - 1)) * 2 * NT, idesc, (k & 7) != 0);
          commit(&bar[2]); mbar_wait(&bar[2], (bi * 2 + aa) & 1);
          t1 = clock64(); if (lane == 0) out[16 + bi * 2 + aa] = (t1 - t0) / 1024;
        }
    }
    // (1) commit + wait round trip with nothing in flight
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { commit(&bar[0]); mbar_wait(&bar[0], ph); ph ^= 1; }
    t1 = clock64(); if (lane == 0) out[0] = (t1 - t0) / iters;
    // (2) issue cost: 8 MMAs (A in TMEM) back to back, no waiting
    t0 = clock64();
    for (int i = 0; i < iters; ++i) for (int k = 0; k < 8; ++k) mma(tmem + 256, tmem + k * 8, bdesc + k * 2 * NT, idesc, 1);
    t1 = clock64(); if (lane == 0) out[1] = (t1 - t0) / (iters * 8);
    commit(&bar[0]); mbar_wait(&bar[0], ph); ph ^= 1;
    // (3) 8 MMAs + commit + wait: the latency of one unit
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { for (int k = 0; k < 8; ++k) mma(tmem + 256, tmem + k * 8, bdesc + k * 2 * NT, idesc, 1); commit(&bar[0]); mbar_wait(&bar[0], ph); ph ^= 1; }
    t1 = clock64(); if (lane == 0) out[2] = (t1 - t0) / iters;
    // (4) throughput: 64 MMAs then one commit+wait
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { for (int k = 0; k < 64; ++k) mma(tmem + 256, tmem + (k & 7) * 8, bdesc + (k & 7) * 2 * NT, idesc, 1); }
    commit(&bar[0]); mbar_wait(&bar[0], ph); ph ^= 1;
    t1 = clock64(); if (lane == 0) out[3] = (t1 - t0) / (iters * 64);
    // (5) same with A from SMEM (SS)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { for (int k = 0; k < 64; ++k) mma_ss(tmem + 256, adesc + (k & 7) * 16, bdesc + (k & 7) * 2 * NT, idesc, 1); }
    commit(&bar[0]); mbar_wait(&bar[0], ph); ph ^= 1;
    t1 = clock64(); if (lane == 0) out[4] = (t1 - t0) / (iters * 64);
    // (6) mbarrier arrive + wait (count 1) by one lane
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { if (lane == 0) mbar_arrive(&bar[1]); mbar_wait(&bar[1], ph1); ph1 ^= 1; }
    t1 = clock64(); if (lane == 0) out[5] = (t1 - t0) / iters;
    // (7) STTM x32 + wait::st
    uint32_t v[32]; for (int i = 0; i < 32; ++i) v[i] = i;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + (i & 3) * 32),
        "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),"r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]),
        "r"(v[16]),"r"(v[17]),"r"(v[18]),"r"(v[19]),"r"(v[20]),"r"(v[21]),"r"(v[22]),"r"(v[23]),"r"(v[24]),"r"(v[25]),"r"(v[26]),"r"(v[27]),"r"(v[28]),"r"(v[29]),"r"(v[30]),"r"(v[31]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    t1 = clock64(); if (lane == 0) out[6] = (t1 - t0) / iters;
    // (8) LDTM x16 + wait::ld
    uint32_t acc = 0;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint32_t d[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(d[0]),"=r"(d[1]),"=r"(d[2]),"=r"(d[3]),"=r"(d[4]),"=r"(d[5]),"=r"(d[6]),"=r"(d[7]),"=r"(d[8]),"=r"(d[9]),"=r"(d[10]),"=r"(d[11]),"=r"(d[12]),"=r"(d[13]),"=r"(d[14]),"=r"(d[15]) : "r"(tmem + 256 + (i & 3) * 16) : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += d[0] ^ d[15];
    }
    t1 = clock64(); if (lane == 0) { out[7] = (t1 - t0) / iters; out[15] = acc; }
    // (9) fence::after_thread_sync
    t0 = clock64();
    for (int i = 0; i < iters; ++i) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    t1 = clock64(); if (lane == 0) out[8] = (t1 - t0) / iters;
    // (11) throughput with rotating operands: A over 32 k16 steps (256 cols), B over 16 KB, D over 2 buffers
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { for (int k = 0; k < 64; ++k) mma(tmem + 256 + ((k >> 3) & 1) * NT, tmem + (k & 31) * 8, bdesc + ((k * 2 * NT) & 1023), idesc, (k & 7) != 0); }
    commit(&bar[0]); mbar_wait(&bar[0], ph); ph ^= 1;
    t1 = clock64(); if (lane == 0) out[10] = (t1 - t0) / (iters * 64);
    // (12) the kernel's 8-MMA asm block, A/B/D rotating like the kernel (D at 384)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      for (int u = 0; u < 8; ++u)
        umma_unit_elect<8, uint32_t((2 * NT * 16) / 16)>(tmem + 384 + (u & 1) * NT, tmem + (u & 3) * 64, bdesc + u * 8 * 2 * NT, idesc, 0);
    }
    commit(&bar[0]); mbar_wait(&bar[0], ph); ph ^= 1;
    t1 = clock64(); if (lane == 0) out[11] = (t1 - t0) / (iters * 64);
    // (10) one UMMA latency: mma + commit + wait
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { mma(tmem + 256, tmem, bdesc, idesc, 1); commit(&bar[0]); mbar_wait(&bar[0], ph); ph ^= 1; }
    t1 = clock64(); if (lane == 0) out[9] = (t1 - t0) / iters;
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) { asm volatile("tcgen05.fence::after_thread_sync;"); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem)); }
}

int main() {
  long long* d; cudaMalloc(&d, 32 * 8);
  const char* names[] = {"commit+wait (idle)", "mma issue (A tmem)", "8 mma+commit+wait", "mma thrpt (A tmem)", "mma thrpt (A smem)",
                         "arrive+wait", "STTM x32 + wait::st", "LDTM x16 + wait::ld", "fence::after", "1 mma+commit+wait", "mma thrpt rotating", "kernel unit asm (per MMA)", "COLD 384 MMAs (per MMA)", "then warm (per MMA)"};
  cudaFuncSetAttribute(micro<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
  for (int cfg = 0; cfg < 1; ++cfg)
  for (int fill : {1})
  for (int nt : {16}) {
    const int threads = (cfg & 1) ? 480 : 128;
    const int dyn = (cfg & 2) ? 180 * 1024 : 0;
    long long h[32];
    for (int rep = 0; rep < 2; ++rep) {
      if (nt == 16) micro<16><<<1, threads, dyn>>>(d, 200, fill); else micro<64><<<1, threads, dyn>>>(d, 200, fill);
      cudaError_t e = cudaDeviceSynchronize(); if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("NT=%d fill=%d threads=%d dyn=%d\n", nt, fill, threads, dyn);
    for (int i = 0; i < 12; ++i) printf("  %-24s %lld cycles\n", names[i], h[i]);
    const int bcyc[5] = {1, 2, 8, 32, 64};
    for (int i = 0; i < 10; ++i) printf("  B tiles %2d, A tiles %2d: %lld cycles/MMA\n", bcyc[i / 2], (i & 1) ? 16 : 1, h[16 + i]);
  }
  return 0;
}
