// Tensor-parallel partial sums over peer memory: the symmetric buffer's size and
// the stand-alone consumer (sum of the ranks' slots of the current round).  The producers are the
// row-split int8 linears (wgemm_i4.cu / wgemm_i8.cu with WgemmArgs::peer); the fused consumer is
// add+RMSNorm (decode.cu, PeerIn).  Protocol: int8_mma.cuh, "partial sums over peer memory".
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "int8_mma.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {

size_t peer_buffer_bytes(int64_t cap) {
    return size_t(kPeerHeader) + size_t(2) * kPeerMax * size_t(cap) * sizeof(__nv_bfloat16);
}

namespace {

// grid-stride over 8-element vectors; thread 0 of each CTA waits for the round, the last CTA to
// finish reading consumes it
__global__ void __launch_bounds__(256) peer_reduce_kernel(PeerIn pin, __nv_bfloat16* __restrict__ out, int64_t n8,
                                                          int accumulate) {
    const int e = *reinterpret_cast<volatile int*>(imma::peer_epoch(pin.buf)) + 1;
    if (threadIdx.x == 0) imma::peer_wait(pin.buf, pin.world, e);
    __syncthreads();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
        float acc[8] = {};
        for (int q = 0; q < pin.world; ++q) {
            const uint4 sv = imma::peer_ld16(imma::peer_slot(pin.buf, pin.cap, e & 1, q) + i * 8);
            const __nv_bfloat162* sp = reinterpret_cast<const __nv_bfloat162*>(&sv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __bfloat1622float2(sp[j]);
                acc[2 * j] += f.x, acc[2 * j + 1] += f.y;
            }
        }
        uint4 ov;
        __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&ov);
        if (accumulate) {  // out += bf16(sum): the same two roundings as out += allreduce(partial)
            const uint4 xv = *reinterpret_cast<const uint4*>(out + i * 8);
            const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&xv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 d = __bfloat1622float2(__floats2bfloat162_rn(acc[2 * j], acc[2 * j + 1]));
                const float2 x = __bfloat1622float2(xp[j]);
                op[j] = __floats2bfloat162_rn(x.x + d.x, x.y + d.y);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) op[j] = __floats2bfloat162_rn(acc[2 * j], acc[2 * j + 1]);
        }
        *reinterpret_cast<uint4*>(out + i * 8) = ov;
    }
    __syncthreads();
    if (threadIdx.x == 0) imma::peer_consumed_by(pin.buf, int(gridDim.x));
}

}  // namespace

cudaError_t launch_peer_reduce(const PeerIn& pin, void* out, int64_t n, bool accumulate, cudaStream_t st) {
    if (!pin.buf || pin.world < 1 || pin.world > kPeerMax || n % 8 || n > pin.cap) return cudaErrorInvalidValue;
    const int64_t n8 = n / 8;
    int64_t blocks = (n8 + 255) / 256;
    blocks = blocks < 1 ? 1 : blocks > 148 ? 148 : blocks;
    peer_reduce_kernel<<<unsigned(blocks), 256, 0, st>>>(pin, static_cast<__nv_bfloat16*>(out), n8, accumulate ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace rtnq_b200
