// kernels.cuh -- launcher declarations shared by the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../common.cuh"

namespace rtnq_b200 {

// quant.cu
void launch_group_scales(const void* w, int dtype, int64_t rows, int64_t cols, int bits,
                         int64_t g, int64_t gpr, float* s32, uint16_t* s16, uint16_t* s16n,
                         int32_t* err, cudaStream_t st);
void launch_codes(const void* w, int dtype, int64_t rows, int64_t cols, int bits, int64_t g,
                  int64_t gpr, const float* s32, int8_t* codes, cudaStream_t st);
void launch_encode_from_logical(const int8_t* logical, Layout dst, int bits, int64_t rows,
                                int64_t cols, uint8_t* out, cudaStream_t st);
void launch_relayout(const uint8_t* src, Layout from, uint8_t* dst, Layout to, int bits,
                     int64_t rows, int64_t cols, cudaStream_t st);
void launch_dequant(const uint8_t* codes, Layout L, int bits, int64_t rows, int64_t cols,
                    int64_t g, int64_t gpr, const void* scales, int sdtype, int sorder,
                    void* out, int odtype, cudaStream_t st);
void launch_native_scales(const void* scales, int dtype, int64_t rows, int64_t gpr,
                          uint16_t* out, cudaStream_t st);
void launch_decode(const uint8_t* src, Layout L, int bits, int64_t rows, int64_t cols,
                   int8_t* out, cudaStream_t st);
void launch_check_finite(const void* p, int dtype, int64_t n, int32_t* err, cudaStream_t st);

// quant_fused.cu: one-pass quantize+pack for 16 x 128 tiles.  Returns false
// (launching nothing) when the shape is outside the fused kernel's domain.
bool quant_fused_supported(int64_t rows, int64_t cols, int bits, int64_t g);
// quant_native.cu: one-pass quantize straight into RTNQ_NATIVE_I4 (W4 g128) / RTNQ_NATIVE_I8
// (W8 per-channel), plus row-major bytes and scales
bool quant_i4_supported(int64_t rows, int64_t cols, int bits, int64_t g);
bool quant_rowwise_supported(int64_t rows, int64_t cols, int bits, int64_t g);
void launch_quant_i4(const void* w, int dtype, int64_t rows, int64_t cols, uint8_t* ni4, uint8_t* rm, float* s32,
                     uint16_t* s16, uint16_t* s16n, int32_t* err, cudaStream_t st);
void launch_quant_rowwise(const void* w, int dtype, int64_t rows, int64_t cols, uint8_t* ni8, uint8_t* rm,
                          float* s32, uint16_t* s16, uint16_t* s16n, int32_t* err, cudaStream_t st);
void launch_quant_fused(const void* w, int dtype, int64_t rows, int64_t cols, int bits,
                        int64_t g, uint8_t* rm, uint8_t* k164, uint8_t* nat, float* s32,
                        uint16_t* s16, uint16_t* s16n, int32_t* err, cudaStream_t st);

// gemm_exact.cu
void launch_gemm_fused_exact(const float* a, int64_t m, int64_t k, const uint8_t* codes,
                             Layout L, int bits, int64_t n, int64_t g, int64_t gpr,
                             const float* scales, float* out, cudaStream_t st);
void launch_dense_blocked(const float* a, int64_t m, int64_t k, const float* w, int64_t n,
                          int64_t blk, float* out, cudaStream_t st);
void launch_gemm_oracle(const float* a, int64_t m, int64_t k, const uint8_t* codes, Layout L,
                        int bits, int64_t n, int64_t g, int64_t gpr, const float* scales,
                        float* out, cudaStream_t st);

// wgemm_sm100.cu: tensor-core W4A16 / W8A16 over the native layout.
// A row-split linear's output pushed into every tensor-parallel rank's symmetric buffer
// (int8_mma.cuh, "partial sums over peer memory"); world 0: plain local output.
constexpr int kPeerMax = 8;
constexpr int kPeerHeader = 256;
struct PeerOut {
    int world = 0, rank = 0;
    char* bufs[kPeerMax] = {};  // every rank's symmetric buffer, mapped into this process
    int64_t cap = 0;            // elements per slot
};
// the consumer side: this rank's own buffer (the slots every rank's partial landed in)
struct PeerIn {
    char* buf = nullptr;
    int world = 0;
    int64_t cap = 0;
};
size_t peer_buffer_bytes(int64_t cap);
// out[i] (+)= sum over ranks of slot[i], i < n (rank order, f32, one bf16 rounding); then the
// round is consumed (peer.cu)
cudaError_t launch_peer_reduce(const PeerIn& pin, void* out, int64_t n, bool accumulate, cudaStream_t st);

struct WgemmArgs {
    const void* a;         // m x k, bf16 or f16, row-major
    int a_dtype;           // RTNQ_BF16 | RTNQ_F16
    int64_t m, n, k;
    const uint8_t* codes;  // native layout
    const uint16_t* scales;  // f16, native order
    int bits;
    int64_t g;             // group size (g >= k: one group per row)
    void* out;             // m x n, row-major
    int out_dtype;
    void* workspace;
    size_t ws_bytes;
    bool pdl;              // launch with programmatic dependent launch (RTNQ_FLAG_PDL)
    // int8 kernels: activation planes computed by the producer of `a` (nullptr: the linear
    // computes them itself); [3][m][k] int8 and [m] exponents
    const int8_t* planes = nullptr;
    const int32_t* texp = nullptr;
    // int8 kernels computing their own planes: |= 1 on a non-finite activation (the planes
    // kernel's max pass checks it; InvalidInputError in the reference, gemm.cpp:13-19)
    int32_t* err = nullptr;
    // tensor parallel: push the output into every rank's slot instead of `out` (world > 0)
    PeerOut peer{};
};
// Validates the shape for the tensor-core path; returns a message or nullptr.
const char* wgemm_unsupported(int64_t m, int64_t n, int64_t k, int bits, int64_t g, int a_dtype);
size_t wgemm_workspace_bytes(int64_t m, int64_t n, int64_t k, int bits, int64_t g);
cudaError_t launch_wgemm(const WgemmArgs& args, cudaStream_t st);

// wgemm_i8.cu: W8 per-channel on tcgen05.mma.kind::i8 over RTNQ_NATIVE_I8 tiles (no dequant)
const char* wgemm_i8_unsupported(int64_t m, int64_t n, int64_t k, int bits, int64_t g, int a_dtype);
size_t wgemm_i8_workspace_bytes(int64_t m, int64_t n, int64_t k);
cudaError_t launch_wgemm_i8(const WgemmArgs& args, cudaStream_t st);

// dequant_first.cu: exact dequant into hi + lo 16-bit terms, then two cuBLAS GEMMs (f32 C)
size_t dequant_first_workspace_bytes(int64_t m, int64_t n, int64_t k, int odtype);
const char* launch_dequant_first(const void* a, int a_dtype, int64_t m, int64_t n, int64_t k,
                                 const uint8_t* codes, Layout L, int bits, int64_t g, int64_t gpr,
                                 const uint16_t* scales, int sorder, void* out, int odtype, void* ws,
                                 cudaStream_t st);
// dense_tc.cu: out[m][n] = a . (hi + lo)^T on tcgen05 (16-bit operands, f32 accumulation)
const char* launch_dense_hilo(const void* a, int64_t lda, const void* hi, const void* lo, int64_t ldw, int a_dtype,
                              int64_t m, int64_t n, int64_t k, void* out, int odtype, cudaStream_t st);

// wgemm_i4.cu: W4 group-128 on tcgen05.mma.kind::i8 over RTNQ_NATIVE_I4 nibble tiles
const char* wgemm_i4_unsupported(int64_t m, int64_t n, int64_t k, int bits, int64_t g, int a_dtype);
size_t wgemm_i4_workspace_bytes(int64_t m, int64_t n, int64_t k);
cudaError_t launch_wgemm_i4(const WgemmArgs& args, cudaStream_t st);

// decode.cu: the non-GEMM kernels of a decode layer (bf16 activations)
// planes/texp (optional, bf16 rows): also write the int8 GEMMs' activation planes of the output
// pin.buf: the delta is the sum of the ranks' partials of the current round (peer memory)
cudaError_t launch_add_rmsnorm(void* x, const void* delta, const void* w, void* out, int64_t m,
                               int64_t h, float eps, cudaStream_t st, int8_t* planes = nullptr,
                               int32_t* texp = nullptr, PeerIn pin = PeerIn{});
cudaError_t launch_silu_mul(const void* gu, void* act, int64_t m, int64_t f, cudaStream_t st,
                            int8_t* planes = nullptr, int32_t* texp = nullptr);
// the activation planes alone ([3][m][k] int8, [m] exponents) of a bf16/f16 activation
cudaError_t launch_act_planes(const void* a, int a_dtype, int64_t m, int64_t k, int8_t* planes,
                              int32_t* texp, cudaStream_t st);
size_t decode_attention_workspace_bytes(int64_t batch, int64_t hq, int64_t hkv, int64_t max_len);
cudaError_t launch_decode_attention(const void* qkv, void* kcache, void* vcache, void* out,
                                    int64_t batch, int64_t hq, int64_t hkv, int64_t head_dim,
                                    int64_t lmax, int64_t pos, float theta, cudaStream_t st,
                                    void* ws = nullptr, size_t ws_bytes = 0, int8_t* planes = nullptr,
                                    int32_t* texp = nullptr);

}  // namespace rtnq_b200
