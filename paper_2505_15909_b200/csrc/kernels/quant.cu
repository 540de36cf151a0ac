// quant.cu -- RTN quantize-and-pack, layout conversion and dequantization.
//
// Two quantize paths, both bit-exact with the reference:
//   * fused (quant_pack_fused_kernel, quant_fused.cu): one pass over 16-row x
//     128-column tiles for the common shapes (even cols, g in {16..128} or g = cols);
//   * generic (this file): group scales -> logical int8 codes -> per-layout
//     encoders, for any shape the reference accepts (odd widths, g = 1..2^k,
//     ragged tails, per-channel groups wider than a tile).
#include <float.h>

#include "../common.cuh"
#include "kernels.cuh"

namespace rtnq_b200 {

// One warp per (row, group): absmax with the reference's finiteness check
// (quant.cpp:50-57), then scale_from_absmax (quant.cpp:58-67).
__global__ void group_scales_kernel(const void* __restrict__ w, int dtype, int64_t rows,
                                    int64_t cols, int bits, int64_t g, int64_t gpr,
                                    float* __restrict__ s32, uint16_t* __restrict__ s16,
                                    uint16_t* __restrict__ s16n, int32_t* __restrict__ err) {
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= rows * gpr) return;
    const int64_t r = warp / gpr, j = warp % gpr, c0 = j * g;
    const int64_t len = min(g, cols - c0);
    float amax = 0.0f;
    bool bad = false;
    const int64_t base = r * cols + c0;
    for (int64_t i = lane; i < len; i += 32) {
        const float a = fabsf(load_elem(w, dtype, base + i));
        bad |= !(a <= FLT_MAX);
        amax = fmaxf(amax, a);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        if (bad && err) atomicOr(err, 1);
        const float s = bad ? 1.0f : scale_from_absmax(amax, bits);
        if (s32) s32[r * gpr + j] = s;
        const uint16_t h = __half_as_ushort(__float2half_rn(s));
        if (s16) s16[r * gpr + j] = h;
        if (s16n) s16n[native_scale_index(rows, gpr, r, j)] = h;
    }
}

// Logical int8 codes (quant.cpp:118-136) from precomputed f32 scales.
__global__ void codes_kernel(const void* __restrict__ w, int dtype, int64_t rows, int64_t cols,
                             int bits, int64_t g, int64_t gpr, const float* __restrict__ s32,
                             int8_t* __restrict__ codes) {
    const int64_t n = rows * cols;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / cols, c = i % cols;
        codes[i] = int8_t(quantize_one(load_elem(w, dtype, i), s32[r * gpr + c / g], bits));
    }
}

// Code for storage slot `slot` of layout `dst`, taken from a logical int8
// matrix (src == nullptr -> logical) or from packed codes in layout `src_l`.
struct CodeSource {
    const int8_t* logical;
    const uint8_t* packed;
    Layout src_l;
};

__device__ __forceinline__ int source_code(const CodeSource& S, int bits, int64_t rows,
                                           int64_t cols, int64_t r, int64_t c) {
    if (S.logical) return S.logical[r * cols + c];
    return code_at_slot(S.packed, bits, layout_slot(S.src_l, bits, rows, cols, r, c), S.src_l.kind);
}

// One thread per output byte: gathers its 1 (8-bit) or 2 (4-bit) slots,
// zero codes in padding (packing.cpp:83-90 + pack, :6-32).
__global__ void encode_layout_kernel(CodeSource S, Layout dst, int bits, int64_t rows,
                                     int64_t cols, int64_t nbytes, uint8_t* __restrict__ out) {
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < nbytes;
         b += int64_t(gridDim.x) * blockDim.x) {
        int64_t r, c;
        if (bits == 8) {
            const int code = layout_coords(dst, bits, rows, cols, b, &r, &c)
                                 ? source_code(S, bits, rows, cols, r, c) : 0;
            out[b] = code_byte8(code, dst.kind);
        } else {
            const int64_t nslots = layout_slots_of(dst, bits, rows, cols);
            uint32_t v = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t slot = 2 * b + h;
                int code = 0;
                if (slot < nslots && layout_coords(dst, bits, rows, cols, slot, &r, &c))
                    code = source_code(S, bits, rows, cols, r, c);
                // pack(): an odd tail leaves the high nibble 0 (packing.cpp:28-29)
                if (slot < nslots) v |= code_nib4(code, dst.kind) << (4 * h);
            }
            out[b] = uint8_t(v);
        }
    }
}

// dequantize_tensor (quant.cpp:143-171): float(code) * S, one rounding.
__global__ void dequant_kernel(const uint8_t* __restrict__ codes, Layout L, int bits,
                               int64_t rows, int64_t cols, int64_t g, int64_t gpr,
                               const void* __restrict__ scales, int sdtype, int sorder,
                               void* __restrict__ out, int odtype) {
    const int64_t n = rows * cols;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / cols, c = i % cols;
        const int code = code_at_slot(codes, bits, layout_slot(L, bits, rows, cols, r, c), L.kind);
        const float s = load_scale(scales, sdtype, sorder, rows, gpr, r, c / g);
        store_elem(out, odtype, i, __fmul_rn(float(code), s));
    }
}

__global__ void native_scales_kernel(const void* __restrict__ scales, int dtype, int64_t rows,
                                     int64_t gpr, uint16_t* __restrict__ out) {
    const int64_t n = gpr * ((rows + 7) / 8 * 8);
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        // invert native_scale_index: i -> (row-block, group, row)
        const int64_t rb = i / (int64_t(kNativeRows) * gpr), off = i % (int64_t(kNativeRows) * gpr);
        const int64_t r8 = native_scale_rows8(rows, rb);
        const int64_t j = off / r8, row = off % r8;
        const int64_t r = rb * kNativeRows + row;
        uint16_t h = 0;
        if (row < native_rows_in(rows, rb)) {
            if (dtype == RTNQ_F16) h = static_cast<const uint16_t*>(scales)[r * gpr + j];
            else h = __half_as_ushort(__float2half_rn(load_elem(scales, dtype, r * gpr + j)));
        }
        out[i] = h;
    }
}

// Any layout -> logical row-major int8 codes (logical_codes / unpack).
__global__ void decode_kernel(const uint8_t* __restrict__ src, Layout L, int bits, int64_t rows,
                              int64_t cols, int8_t* __restrict__ out) {
    const int64_t n = rows * cols;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / cols, c = i % cols;
        out[i] = int8_t(code_at_slot(src, bits, layout_slot(L, bits, rows, cols, r, c), L.kind));
    }
}

__global__ void check_finite_kernel(const void* __restrict__ p, int dtype, int64_t n,
                                    int32_t* __restrict__ err) {
    bool bad = false;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        bad |= !isfinite(load_elem(p, dtype, i));
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1);
}

// ---- launchers -----------------------------------------------------------------------

static int grid_for(int64_t n, int threads = 256) {
    const int64_t b = (n + threads - 1) / threads;
    return int(b < 1 ? 1 : (b > 148 * 64 ? 148 * 64 : b));
}

void launch_group_scales(const void* w, int dtype, int64_t rows, int64_t cols, int bits,
                         int64_t g, int64_t gpr, float* s32, uint16_t* s16, uint16_t* s16n,
                         int32_t* err, cudaStream_t st) {
    const int64_t warps = rows * gpr;
    if (warps == 0) return;
    const int64_t blocks = (warps * 32 + 255) / 256;
    group_scales_kernel<<<unsigned(blocks), 256, 0, st>>>(w, dtype, rows, cols, bits, g, gpr,
                                                          s32, s16, s16n, err);
}

void launch_codes(const void* w, int dtype, int64_t rows, int64_t cols, int bits, int64_t g,
                  int64_t gpr, const float* s32, int8_t* codes, cudaStream_t st) {
    if (rows * cols == 0) return;
    codes_kernel<<<grid_for(rows * cols), 256, 0, st>>>(w, dtype, rows, cols, bits, g, gpr, s32,
                                                        codes);
}

void launch_encode_from_logical(const int8_t* logical, Layout dst, int bits, int64_t rows,
                                int64_t cols, uint8_t* out, cudaStream_t st) {
    const int64_t nbytes = (layout_slots_of(dst, bits, rows, cols) * bits + 7) / 8;
    if (nbytes == 0) return;
    CodeSource S{logical, nullptr, Layout{0, 16, 4}};
    encode_layout_kernel<<<grid_for(nbytes), 256, 0, st>>>(S, dst, bits, rows, cols, nbytes, out);
}

void launch_relayout(const uint8_t* src, Layout from, uint8_t* dst, Layout to, int bits,
                     int64_t rows, int64_t cols, cudaStream_t st) {
    const int64_t nbytes = (layout_slots_of(to, bits, rows, cols) * bits + 7) / 8;
    if (nbytes == 0) return;
    CodeSource S{nullptr, src, from};
    encode_layout_kernel<<<grid_for(nbytes), 256, 0, st>>>(S, to, bits, rows, cols, nbytes, dst);
}

void launch_dequant(const uint8_t* codes, Layout L, int bits, int64_t rows, int64_t cols,
                    int64_t g, int64_t gpr, const void* scales, int sdtype, int sorder,
                    void* out, int odtype, cudaStream_t st) {
    if (rows * cols == 0) return;
    dequant_kernel<<<grid_for(rows * cols), 256, 0, st>>>(codes, L, bits, rows, cols, g, gpr,
                                                          scales, sdtype, sorder, out, odtype);
}

void launch_native_scales(const void* scales, int dtype, int64_t rows, int64_t gpr,
                          uint16_t* out, cudaStream_t st) {
    const int64_t n = gpr * ((rows + 7) / 8 * 8);
    if (n == 0) return;
    native_scales_kernel<<<grid_for(n), 256, 0, st>>>(scales, dtype, rows, gpr, out);
}

void launch_decode(const uint8_t* src, Layout L, int bits, int64_t rows, int64_t cols,
                   int8_t* out, cudaStream_t st) {
    if (rows * cols == 0) return;
    decode_kernel<<<grid_for(rows * cols), 256, 0, st>>>(src, L, bits, rows, cols, out);
}

void launch_check_finite(const void* p, int dtype, int64_t n, int32_t* err, cudaStream_t st) {
    if (n == 0) return;
    check_finite_kernel<<<grid_for(n), 256, 0, st>>>(p, dtype, n, err);
}

}  // namespace rtnq_b200
