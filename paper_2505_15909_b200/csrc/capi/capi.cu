// capi.cu -- the extern "C" boundary (include/rtnq_capi.h).
//
// rtnq_dev_*: validate, pick a kernel, launch on the caller's stream.
// rtnq_* (host): reference-identical validation, then H2D -> the same kernels
// -> D2H on a library-private stream.  No host compute path exists: every
// number these functions return was produced by a kernel in csrc/kernels/.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "../../../include/rtnq_capi.h"
#include "../kernels/kernels.cuh"

using namespace rtnq_b200;

namespace {

thread_local std::string g_err;

rtnq_status fail(rtnq_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

#define RTNQ_CUDA(expr)                                                                \
    do {                                                                               \
        cudaError_t e_ = (expr);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return fail(RTNQ_E_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
    } while (0)

Layout to_layout(rtnq_layout l) { return Layout{l.kind, l.tile_rows, l.tile_cols}; }

bool valid_bits(int bits) { return bits == 4 || bits == 8; }

rtnq_status check_layout(rtnq_layout l) {
    if (l.kind < RTNQ_ROW_MAJOR || l.kind > RTNQ_NATIVE_I4)
        return fail(RTNQ_E_INVALID_INPUT, "unknown layout kind");
    if (l.kind == RTNQ_KERNEL_INTERLEAVED && (l.tile_rows <= 0 || l.tile_cols <= 0))
        return fail(RTNQ_E_INVALID_INPUT, "kernel tile dimensions must be positive");
    return RTNQ_OK;
}

// ---- host-API device plumbing ------------------------------------------------------
cudaStream_t host_stream() {
    static cudaStream_t s = [] {
        cudaStream_t t = nullptr;
        cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking);
        return t;
    }();
    return s;
}

struct Dev {
    void* p = nullptr;
    cudaError_t err = cudaSuccess;
    explicit Dev(size_t bytes) {
        if (bytes) err = cudaMallocAsync(&p, bytes, host_stream());
    }
    ~Dev() {
        if (p) cudaFreeAsync(p, host_stream());
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

#define RTNQ_ALLOC(name, bytes)                                                  \
    Dev name{bytes};                                                             \
    if (name.err != cudaSuccess)                                                 \
        return fail(RTNQ_E_CUDA, std::string("device allocation: ") +            \
                                     cudaGetErrorString(name.err))

rtnq_status h2d(void* d, const void* h, size_t n) {
    if (n) RTNQ_CUDA(cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, host_stream()));
    return RTNQ_OK;
}
rtnq_status d2h(void* h, const void* d, size_t n) {
    if (n) RTNQ_CUDA(cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, host_stream()));
    return RTNQ_OK;
}
rtnq_status sync_host() {
    RTNQ_CUDA(cudaGetLastError());
    RTNQ_CUDA(cudaStreamSynchronize(host_stream()));
    return RTNQ_OK;
}

#define RTNQ_TRY(expr)                   \
    do {                                 \
        rtnq_status s_ = (expr);         \
        if (s_ != RTNQ_OK) return s_;    \
    } while (0)

int64_t gpr_of(int64_t g, int64_t cols) { return g >= cols ? 1 : (cols + g - 1) / g; }

}  // namespace

extern "C" {

int rtnq_version(void) { return RTNQ_CAPI_VERSION; }
const char* rtnq_last_error(void) { return g_err.c_str(); }

rtnq_status rtnq_device_info(int* sm_count, int* cc_major, int* cc_minor) {
    int dev = 0;
    RTNQ_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp p;
    RTNQ_CUDA(cudaGetDeviceProperties(&p, dev));
    if (sm_count) *sm_count = p.multiProcessorCount;
    if (cc_major) *cc_major = p.major;
    if (cc_minor) *cc_minor = p.minor;
    return RTNQ_OK;
}

// ---- geometry ------------------------------------------------------------------------

int64_t rtnq_groups_per_row(int64_t g, int ragged, int64_t cols) {
    if (g <= 0 || (g & (g - 1)) != 0) {
        fail(RTNQ_E_INVALID_INPUT, "group size must be a positive power of two");
        return -RTNQ_E_INVALID_INPUT;
    }
    if (cols % g != 0 && !ragged) {
        fail(RTNQ_E_SHAPE, "row length " + std::to_string(cols) +
                               " is not a multiple of group size " + std::to_string(g) +
                               " (ragged groups are disabled)");
        return -RTNQ_E_SHAPE;
    }
    return (cols + g - 1) / g;
}

int64_t rtnq_layout_slots(rtnq_layout l, int bits, int64_t rows, int64_t cols) {
    if (check_layout(l) != RTNQ_OK) return -RTNQ_E_INVALID_INPUT;
    return layout_slots_of(to_layout(l), bits, rows, cols);
}

int64_t rtnq_layout_bytes(rtnq_layout l, int bits, int64_t rows, int64_t cols) {
    const int64_t s = rtnq_layout_slots(l, bits, rows, cols);
    return s < 0 ? s : (s * bits + 7) / 8;
}

int64_t rtnq_layout_index(rtnq_layout l, int bits, int64_t rows, int64_t cols, int64_t r,
                          int64_t c) {
    if (r < 0 || r >= rows || c < 0 || c >= cols) {
        fail(RTNQ_E_SHAPE, "layout index out of bounds");
        return -RTNQ_E_SHAPE;
    }
    if (check_layout(l) != RTNQ_OK) return -RTNQ_E_INVALID_INPUT;
    return layout_slot(to_layout(l), bits, rows, cols, r, c);
}

int64_t rtnq_native_scale_count(int64_t rows, int64_t gpr) { return gpr * ((rows + 7) / 8 * 8); }

// ---- device API ----------------------------------------------------------------------

size_t rtnq_dev_quantize_workspace_bytes(int64_t rows, int64_t cols, int bits, int64_t g,
                                         int ragged) {
    (void)ragged;
    if (quant_fused_supported(rows, cols, bits, g)) return 0;
    const int64_t gpr = gpr_of(g, cols);
    // logical int8 codes + f32 scales (when the caller does not want them)
    return size_t(rows * cols + 15) / 16 * 16 + size_t(rows * gpr) * sizeof(float);
}

rtnq_status rtnq_dev_quantize_pack(const void* w, int w_dtype, int64_t rows, int64_t cols,
                                   int bits, int64_t g, int ragged, uint8_t* rm, uint8_t* k164,
                                   uint8_t* nat, float* s32, uint16_t* s16, uint16_t* s16n,
                                   int32_t* err, void* ws, size_t ws_bytes, void* stream) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    if (rows < 0 || cols < 0) return fail(RTNQ_E_SHAPE, "negative tensor dimension");
    const int64_t gpr = rtnq_groups_per_row(g, ragged, cols);
    if (gpr < 0) return rtnq_status(-gpr);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (rows * cols == 0) return RTNQ_OK;
    if (s16n)  // padded rows of the native scale order are zero
        RTNQ_CUDA(cudaMemsetAsync(s16n, 0, size_t(rtnq_native_scale_count(rows, gpr)) * 2, st));
    if (quant_fused_supported(rows, cols, bits, g)) {
        launch_quant_fused(w, w_dtype, rows, cols, bits, g, rm, k164, nat, s32, s16, s16n, err,
                           st);
        RTNQ_CUDA(cudaGetLastError());
        return RTNQ_OK;
    }
    const size_t need = rtnq_dev_quantize_workspace_bytes(rows, cols, bits, g, ragged);
    if (!ws || ws_bytes < need)
        return fail(RTNQ_E_INVALID_INPUT, "quantize workspace too small: need " +
                                              std::to_string(need) + " bytes");
    int8_t* logical = static_cast<int8_t*>(ws);
    float* sc = s32 ? s32
                    : reinterpret_cast<float*>(static_cast<char*>(ws) +
                                               size_t(rows * cols + 15) / 16 * 16);
    launch_group_scales(w, w_dtype, rows, cols, bits, g, gpr, sc, s16, s16n, err, st);
    launch_codes(w, w_dtype, rows, cols, bits, g, gpr, sc, logical, st);
    if (rm) launch_encode_from_logical(logical, Layout{RTNQ_ROW_MAJOR, 16, 4}, bits, rows, cols, rm, st);
    if (k164)
        launch_encode_from_logical(logical, Layout{RTNQ_KERNEL_INTERLEAVED, 16, 4}, bits, rows,
                                   cols, k164, st);
    if (nat) launch_encode_from_logical(logical, Layout{RTNQ_NATIVE_SM100, 16, 4}, bits, rows, cols, nat, st);
    RTNQ_CUDA(cudaGetLastError());
    return RTNQ_OK;
}

size_t rtnq_dev_quantize_workspace_bytes_ex(int64_t rows, int64_t cols, int bits, int64_t g,
                                            int ragged, int native_kind) {
    const size_t base = rtnq_dev_quantize_workspace_bytes(rows, cols, bits, g, ragged);
    if (native_kind != RTNQ_NATIVE_I4 && native_kind != RTNQ_NATIVE_I8) return base;
    // the general route quantizes into row-major bytes first, then relays them out
    return base + (size_t(rows * cols * bits / 8) + 255) / 256 * 256;
}

rtnq_status rtnq_dev_quantize_pack_ex(const void* w, int w_dtype, int64_t rows, int64_t cols,
                                      int bits, int64_t g, int ragged, int native_kind,
                                      uint8_t* rm, uint8_t* k164, uint8_t* nat, float* s32,
                                      uint16_t* s16, uint16_t* s16n, int32_t* err, void* ws,
                                      size_t ws_bytes, void* stream) {
    if (native_kind == RTNQ_NATIVE_SM100)
        return rtnq_dev_quantize_pack(w, w_dtype, rows, cols, bits, g, ragged, rm, k164, nat, s32,
                                      s16, s16n, err, ws, ws_bytes, stream);
    if (native_kind != RTNQ_NATIVE_I4 && native_kind != RTNQ_NATIVE_I8)
        return fail(RTNQ_E_INVALID_INPUT, "native_kind must be RTNQ_NATIVE_SM100, _I4 or _I8");
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    if (rows < 0 || cols < 0) return fail(RTNQ_E_SHAPE, "negative tensor dimension");
    const int64_t gpr = rtnq_groups_per_row(g, ragged, cols);
    if (gpr < 0) return rtnq_status(-gpr);
    if (native_kind == RTNQ_NATIVE_I4 && (bits != 4 || g != 128))
        return fail(RTNQ_E_UNSUPPORTED, "RTNQ_NATIVE_I4 holds W4 group-128 codes");
    if (native_kind == RTNQ_NATIVE_I8 && (bits != 8 || (g < cols && g != 128)))
        return fail(RTNQ_E_UNSUPPORTED, "RTNQ_NATIVE_I8 holds W8 per-channel or group-128 codes");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (rows * cols == 0) return RTNQ_OK;
    if (s16n) RTNQ_CUDA(cudaMemsetAsync(s16n, 0, size_t(rtnq_native_scale_count(rows, gpr)) * 2, st));
    // one pass straight into the int8-MMA tiles
    if (!k164 && nat && native_kind == RTNQ_NATIVE_I4 && quant_i4_supported(rows, cols, bits, g)) {
        launch_quant_i4(w, w_dtype, rows, cols, nat, rm, s32, s16, s16n, err, st);
        RTNQ_CUDA(cudaGetLastError());
        return RTNQ_OK;
    }
    if (!k164 && nat && native_kind == RTNQ_NATIVE_I8 && quant_rowwise_supported(rows, cols, bits, g)) {
        launch_quant_rowwise(w, w_dtype, rows, cols, nat, rm, s32, s16, s16n, err, st);
        RTNQ_CUDA(cudaGetLastError());
        return RTNQ_OK;
    }
    // general route: the reference-layout kernels into row-major bytes, then a relayout
    const size_t need = rtnq_dev_quantize_workspace_bytes_ex(rows, cols, bits, g, ragged, native_kind);
    if (!ws || ws_bytes < need)
        return fail(RTNQ_E_INVALID_INPUT, "quantize workspace too small: need " + std::to_string(need) + " bytes");
    const size_t base = rtnq_dev_quantize_workspace_bytes(rows, cols, bits, g, ragged);
    uint8_t* rmb = rm ? rm : static_cast<uint8_t*>(ws) + base;
    // (the native scale order is the same for every native code layout)
    RTNQ_TRY(rtnq_dev_quantize_pack(w, w_dtype, rows, cols, bits, g, ragged, rmb, k164, nullptr, s32,
                                    s16, s16n, err, ws, base, stream));
    if (nat)
        launch_relayout(rmb, Layout{RTNQ_ROW_MAJOR, 16, 4}, nat, Layout{native_kind, 16, 4}, bits, rows, cols, st);
    RTNQ_CUDA(cudaGetLastError());
    return RTNQ_OK;
}

rtnq_status rtnq_dev_relayout(const uint8_t* src, rtnq_layout from, uint8_t* dst, rtnq_layout to,
                              int bits, int64_t rows, int64_t cols, void* stream) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    RTNQ_TRY(check_layout(from));
    RTNQ_TRY(check_layout(to));
    launch_relayout(src, to_layout(from), dst, to_layout(to), bits, rows, cols,
                    static_cast<cudaStream_t>(stream));
    RTNQ_CUDA(cudaGetLastError());
    return RTNQ_OK;
}

rtnq_status rtnq_dev_native_scales(const void* scales, int dtype, int64_t rows, int64_t gpr,
                                   uint16_t* out, void* stream) {
    launch_native_scales(scales, dtype, rows, gpr, out, static_cast<cudaStream_t>(stream));
    RTNQ_CUDA(cudaGetLastError());
    return RTNQ_OK;
}

rtnq_status rtnq_dev_dequantize(const uint8_t* codes, rtnq_layout layout, int bits, int64_t rows,
                                int64_t cols, int64_t g, const void* scales, int sdtype,
                                int sorder, void* out, int odtype, void* stream) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    RTNQ_TRY(check_layout(layout));
    if (g <= 0) return fail(RTNQ_E_INVALID_INPUT, "group size must be a positive power of two");
    launch_dequant(codes, to_layout(layout), bits, rows, cols, g, gpr_of(g, cols), scales, sdtype,
                   sorder, out, odtype, static_cast<cudaStream_t>(stream));
    RTNQ_CUDA(cudaGetLastError());
    return RTNQ_OK;
}

// W8 per-channel over the reference's row-major bytes: the int8 tensor-core kernel.
static bool i8_path(int a_dtype, rtnq_layout layout, int bits, int64_t g, int64_t k, int sdtype) {
    return layout.kind == RTNQ_NATIVE_I8 && bits == 8 && g >= k &&
           (a_dtype == RTNQ_BF16 || a_dtype == RTNQ_F16) && sdtype == RTNQ_F16;
}

// Group 128 (per-group accumulators, wgemm_i4.cu): W4 over RTNQ_NATIVE_I4 nibble tiles or W8 over
// RTNQ_NATIVE_I8 tiles, on the int8 tensor-core kernel.
static bool i4_path(int a_dtype, rtnq_layout layout, int bits, int64_t g, int sdtype, int sorder) {
    return ((layout.kind == RTNQ_NATIVE_I4 && bits == 4) || (layout.kind == RTNQ_NATIVE_I8 && bits == 8)) && g == 128 &&
           (a_dtype == RTNQ_BF16 || a_dtype == RTNQ_F16) && sdtype == RTNQ_F16 &&
           sorder == RTNQ_SCALES_NATIVE;
}

// The first 64 KiB of a linear workspace hold the fused kernels' per-row-block counters, which
// must stay zero between launches; the dequant-first paths put their scratch after them.
constexpr size_t kCountersReserve = 64 * 1024;

static bool tensor_path(int a_dtype, rtnq_layout layout, int sdtype, int sorder) {
    return layout.kind == RTNQ_NATIVE_SM100 && (a_dtype == RTNQ_BF16 || a_dtype == RTNQ_F16) &&
           sdtype == RTNQ_F16 && sorder == RTNQ_SCALES_NATIVE;
}

size_t rtnq_dev_linear_workspace_bytes(int64_t m, int64_t n, int64_t k, int bits, int64_t g,
                                       int path, rtnq_layout layout) {
    size_t ws = 0;
    if (path == RTNQ_PATH_FUSED || path == RTNQ_PATH_AUTO) {
        if (layout.kind == RTNQ_NATIVE_SM100) ws = wgemm_workspace_bytes(m, n, k, bits, g);
        if (layout.kind == RTNQ_NATIVE_I8 && bits == 8 && g >= k) ws = wgemm_i8_workspace_bytes(m, n, k);
        if ((layout.kind == RTNQ_NATIVE_I4 && bits == 4 || layout.kind == RTNQ_NATIVE_I8 && bits == 8 && g < k) &&
            g == 128)
            ws = wgemm_i4_workspace_bytes(m, n, k);
    }
    if (path == RTNQ_PATH_DEQUANT_FIRST || path == RTNQ_PATH_AUTO) {
        // f32 reference-exact materialization, or the tensor-core hi/lo split (+ f32 C), after
        // the fused kernels' self-resetting counters (never overwritten)
        size_t d = size_t(n) * size_t(k) * sizeof(float);
        const size_t t = dequant_first_workspace_bytes(m, n, k, RTNQ_BF16);
        d = (d > t ? d : t) + kCountersReserve;
        ws = ws > d ? ws : d;
    }
    return ws;
}

rtnq_status rtnq_dev_linear(const void* a, int a_dtype, int64_t m, int64_t k,
                            const uint8_t* codes, rtnq_layout layout, int bits, int64_t n,
                            int64_t g, int ragged, const void* scales, int sdtype, int sorder,
                            void* out, int odtype, int path, int64_t threshold, int* chosen,
                            int32_t* err, void* ws, size_t ws_bytes, void* stream) {
    return rtnq_dev_linear_ex(a, a_dtype, m, k, codes, layout, bits, n, g, ragged, scales, sdtype,
                              sorder, out, odtype, path, threshold, chosen, err, ws, ws_bytes,
                              stream, 0u);
}

rtnq_status rtnq_dev_linear_ex(const void* a, int a_dtype, int64_t m, int64_t k,
                               const uint8_t* codes, rtnq_layout layout, int bits, int64_t n,
                               int64_t g, int ragged, const void* scales, int sdtype, int sorder,
                               void* out, int odtype, int path, int64_t threshold, int* chosen,
                               int32_t* err, void* ws, size_t ws_bytes, void* stream,
                               unsigned flags) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    RTNQ_TRY(check_layout(layout));
    if (m < 0 || n < 0 || k < 0) return fail(RTNQ_E_SHAPE, "negative tensor dimension");
    const int64_t gpr = rtnq_groups_per_row(g, ragged, k);
    if (gpr < 0) return rtnq_status(-gpr);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (path == RTNQ_PATH_AUTO) {
        if (threshold < 1) return fail(RTNQ_E_INVALID_INPUT, "dispatch threshold must be >= 1");
        path = m >= threshold ? RTNQ_PATH_DEQUANT_FIRST : RTNQ_PATH_FUSED;
    }
    if (chosen) *chosen = path;
    const Layout L = to_layout(layout);
    // the int8 kernels check the activations in their planes pass; every other path runs a
    // separate finiteness pass (InvalidInputError, gemm.cpp:13-19)
    const bool planes_check = path == RTNQ_PATH_FUSED && n > 0 &&
                              (i8_path(a_dtype, layout, bits, g, k, sdtype) ||
                               i4_path(a_dtype, layout, bits, g, sdtype, sorder));
    if (err && m * k && !planes_check) launch_check_finite(a, a_dtype, m * k, err, st);
    if (m * n == 0) return RTNQ_OK;
    if (path == RTNQ_PATH_FUSED && tensor_path(a_dtype, layout, sdtype, sorder)) {
        if (const char* why = wgemm_unsupported(m, n, k, bits, g, a_dtype))
            return fail(RTNQ_E_UNSUPPORTED, why);
        const size_t need = wgemm_workspace_bytes(m, n, k, bits, g);
        if (ws_bytes < need)
            return fail(RTNQ_E_INVALID_INPUT, "linear workspace too small: need " +
                                                  std::to_string(need) + " bytes");
        if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(codes) |
             reinterpret_cast<uintptr_t>(scales)) & 15)
            return fail(RTNQ_E_INVALID_INPUT, "tensor-core path needs 16-byte aligned operands");
        WgemmArgs A{a, a_dtype, m, n, k, codes, static_cast<const uint16_t*>(scales), bits, g,
                    out, odtype, ws, ws_bytes, (flags & RTNQ_FLAG_PDL) != 0};
        RTNQ_CUDA(launch_wgemm(A, st));
        return RTNQ_OK;
    }
    if (path == RTNQ_PATH_FUSED && i8_path(a_dtype, layout, bits, g, k, sdtype)) {
        if (const char* why = wgemm_i8_unsupported(m, n, k, bits, g, a_dtype))
            return fail(RTNQ_E_UNSUPPORTED, why);
        const size_t need = wgemm_i8_workspace_bytes(m, n, k);
        if (ws_bytes < need)
            return fail(RTNQ_E_INVALID_INPUT, "linear workspace too small: need " +
                                                  std::to_string(need) + " bytes");
        if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(codes) |
             reinterpret_cast<uintptr_t>(scales)) & 15)
            return fail(RTNQ_E_INVALID_INPUT, "tensor-core path needs 16-byte aligned operands");
        WgemmArgs A{a, a_dtype, m, n, k, codes, static_cast<const uint16_t*>(scales), bits, g,
                    out, odtype, ws, ws_bytes, (flags & RTNQ_FLAG_PDL) != 0};
        A.err = err;
        RTNQ_CUDA(launch_wgemm_i8(A, st));
        return RTNQ_OK;
    }
    if (path == RTNQ_PATH_FUSED && i4_path(a_dtype, layout, bits, g, sdtype, sorder)) {
        if (const char* why = wgemm_i4_unsupported(m, n, k, bits, g, a_dtype))
            return fail(RTNQ_E_UNSUPPORTED, why);
        const size_t need = wgemm_i4_workspace_bytes(m, n, k);
        if (ws_bytes < need)
            return fail(RTNQ_E_INVALID_INPUT, "linear workspace too small: need " +
                                                  std::to_string(need) + " bytes");
        if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(codes) |
             reinterpret_cast<uintptr_t>(scales)) & 15)
            return fail(RTNQ_E_INVALID_INPUT, "tensor-core path needs 16-byte aligned operands");
        WgemmArgs A{a, a_dtype, m, n, k, codes, static_cast<const uint16_t*>(scales), bits, g,
                    out, odtype, ws, ws_bytes, (flags & RTNQ_FLAG_PDL) != 0};
        A.err = err;
        RTNQ_CUDA(launch_wgemm_i4(A, st));
        return RTNQ_OK;
    }
    // Dequant-first on the tensor cores: 16-bit activations, f16 scales, any
    // codes layout; exact hi + lo weight split, two cuBLAS GEMMs with f32 accumulation.
    if (path == RTNQ_PATH_DEQUANT_FIRST && (a_dtype == RTNQ_BF16 || a_dtype == RTNQ_F16) &&
        sdtype == RTNQ_F16) {
        const size_t need = dequant_first_workspace_bytes(m, n, k, odtype) + kCountersReserve;
        if (ws_bytes < need)
            return fail(RTNQ_E_INVALID_INPUT, "linear workspace too small: need " +
                                                  std::to_string(need) + " bytes");
        if (const char* why = launch_dequant_first(a, a_dtype, m, n, k, codes, L, bits, g, gpr,
                                                   static_cast<const uint16_t*>(scales), sorder, out,
                                                   odtype, static_cast<char*>(ws) + kCountersReserve, st))
            return fail(RTNQ_E_CUDA, why);
        return RTNQ_OK;
    }
    // Reference-exact CUDA-core paths: f32 activations, f32 reference-order scales.
    if (a_dtype != RTNQ_F32 || odtype != RTNQ_F32 || sdtype != RTNQ_F32 ||
        sorder != RTNQ_SCALES_REF)
        return fail(RTNQ_E_UNSUPPORTED,
                    "this path needs f32 activations/outputs and f32 reference-order scales "
                    "(tensor-core path: native layout, bf16/f16 activations, native f16 scales)");
    const float* af = static_cast<const float*>(a);
    const float* sf = static_cast<const float*>(scales);
    float* of = static_cast<float*>(out);
    if (path == RTNQ_PATH_FUSED) {
        launch_gemm_fused_exact(af, m, k, codes, L, bits, n, g, gpr, sf, of, st);
    } else if (path == RTNQ_PATH_DEQUANT_FIRST) {
        const size_t need = size_t(n) * size_t(k) * sizeof(float) + kCountersReserve;
        if (ws_bytes < need) return fail(RTNQ_E_INVALID_INPUT, "linear workspace too small");
        float* wf = reinterpret_cast<float*>(static_cast<char*>(ws) + kCountersReserve);
        launch_dequant(codes, L, bits, n, k, g, gpr, sf, RTNQ_F32, RTNQ_SCALES_REF, wf, RTNQ_F32, st);
        launch_dense_blocked(af, m, k, wf, n, g, of, st);
    } else if (path == RTNQ_PATH_ORACLE) {
        launch_gemm_oracle(af, m, k, codes, L, bits, n, g, gpr, sf, of, st);
    } else {
        return fail(RTNQ_E_INVALID_INPUT, "unknown GEMM path");
    }
    RTNQ_CUDA(cudaGetLastError());
    return RTNQ_OK;
}

rtnq_status rtnq_dev_gemm_float(const float* a, int64_t m, int64_t k, const float* w, int64_t n,
                                int64_t block, float* out, void* stream) {
    if (block < 1) return fail(RTNQ_E_INVALID_INPUT, "accumulation block must be >= 1");
    launch_dense_blocked(a, m, k, w, n, block, out, static_cast<cudaStream_t>(stream));
    RTNQ_CUDA(cudaGetLastError());
    return RTNQ_OK;
}

// ---- decode-layer kernels (decode.cu) ------------------------------------------------

rtnq_status rtnq_dev_add_rmsnorm(void* x, const void* delta, const void* weight, void* out,
                                 int64_t m, int64_t h, float eps, void* stream) {
    if (m < 0 || h <= 0 || h % 8) return fail(RTNQ_E_SHAPE, "rmsnorm needs h % 8 == 0");
    if (m == 0) return RTNQ_OK;
    RTNQ_CUDA(launch_add_rmsnorm(x, delta, weight, out, m, h, eps, static_cast<cudaStream_t>(stream)));
    return RTNQ_OK;
}

rtnq_status rtnq_dev_add_rmsnorm_planes(void* x, const void* delta, const void* weight, void* out,
                                        int64_t m, int64_t h, float eps, int8_t* planes, int32_t* texp,
                                        void* stream) {
    if (m < 0 || h <= 0 || h % 16) return fail(RTNQ_E_SHAPE, "rmsnorm with planes needs h % 16 == 0");
    if (!planes || !texp) return fail(RTNQ_E_INVALID_INPUT, "planes and texp are required");
    if (m == 0) return RTNQ_OK;
    RTNQ_CUDA(launch_add_rmsnorm(x, delta, weight, out, m, h, eps, static_cast<cudaStream_t>(stream), planes,
                                 texp));
    return RTNQ_OK;
}

rtnq_status rtnq_dev_silu_mul_planes(const void* gate_up, void* act, int64_t m, int64_t f, int8_t* planes,
                                     int32_t* texp, void* stream) {
    if (m < 0 || f <= 0 || f % 16) return fail(RTNQ_E_SHAPE, "silu_mul with planes needs f % 16 == 0");
    if (!planes || !texp) return fail(RTNQ_E_INVALID_INPUT, "planes and texp are required");
    if (m == 0) return RTNQ_OK;
    RTNQ_CUDA(launch_silu_mul(gate_up, act, m, f, static_cast<cudaStream_t>(stream), planes, texp));
    return RTNQ_OK;
}

rtnq_status rtnq_dev_act_planes(const void* a, int a_dtype, int64_t m, int64_t k, int8_t* planes,
                                int32_t* texp, void* stream) {
    if (a_dtype != RTNQ_BF16 && a_dtype != RTNQ_F16) return fail(RTNQ_E_INVALID_INPUT, "bf16/f16 activations");
    if (m < 0 || k <= 0 || k % 16) return fail(RTNQ_E_SHAPE, "activation planes need k % 16 == 0");
    if (m == 0) return RTNQ_OK;
    RTNQ_CUDA(launch_act_planes(a, a_dtype, m, k, planes, texp, static_cast<cudaStream_t>(stream)));
    return RTNQ_OK;
}

rtnq_status rtnq_dev_linear_planes(const int8_t* planes, const int32_t* texp, int64_t m, int64_t k,
                                   const uint8_t* codes, rtnq_layout layout, int bits, int64_t n, int64_t g,
                                   int ragged, const void* scales, int sdtype, int sorder, void* out,
                                   int odtype, void* ws, size_t ws_bytes, void* stream, unsigned flags) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    RTNQ_TRY(check_layout(layout));
    if (m < 0 || n < 0 || k < 0) return fail(RTNQ_E_SHAPE, "negative tensor dimension");
    const int64_t gpr = rtnq_groups_per_row(g, ragged, k);
    if (gpr < 0) return rtnq_status(-gpr);
    if (!planes || !texp) return fail(RTNQ_E_INVALID_INPUT, "planes and texp are required");
    if (m * n == 0) return RTNQ_OK;
    const bool i8 = i8_path(RTNQ_BF16, layout, bits, g, k, sdtype);
    const bool i4 = i4_path(RTNQ_BF16, layout, bits, g, sdtype, sorder);
    if (!i8 && !i4)
        return fail(RTNQ_E_UNSUPPORTED, "precomputed planes feed the int8 kernels: RTNQ_NATIVE_I4 (W4 g128) or "
                                        "RTNQ_NATIVE_I8 (W8 per-channel) codes, native f16 scales");
    if (const char* why = i8 ? wgemm_i8_unsupported(m, n, k, bits, g, RTNQ_BF16)
                             : wgemm_i4_unsupported(m, n, k, bits, g, RTNQ_BF16))
        return fail(RTNQ_E_UNSUPPORTED, why);
    const size_t need = i8 ? wgemm_i8_workspace_bytes(m, n, k) : wgemm_i4_workspace_bytes(m, n, k);
    if (ws_bytes < need)
        return fail(RTNQ_E_INVALID_INPUT, "linear workspace too small: need " + std::to_string(need) + " bytes");
    WgemmArgs A{nullptr, RTNQ_BF16, m, n, k, codes, static_cast<const uint16_t*>(scales), bits, g,
                out, odtype, ws, ws_bytes, (flags & RTNQ_FLAG_PDL) != 0};
    A.planes = planes;
    A.texp = texp;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    RTNQ_CUDA(i8 ? launch_wgemm_i8(A, st) : launch_wgemm_i4(A, st));
    return RTNQ_OK;
}

// ---- tensor-parallel partial sums over peer memory (int8_mma.cuh protocol) --------

size_t rtnq_peer_buffer_bytes(int64_t cap) { return cap < 0 ? 0 : peer_buffer_bytes(cap); }

rtnq_status rtnq_peer_alloc(int64_t cap, void** dev_ptr) {
    if (!dev_ptr || cap <= 0 || cap % 8) return fail(RTNQ_E_INVALID_INPUT, "cap must be a positive multiple of 8");
    // a dedicated allocation: an IPC handle maps a whole allocation, so the buffer must start one
    *dev_ptr = nullptr;
    RTNQ_CUDA(cudaMalloc(dev_ptr, peer_buffer_bytes(cap)));
    RTNQ_CUDA(cudaMemset(*dev_ptr, 0, peer_buffer_bytes(cap)));
    RTNQ_CUDA(cudaDeviceSynchronize());
    return RTNQ_OK;
}

rtnq_status rtnq_peer_free(void* dev_ptr) {
    RTNQ_CUDA(cudaFree(dev_ptr));
    return RTNQ_OK;
}

rtnq_status rtnq_ipc_get_handle(void* dev_ptr, void* handle) {
    if (!dev_ptr || !handle) return fail(RTNQ_E_INVALID_INPUT, "null pointer");
    static_assert(sizeof(cudaIpcMemHandle_t) == RTNQ_IPC_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    RTNQ_CUDA(cudaIpcGetMemHandle(&h, dev_ptr));
    std::memcpy(handle, &h, sizeof(h));
    return RTNQ_OK;
}

rtnq_status rtnq_ipc_open(const void* handle, void** dev_ptr) {
    if (!dev_ptr || !handle) return fail(RTNQ_E_INVALID_INPUT, "null pointer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    RTNQ_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return RTNQ_OK;
}

rtnq_status rtnq_ipc_close(void* dev_ptr) {
    RTNQ_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return RTNQ_OK;
}

rtnq_status rtnq_peer_enable(int device, int peer) {
    if (device == peer) return RTNQ_OK;
    int can = 0;
    RTNQ_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
    if (!can) return fail(RTNQ_E_UNSUPPORTED, "no peer access between the two devices");
    int cur = 0;
    RTNQ_CUDA(cudaGetDevice(&cur));
    RTNQ_CUDA(cudaSetDevice(device));
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError(), e = cudaSuccess;
    cudaSetDevice(cur);
    RTNQ_CUDA(e);
    return RTNQ_OK;
}

static rtnq_status peer_in(void* buf, int world, int64_t cap, PeerIn* pin) {
    if (!buf) return fail(RTNQ_E_INVALID_INPUT, "null peer buffer");
    if (world < 1 || world > kPeerMax) return fail(RTNQ_E_INVALID_INPUT, "peer world must be 1..8");
    if (cap <= 0 || cap % 8 || (reinterpret_cast<uintptr_t>(buf) & 255))
        return fail(RTNQ_E_INVALID_INPUT, "peer slot capacity must be a positive multiple of 8 elements, the "
                                          "buffer 256-byte aligned");
    pin->buf = static_cast<char*>(buf);
    pin->world = world;
    pin->cap = cap;
    return RTNQ_OK;
}

rtnq_status rtnq_dev_linear_peer(const void* a, const int8_t* planes, const int32_t* texp, int64_t m, int64_t k,
                                 const uint8_t* codes, rtnq_layout layout, int bits, int64_t n, int64_t g,
                                 int ragged, const void* scales, int sdtype, int sorder, void* const* peer_bufs,
                                 int world, int rank, int64_t cap, int32_t* err, void* ws, size_t ws_bytes,
                                 void* stream, unsigned flags) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    RTNQ_TRY(check_layout(layout));
    if (m <= 0 || n <= 0 || k <= 0) return fail(RTNQ_E_SHAPE, "peer linear needs a non-empty output");
    const int64_t gpr = rtnq_groups_per_row(g, ragged, k);
    if (gpr < 0) return rtnq_status(-gpr);
    if (!a == !planes || (planes && !texp))
        return fail(RTNQ_E_INVALID_INPUT, "give either bf16 activations or their planes + exponents");
    if (!peer_bufs || rank < 0 || rank >= world) return fail(RTNQ_E_INVALID_INPUT, "rank outside the world");
    PeerIn own;
    RTNQ_TRY(peer_in(peer_bufs[rank], world, cap, &own));
    PeerOut po;
    po.world = world;
    po.rank = rank;
    po.cap = cap;
    for (int q = 0; q < world; ++q) {
        if (!peer_bufs[q] || (reinterpret_cast<uintptr_t>(peer_bufs[q]) & 255))
            return fail(RTNQ_E_INVALID_INPUT, "null or unaligned peer buffer");
        po.bufs[q] = static_cast<char*>(peer_bufs[q]);
    }
    if (m * n > cap) return fail(RTNQ_E_INVALID_INPUT, "output larger than the peer slot");
    const bool i8 = i8_path(RTNQ_BF16, layout, bits, g, k, sdtype);
    const bool i4 = i4_path(RTNQ_BF16, layout, bits, g, sdtype, sorder);
    if (!i8 && !i4)
        return fail(RTNQ_E_UNSUPPORTED, "peer output comes from the int8 kernels: RTNQ_NATIVE_I4 (W4 g128) or "
                                        "RTNQ_NATIVE_I8 codes, native f16 scales");
    if (m > 64) return fail(RTNQ_E_UNSUPPORTED, "peer output: at most 64 tokens per launch");
    if (const char* why = i8 ? wgemm_i8_unsupported(m, n, k, bits, g, RTNQ_BF16)
                             : wgemm_i4_unsupported(m, n, k, bits, g, RTNQ_BF16))
        return fail(RTNQ_E_UNSUPPORTED, why);
    const size_t need = i8 ? wgemm_i8_workspace_bytes(m, n, k) : wgemm_i4_workspace_bytes(m, n, k);
    if (ws_bytes < need)
        return fail(RTNQ_E_INVALID_INPUT, "linear workspace too small: need " + std::to_string(need) + " bytes");
    if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(codes) | reinterpret_cast<uintptr_t>(scales)) & 15)
        return fail(RTNQ_E_INVALID_INPUT, "tensor-core path needs 16-byte aligned operands");
    WgemmArgs A{a, RTNQ_BF16, m, n, k, codes, static_cast<const uint16_t*>(scales), bits, g,
                nullptr, RTNQ_BF16, ws, ws_bytes, (flags & RTNQ_FLAG_PDL) != 0};
    A.planes = planes;
    A.texp = texp;
    A.err = err;
    A.peer = po;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    RTNQ_CUDA(i8 ? launch_wgemm_i8(A, st) : launch_wgemm_i4(A, st));
    return RTNQ_OK;
}

rtnq_status rtnq_dev_add_rmsnorm_peer(void* x, void* peer_buf, int world, int64_t cap, const void* weight,
                                      void* out, int64_t m, int64_t h, float eps, int8_t* planes, int32_t* texp,
                                      void* stream) {
    if (m <= 0 || h <= 0 || h % 16 || h / 8 > 32 * 256)
        return fail(RTNQ_E_SHAPE, "peer rmsnorm needs h % 16 == 0, h <= 65536 and m > 0");
    if (!planes != !texp) return fail(RTNQ_E_INVALID_INPUT, "planes and texp go together");
    PeerIn pin;
    RTNQ_TRY(peer_in(peer_buf, world, cap, &pin));
    if (m * h > cap) return fail(RTNQ_E_INVALID_INPUT, "rows larger than the peer slot");
    RTNQ_CUDA(launch_add_rmsnorm(x, nullptr, weight, out, m, h, eps, static_cast<cudaStream_t>(stream), planes,
                                 texp, pin));
    return RTNQ_OK;
}

rtnq_status rtnq_dev_peer_reduce(void* peer_buf, int world, int64_t cap, void* out, int64_t n, int accumulate,
                                 void* stream) {
    PeerIn pin;
    RTNQ_TRY(peer_in(peer_buf, world, cap, &pin));
    if (n <= 0 || n % 8 || n > cap) return fail(RTNQ_E_SHAPE, "reduce length must be a positive multiple of 8 "
                                                              "within the slot");
    if (reinterpret_cast<uintptr_t>(out) & 15) return fail(RTNQ_E_INVALID_INPUT, "out must be 16-byte aligned");
    RTNQ_CUDA(launch_peer_reduce(pin, out, n, accumulate != 0, static_cast<cudaStream_t>(stream)));
    return RTNQ_OK;
}

rtnq_status rtnq_dev_silu_mul(const void* gate_up, void* act, int64_t m, int64_t f, void* stream) {
    if (m < 0 || f <= 0 || f % 8) return fail(RTNQ_E_SHAPE, "silu_mul needs f % 8 == 0");
    if (m == 0) return RTNQ_OK;
    RTNQ_CUDA(launch_silu_mul(gate_up, act, m, f, static_cast<cudaStream_t>(stream)));
    return RTNQ_OK;
}

rtnq_status rtnq_dev_decode_attention(const void* qkv, void* k_cache, void* v_cache, void* out,
                                      int64_t batch, int64_t hq, int64_t hkv, int64_t head_dim,
                                      int64_t max_len, int64_t pos, float rope_theta,
                                      void* stream) {
    if (head_dim != 128) return fail(RTNQ_E_UNSUPPORTED, "decode attention needs head_dim 128");
    if (hkv <= 0 || hq % hkv || hq / hkv > 32)
        return fail(RTNQ_E_SHAPE, "query heads must be a multiple (<= 32x) of kv heads");
    if (pos < 0 || pos >= max_len) return fail(RTNQ_E_INVALID_INPUT, "position outside the cache");
    if (batch == 0) return RTNQ_OK;
    RTNQ_CUDA(launch_decode_attention(qkv, k_cache, v_cache, out, batch, hq, hkv, head_dim, max_len,
                                      pos, rope_theta, static_cast<cudaStream_t>(stream)));
    return RTNQ_OK;
}

size_t rtnq_dev_decode_attention_workspace_bytes(int64_t batch, int64_t hq, int64_t hkv, int64_t max_len) {
    return decode_attention_workspace_bytes(batch, hq, hkv, max_len);
}

rtnq_status rtnq_dev_decode_attention_ws(const void* qkv, void* k_cache, void* v_cache, void* out,
                                         int64_t batch, int64_t hq, int64_t hkv, int64_t head_dim,
                                         int64_t max_len, int64_t pos, float rope_theta, void* ws,
                                         size_t ws_bytes, void* stream) {
    return rtnq_dev_decode_attention_planes(qkv, k_cache, v_cache, out, batch, hq, hkv, head_dim, max_len, pos,
                                            rope_theta, nullptr, nullptr, ws, ws_bytes, stream);
}

rtnq_status rtnq_dev_decode_attention_planes(const void* qkv, void* k_cache, void* v_cache, void* out,
                                             int64_t batch, int64_t hq, int64_t hkv, int64_t head_dim,
                                             int64_t max_len, int64_t pos, float rope_theta, int8_t* planes,
                                             int32_t* texp, void* ws, size_t ws_bytes, void* stream) {
    if (head_dim != 128) return fail(RTNQ_E_UNSUPPORTED, "decode attention needs head_dim 128");
    if (hkv <= 0 || hq % hkv || hq / hkv > 32)
        return fail(RTNQ_E_SHAPE, "query heads must be a multiple (<= 32x) of kv heads");
    if (pos < 0 || pos >= max_len) return fail(RTNQ_E_INVALID_INPUT, "position outside the cache");
    if (!planes != !texp) return fail(RTNQ_E_INVALID_INPUT, "planes and texp go together");
    if (ws && ws_bytes < decode_attention_workspace_bytes(batch, hq, hkv, pos + 1))
        return fail(RTNQ_E_INVALID_INPUT, "decode attention workspace too small");
    if (batch == 0) return RTNQ_OK;
    RTNQ_CUDA(launch_decode_attention(qkv, k_cache, v_cache, out, batch, hq, hkv, head_dim, max_len, pos,
                                      rope_theta, static_cast<cudaStream_t>(stream), ws, ws_bytes, planes, texp));
    return RTNQ_OK;
}


rtnq_status rtnq_dev_check_flag(int32_t* err, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int32_t h = 0;
    RTNQ_CUDA(cudaMemcpyAsync(&h, err, sizeof(h), cudaMemcpyDeviceToHost, st));
    RTNQ_CUDA(cudaStreamSynchronize(st));
    if (h) {
        RTNQ_CUDA(cudaMemsetAsync(err, 0, sizeof(int32_t), st));
        return fail(RTNQ_E_INVALID_INPUT, "non-finite value");
    }
    return RTNQ_OK;
}

// ---- host API --------------------------------------------------------------------------

// The group-level entry points run the tensor kernels on a 1 x n "tensor" with
// one group spanning the row (g = n), exactly like compute_scale does.
rtnq_status rtnq_compute_scale(const float* v, int64_t n, int bits, float* out) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    if (n <= 0) return fail(RTNQ_E_INVALID_INPUT, "cannot compute a scale for an empty group");
    RTNQ_ALLOC(dv, size_t(n) * 4);
    RTNQ_ALLOC(ds, 4 + 4);
    RTNQ_TRY(h2d(dv.p, v, size_t(n) * 4));
    RTNQ_CUDA(cudaMemsetAsync(ds.p, 0, 8, host_stream()));
    int32_t* derr = reinterpret_cast<int32_t*>(ds.as<char>() + 4);
    launch_group_scales(dv.p, RTNQ_F32, 1, n, bits, n, 1, ds.as<float>(), nullptr, nullptr, derr,
                        host_stream());
    int32_t herr = 0;
    RTNQ_TRY(d2h(out, ds.p, 4));
    RTNQ_TRY(d2h(&herr, derr, 4));
    RTNQ_TRY(sync_host());
    if (herr) return fail(RTNQ_E_INVALID_INPUT, "non-finite value in quantization group");
    return RTNQ_OK;
}

rtnq_status rtnq_quantize_group(const float* v, int64_t n, int bits, const float* scale_in,
                                float* scale_out, int8_t* codes) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    float s = 0.0f;
    if (scale_in) {
        s = *scale_in;
    } else {
        RTNQ_TRY(rtnq_compute_scale(v, n, bits, &s));
    }
    if (scale_out) *scale_out = s;
    if (n <= 0) return RTNQ_OK;
    RTNQ_ALLOC(dv, size_t(n) * 4);
    RTNQ_ALLOC(ds, 4);
    RTNQ_ALLOC(dc, size_t(n));
    RTNQ_TRY(h2d(dv.p, v, size_t(n) * 4));
    RTNQ_TRY(h2d(ds.p, &s, 4));
    launch_codes(dv.p, RTNQ_F32, 1, n, bits, n, 1, ds.as<float>(), dc.as<int8_t>(), host_stream());
    RTNQ_TRY(d2h(codes, dc.p, size_t(n)));
    return sync_host();
}

rtnq_status rtnq_dequantize_group(const int8_t* codes, int64_t n, float scale, int bits,
                                  float* out) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    const int lo = -(1 << (bits - 1)), hi = (1 << (bits - 1)) - 1;
    for (int64_t i = 0; i < n; ++i)  // input validation, quant.cpp:88-92
        if (codes[i] < lo || codes[i] > hi)
            return fail(RTNQ_E_CORRUPT, "code " + std::to_string(int(codes[i])) + " outside the " +
                                            std::to_string(bits) + "-bit range");
    if (n <= 0) return RTNQ_OK;
    // upload the logical codes, pack them on the device (row-major), and run
    // the tensor dequantizer with one group spanning the row
    RTNQ_ALLOC(dc, size_t(n));
    RTNQ_ALLOC(dd, size_t((n * bits + 7) / 8));
    RTNQ_ALLOC(ds, 4);
    RTNQ_ALLOC(dout, size_t(n) * 4);
    RTNQ_TRY(h2d(dc.p, codes, size_t(n)));
    RTNQ_TRY(h2d(ds.p, &scale, 4));
    const Layout rm{RTNQ_ROW_MAJOR, 16, 4};
    launch_encode_from_logical(dc.as<int8_t>(), rm, bits, 1, n, dd.as<uint8_t>(), host_stream());
    launch_dequant(dd.as<uint8_t>(), rm, bits, 1, n, n, 1, ds.p, RTNQ_F32, RTNQ_SCALES_REF,
                   dout.p, RTNQ_F32, host_stream());
    RTNQ_TRY(d2h(out, dout.p, size_t(n) * 4));
    return sync_host();
}

rtnq_status rtnq_quantize_tensor(const float* w, int64_t rows, int64_t cols, int bits, int64_t g,
                                 int ragged, uint8_t* data, float* scales) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    const int64_t gpr = rtnq_groups_per_row(g, ragged, cols);  // quant.cpp:103
    if (gpr < 0) return rtnq_status(-gpr);
    if (rows * cols == 0) return RTNQ_OK;
    const size_t nbytes = size_t((rows * cols * bits + 7) / 8);
    const size_t wsb = rtnq_dev_quantize_workspace_bytes(rows, cols, bits, g, ragged);
    RTNQ_ALLOC(dw, size_t(rows * cols) * 4);
    RTNQ_ALLOC(dd, nbytes);
    RTNQ_ALLOC(ds, size_t(rows * gpr) * 4 + 4);
    RTNQ_ALLOC(dws, wsb);
    int32_t* derr = reinterpret_cast<int32_t*>(ds.as<char>() + size_t(rows * gpr) * 4);
    RTNQ_CUDA(cudaMemsetAsync(derr, 0, 4, host_stream()));
    RTNQ_TRY(h2d(dw.p, w, size_t(rows * cols) * 4));
    RTNQ_TRY(rtnq_dev_quantize_pack(dw.p, RTNQ_F32, rows, cols, bits, g, ragged, dd.as<uint8_t>(),
                                    nullptr, nullptr, ds.as<float>(), nullptr, nullptr, derr,
                                    dws.p, wsb, host_stream()));
    int32_t herr = 0;
    RTNQ_TRY(d2h(&herr, derr, 4));
    RTNQ_TRY(d2h(data, dd.p, nbytes));
    RTNQ_TRY(d2h(scales, ds.p, size_t(rows * gpr) * 4));
    RTNQ_TRY(sync_host());
    if (herr) return fail(RTNQ_E_INVALID_INPUT, "non-finite value in quantization group");
    return RTNQ_OK;
}

void rtnq_internal_set_error(const char* msg) { g_err = msg ? msg : ""; }

rtnq_status rtnq_pack(const int8_t* codes, int64_t n, int bits, uint8_t* out) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    const int lo = -(1 << (bits - 1)), hi = (1 << (bits - 1)) - 1;
    for (int64_t i = 0; i < n; ++i)  // input validation, packing.cpp:7-12
        if (codes[i] < lo || codes[i] > hi)
            return fail(RTNQ_E_INVALID_INPUT, "code " + std::to_string(int(codes[i])) +
                                                  " outside the " + std::to_string(bits) +
                                                  "-bit range");
    if (n <= 0) return RTNQ_OK;
    const size_t nbytes = size_t((n * bits + 7) / 8);
    RTNQ_ALLOC(dc, size_t(n));
    RTNQ_ALLOC(dd, nbytes);
    RTNQ_TRY(h2d(dc.p, codes, size_t(n)));
    launch_encode_from_logical(dc.as<int8_t>(), Layout{RTNQ_ROW_MAJOR, 16, 4}, bits, 1, n,
                               dd.as<uint8_t>(), host_stream());
    RTNQ_TRY(d2h(out, dd.p, nbytes));
    return sync_host();
}

rtnq_status rtnq_unpack(const uint8_t* bytes, int64_t nbytes, int64_t n, int bits, int8_t* out) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    const int64_t want = (n * bits + 7) / 8;
    if (n < 0 || nbytes != want)  // packing.cpp:35-41
        return fail(RTNQ_E_CORRUPT, "packed buffer is " + std::to_string(nbytes) +
                                        " bytes; expected " + std::to_string(want) + " for " +
                                        std::to_string(n) + " codes at " + std::to_string(bits) +
                                        " bits");
    if (n == 0) return RTNQ_OK;
    RTNQ_ALLOC(dd, size_t(nbytes));
    RTNQ_ALLOC(dc, size_t(n));
    RTNQ_TRY(h2d(dd.p, bytes, size_t(nbytes)));
    launch_decode(dd.as<uint8_t>(), Layout{RTNQ_ROW_MAJOR, 16, 4}, bits, 1, n, dc.as<int8_t>(),
                  host_stream());
    RTNQ_TRY(d2h(out, dc.p, size_t(n)));
    return sync_host();
}

rtnq_status rtnq_logical_codes(const uint8_t* data, int64_t nbytes, rtnq_layout layout, int bits,
                               int64_t rows, int64_t cols, int8_t* out) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    RTNQ_TRY(check_layout(layout));
    if (nbytes != rtnq_layout_bytes(layout, bits, rows, cols))
        return fail(RTNQ_E_CORRUPT, "packed buffer size does not match its layout");
    if (rows * cols == 0) return RTNQ_OK;
    RTNQ_ALLOC(dd, size_t(nbytes));
    RTNQ_ALLOC(dc, size_t(rows * cols));
    RTNQ_TRY(h2d(dd.p, data, size_t(nbytes)));
    launch_decode(dd.as<uint8_t>(), to_layout(layout), bits, rows, cols, dc.as<int8_t>(),
                  host_stream());
    RTNQ_TRY(d2h(out, dc.p, size_t(rows * cols)));
    return sync_host();
}

rtnq_status rtnq_reshuffle(const uint8_t* data, int64_t nbytes, rtnq_layout from, rtnq_layout to,
                           int bits, int64_t rows, int64_t cols, uint8_t* out) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    RTNQ_TRY(check_layout(from));
    RTNQ_TRY(check_layout(to));
    if (nbytes != rtnq_layout_bytes(from, bits, rows, cols))
        return fail(RTNQ_E_CORRUPT, "packed buffer size does not match its layout");
    const int64_t obytes = rtnq_layout_bytes(to, bits, rows, cols);
    if (obytes == 0) return RTNQ_OK;
    RTNQ_ALLOC(dsrc, size_t(nbytes));
    RTNQ_ALLOC(ddst, size_t(obytes));
    RTNQ_TRY(h2d(dsrc.p, data, size_t(nbytes)));
    launch_relayout(dsrc.as<uint8_t>(), to_layout(from), ddst.as<uint8_t>(), to_layout(to), bits,
                    rows, cols, host_stream());
    RTNQ_TRY(d2h(out, ddst.p, size_t(obytes)));
    return sync_host();
}

rtnq_status rtnq_dequantize_tensor(const uint8_t* data, int64_t nbytes, rtnq_layout layout,
                                   int bits, int64_t rows, int64_t cols, int64_t g, int ragged,
                                   const float* scales, float* out) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    RTNQ_TRY(check_layout(layout));
    const int64_t gpr = rtnq_groups_per_row(g, ragged, cols);
    if (gpr < 0) return rtnq_status(-gpr);
    if (nbytes != rtnq_layout_bytes(layout, bits, rows, cols))
        return fail(RTNQ_E_CORRUPT, "packed buffer size does not match its layout");
    if (rows * cols == 0) return RTNQ_OK;
    RTNQ_ALLOC(dd, size_t(nbytes));
    RTNQ_ALLOC(ds, size_t(rows * gpr) * 4);
    RTNQ_ALLOC(dout, size_t(rows * cols) * 4);
    RTNQ_TRY(h2d(dd.p, data, size_t(nbytes)));
    RTNQ_TRY(h2d(ds.p, scales, size_t(rows * gpr) * 4));
    launch_dequant(dd.as<uint8_t>(), to_layout(layout), bits, rows, cols, g, gpr, ds.p, RTNQ_F32,
                   RTNQ_SCALES_REF, dout.p, RTNQ_F32, host_stream());
    RTNQ_TRY(d2h(out, dout.p, size_t(rows * cols) * 4));
    return sync_host();
}

rtnq_status rtnq_gemm(int path, const float* a, int64_t m, int64_t k, const uint8_t* data,
                      int64_t nbytes, rtnq_layout layout, int bits, int64_t n, int64_t g,
                      int ragged, const float* scales, int64_t threshold, int* chosen,
                      float* out) {
    if (!valid_bits(bits)) return fail(RTNQ_E_INVALID_INPUT, "bits must be 4 or 8");
    RTNQ_TRY(check_layout(layout));
    // gemm_auto validates the threshold and the layout first (gemm.cpp:102-104)
    if (path == RTNQ_PATH_AUTO) {
        if (threshold < 1) return fail(RTNQ_E_INVALID_INPUT, "dispatch threshold must be >= 1");
        if (layout.kind != RTNQ_KERNEL_INTERLEAVED)
            return fail(RTNQ_E_SHAPE, "auto GEMM requires the kernel_interleaved layout");
        path = m >= threshold ? RTNQ_PATH_DEQUANT_FIRST : RTNQ_PATH_FUSED;
        if (chosen) *chosen = path;
    }
    const int64_t gpr = rtnq_groups_per_row(g, ragged, k);
    if (gpr < 0) return rtnq_status(-gpr);
    if (nbytes != rtnq_layout_bytes(layout, bits, n, k))
        return fail(RTNQ_E_CORRUPT, "packed buffer size does not match its layout");
    RTNQ_ALLOC(da, size_t(m * k) * 4 + 4);
    int32_t* derr = reinterpret_cast<int32_t*>(da.as<char>() + size_t(m * k) * 4);
    RTNQ_CUDA(cudaMemsetAsync(derr, 0, 4, host_stream()));
    RTNQ_TRY(h2d(da.p, a, size_t(m * k) * 4));
    // check_shapes (gemm.cpp:14-19): non-finite activations first
    if (m * k) {
        launch_check_finite(da.p, RTNQ_F32, m * k, derr, host_stream());
        int32_t herr = 0;
        RTNQ_TRY(d2h(&herr, derr, 4));
        RTNQ_TRY(sync_host());
        if (herr) return fail(RTNQ_E_INVALID_INPUT, "non-finite activation value");
    }
    if (path == RTNQ_PATH_FUSED && layout.kind != RTNQ_KERNEL_INTERLEAVED)
        return fail(RTNQ_E_SHAPE, "fused GEMM requires the kernel_interleaved layout");
    if (m * n == 0) return RTNQ_OK;
    const size_t wsb = path == RTNQ_PATH_DEQUANT_FIRST ? size_t(n * k) * 4 + kCountersReserve : 0;
    RTNQ_ALLOC(dd, size_t(nbytes));
    RTNQ_ALLOC(ds, size_t(n * gpr) * 4);
    RTNQ_ALLOC(dout, size_t(m * n) * 4);
    RTNQ_ALLOC(dws, wsb);
    RTNQ_TRY(h2d(dd.p, data, size_t(nbytes)));
    RTNQ_TRY(h2d(ds.p, scales, size_t(n * gpr) * 4));
    RTNQ_TRY(rtnq_dev_linear(da.p, RTNQ_F32, m, k, dd.as<uint8_t>(), layout, bits, n, g, ragged,
                             ds.p, RTNQ_F32, RTNQ_SCALES_REF, dout.p, RTNQ_F32, path, 1, nullptr,
                             nullptr, dws.p, wsb, host_stream()));
    RTNQ_TRY(d2h(out, dout.p, size_t(m * n) * 4));
    return sync_host();
}

rtnq_status rtnq_gemm_float(const float* a, int64_t m, int64_t k, const float* w, int64_t n,
                            int64_t block, float* out) {
    if (block < 1) return fail(RTNQ_E_INVALID_INPUT, "accumulation block must be >= 1");
    RTNQ_ALLOC(da, size_t(m * k) * 4 + 4);
    int32_t* derr = reinterpret_cast<int32_t*>(da.as<char>() + size_t(m * k) * 4);
    RTNQ_CUDA(cudaMemsetAsync(derr, 0, 4, host_stream()));
    RTNQ_TRY(h2d(da.p, a, size_t(m * k) * 4));
    if (m * k) {
        launch_check_finite(da.p, RTNQ_F32, m * k, derr, host_stream());
        int32_t herr = 0;
        RTNQ_TRY(d2h(&herr, derr, 4));
        RTNQ_TRY(sync_host());
        if (herr) return fail(RTNQ_E_INVALID_INPUT, "non-finite activation value");
    }
    if (m * n == 0) return RTNQ_OK;
    RTNQ_ALLOC(dw, size_t(n * k) * 4);
    RTNQ_ALLOC(dout, size_t(m * n) * 4);
    RTNQ_TRY(h2d(dw.p, w, size_t(n * k) * 4));
    launch_dense_blocked(da.as<float>(), m, k, dw.as<float>(), n, block, dout.as<float>(),
                         host_stream());
    RTNQ_TRY(d2h(out, dout.p, size_t(m * n) * 4));
    return sync_host();
}

}  // extern "C"
