// device.cpp -- rtnq/device.hpp on top of the C-ABI (rtnq_capi.h).
#include "rtnq/device.hpp"

#include <cuda_runtime.h>

#include <utility>

#include "rtnq/quant.hpp"
#include "status.hpp"

namespace rtnq {

using detail::check;

namespace {
void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}
template <class T>
T* dev_alloc(std::size_t bytes) {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, bytes ? bytes : 1), "cudaMalloc");
    return static_cast<T*>(p);
}
std::int64_t gpr_of(GroupSpec g, std::int64_t cols) { return g.groups_per_row(cols); }
}  // namespace

DeviceQuantTensor::DeviceQuantTensor(DeviceQuantTensor&& o) noexcept { *this = std::move(o); }

DeviceQuantTensor& DeviceQuantTensor::operator=(DeviceQuantTensor&& o) noexcept {
    if (this != &o) {
        cudaFree(codes_);
        cudaFree(scales_);
        rows_ = o.rows_, cols_ = o.cols_, bits_ = o.bits_, group_ = o.group_, kind_ = o.kind_;
        codes_ = std::exchange(o.codes_, nullptr);
        scales_ = std::exchange(o.scales_, nullptr);
    }
    return *this;
}

DeviceQuantTensor::~DeviceQuantTensor() {
    cudaFree(codes_);
    cudaFree(scales_);
}

// The fastest kernel's operand layout for a shape (same rule as the Python quantize_pack).
static int best_kind(int bits, std::int64_t g, std::int64_t cols) {
    if (bits == 8 && g >= cols) return RTNQ_NATIVE_I8;
    if (bits == 4 && g == 128) return RTNQ_NATIVE_I4;
    return RTNQ_NATIVE_SM100;
}

DeviceQuantTensor DeviceQuantTensor::quantize(const void* weights, std::int64_t rows,
                                              std::int64_t cols, DType dtype, BitWidth bits,
                                              GroupSpec group, void* stream) {
    DeviceQuantTensor t;
    t.rows_ = rows, t.cols_ = cols, t.bits_ = bits, t.group_ = group;
    const int b = bit_count(bits);
    t.kind_ = best_kind(b, group.g, cols);
    const rtnq_layout lay{t.kind_, 16, 4};
    const std::int64_t gpr = gpr_of(group, cols);
    t.codes_ = dev_alloc<std::uint8_t>(std::size_t(rtnq_layout_bytes(lay, b, rows, cols)));
    t.scales_ = dev_alloc<std::uint16_t>(std::size_t(rtnq_native_scale_count(rows, gpr)) * 2);
    const int ragged = group.allow_ragged ? 1 : 0;
    const std::size_t wsb = rtnq_dev_quantize_workspace_bytes(rows, cols, b, group.g, ragged);
    void* ws = dev_alloc<char>(wsb + 4);
    auto* err = reinterpret_cast<std::int32_t*>(static_cast<char*>(ws) + wsb);
    cuda_check(cudaMemsetAsync(err, 0, 4, static_cast<cudaStream_t>(stream)), "cudaMemsetAsync");
    // the int8-MMA layouts are relaid out from the reference's row-major bytes
    const rtnq_layout rm{RTNQ_ROW_MAJOR, 16, 4};
    std::uint8_t* rmb = t.kind_ == RTNQ_NATIVE_SM100
        ? nullptr : dev_alloc<std::uint8_t>(std::size_t(rtnq_layout_bytes(rm, b, rows, cols)));
    rtnq_status st = rtnq_dev_quantize_pack(weights, int(dtype), rows, cols, b, group.g, ragged,
                                            rmb, nullptr, rmb ? nullptr : t.codes_, nullptr, nullptr,
                                            t.scales_, err, ws, wsb, stream);
    if (st == RTNQ_OK) st = rtnq_dev_check_flag(err, stream);
    if (st == RTNQ_OK && rmb) st = rtnq_dev_relayout(rmb, rm, t.codes_, lay, b, rows, cols, stream);
    if (rmb) cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
    cudaFree(rmb);
    cudaFree(ws);
    check(st);
    return t;
}

DeviceQuantTensor DeviceQuantTensor::from_host(const QuantTensor& q, void* stream) {
    DeviceQuantTensor t;
    t.rows_ = q.rows, t.cols_ = q.cols, t.bits_ = q.bits, t.group_ = q.group;
    const int b = bit_count(q.bits);
    t.kind_ = best_kind(b, q.group.g, q.cols);
    const rtnq_layout nat{t.kind_, 16, 4};
    const std::int64_t gpr = q.groups_per_row();
    auto st_ = static_cast<cudaStream_t>(stream);
    std::uint8_t* src = dev_alloc<std::uint8_t>(q.data.size());
    float* s32 = dev_alloc<float>(q.scales.size() * 4);
    cuda_check(cudaMemcpyAsync(src, q.data.data(), q.data.size(), cudaMemcpyHostToDevice, st_),
               "cudaMemcpyAsync");
    cuda_check(cudaMemcpyAsync(s32, q.scales.data(), q.scales.size() * 4, cudaMemcpyHostToDevice,
                               st_),
               "cudaMemcpyAsync");
    t.codes_ = dev_alloc<std::uint8_t>(std::size_t(rtnq_layout_bytes(nat, b, q.rows, q.cols)));
    t.scales_ = dev_alloc<std::uint16_t>(std::size_t(rtnq_native_scale_count(q.rows, gpr)) * 2);
    rtnq_status st = rtnq_dev_relayout(src, detail::to_c(q.layout), t.codes_, nat, b, q.rows,
                                       q.cols, stream);
    if (st == RTNQ_OK) st = rtnq_dev_native_scales(s32, RTNQ_F32, q.rows, gpr, t.scales_, stream);
    cudaStreamSynchronize(st_);
    cudaFree(src);
    cudaFree(s32);
    check(st);
    return t;
}

DeviceWorkspace::~DeviceWorkspace() { cudaFree(ptr_); }

void* DeviceWorkspace::ensure(std::size_t bytes, void* stream) {
    if (bytes <= bytes_) return ptr_;
    cudaFree(ptr_);
    ptr_ = dev_alloc<char>(bytes);
    bytes_ = bytes;
    cuda_check(cudaMemsetAsync(ptr_, 0, bytes, static_cast<cudaStream_t>(stream)), "cudaMemsetAsync");
    return ptr_;
}

void linear(const void* a, std::int64_t m, DType a_dtype, const DeviceQuantTensor& w, void* out,
            DType out_dtype, DeviceWorkspace& ws, void* stream, bool pdl) {
    const rtnq_layout nat{w.layout_kind(), 16, 4};
    const int b = bit_count(w.bits());
    const std::size_t need = rtnq_dev_linear_workspace_bytes(m, w.rows(), w.cols(), b, w.group().g,
                                                             RTNQ_PATH_FUSED, nat);
    void* p = ws.ensure(need, stream);
    check(rtnq_dev_linear_ex(a, int(a_dtype), m, w.cols(), w.codes(), nat, b, w.rows(),
                             w.group().g, w.group().allow_ragged ? 1 : 0, w.scales(), RTNQ_F16,
                             RTNQ_SCALES_NATIVE, out, int(out_dtype), RTNQ_PATH_FUSED, 1, nullptr,
                             nullptr, p, ws.bytes(), stream, pdl ? RTNQ_FLAG_PDL : 0u));
}

}  // namespace rtnq
