// rtnq/device.hpp -- device-resident quantized weights and the tensor-core linear for
// C++ consumers (the B200 performance path; no reference counterpart -- the reference's
// QuantTensor lives in host memory, quant.hpp:26-46).
//
//   rtnq::DeviceQuantTensor w = rtnq::DeviceQuantTensor::quantize(d_weights, rows, cols,
//                                   rtnq::DType::bf16, rtnq::BitWidth::b4, rtnq::GroupSpec{128},
//                                   stream);
//   rtnq::linear(d_act, m, rtnq::DType::bf16, w, d_out, rtnq::DType::bf16, ws, stream);
//
// Every call is asynchronous on `stream` (a cudaStream_t passed as void*) and throws the
// reference's exception classes on invalid arguments.
#pragma once

#include <cstddef>
#include <cstdint>

#include "rtnq/types.hpp"

namespace rtnq {

enum class DType : int { f32 = 0, f16 = 1, bf16 = 2 };  // RTNQ_F32 / RTNQ_F16 / RTNQ_BF16

// Owns device memory for native-layout codes and native-order f16 scales.
class DeviceQuantTensor {
public:
    DeviceQuantTensor() = default;
    DeviceQuantTensor(const DeviceQuantTensor&) = delete;
    DeviceQuantTensor& operator=(const DeviceQuantTensor&) = delete;
    DeviceQuantTensor(DeviceQuantTensor&& o) noexcept;
    DeviceQuantTensor& operator=(DeviceQuantTensor&& o) noexcept;
    ~DeviceQuantTensor();

    // RTN quantize-and-pack of a device weight matrix (rows x cols, row-major) on the
    // GPU, bit-exact with quantize_tensor (quant.cpp:100-141).  Throws InvalidInputError
    // for non-finite weights (synchronizes `stream` to check).
    static DeviceQuantTensor quantize(const void* weights, std::int64_t rows, std::int64_t cols,
                                      DType dtype, BitWidth bits, GroupSpec group,
                                      void* stream = nullptr);
    // Upload a reference QuantTensor (any layout, f32 scales) into the native layout.
    static DeviceQuantTensor from_host(const struct QuantTensor& q, void* stream = nullptr);

    std::int64_t rows() const { return rows_; }
    std::int64_t cols() const { return cols_; }
    BitWidth bits() const { return bits_; }
    GroupSpec group() const { return group_; }
    const std::uint8_t* codes() const { return codes_; }
    const std::uint16_t* scales() const { return scales_; }
    // codes layout: RTNQ_NATIVE_I4 (W4 group 128), RTNQ_NATIVE_I8 (W8 per-channel) -- the
    // operands of the int8 tensor-core kernels -- else RTNQ_NATIVE_SM100
    int layout_kind() const { return kind_; }

private:
    std::int64_t rows_ = 0, cols_ = 0;
    BitWidth bits_ = BitWidth::b4;
    GroupSpec group_;
    std::uint8_t* codes_ = nullptr;
    std::uint16_t* scales_ = nullptr;
    int kind_ = 2;
};

// Scratch for linear(): stream-K partials and self-resetting counters (zeroed once).
class DeviceWorkspace {
public:
    DeviceWorkspace() = default;
    DeviceWorkspace(const DeviceWorkspace&) = delete;
    DeviceWorkspace& operator=(const DeviceWorkspace&) = delete;
    ~DeviceWorkspace();
    void* ensure(std::size_t bytes, void* stream);
    std::size_t bytes() const { return bytes_; }

private:
    void* ptr_ = nullptr;
    std::size_t bytes_ = 0;
};

// out (m x rows) = a (m x cols) * W^T on the tcgen05 kernel (rtnq_dev_linear_ex, FUSED
// path).  a: bf16 or f16, device, row-major; out: f32 / f16 / bf16.  pdl: overlap this
// kernel's prologue and weight prefetch with the previous kernel in the stream.
void linear(const void* a, std::int64_t m, DType a_dtype, const DeviceQuantTensor& w, void* out,
            DType out_dtype, DeviceWorkspace& ws, void* stream = nullptr, bool pdl = false);

}  // namespace rtnq
