// quant.cpp -- rtnq quantization API on the B200 (drop-in for proj/core/src/quant.cpp).
// Each function validates like the reference and delegates the arithmetic to the
// C-ABI (GPU kernels in csrc/kernels).
#include "rtnq/quant.hpp"

#include "rtnq/packing.hpp"
#include "status.hpp"

namespace rtnq {

using detail::check;
using detail::to_c;

std::int64_t QuantTensor::padded_rows() const {
    if (layout.kind == LayoutTag::Kind::row_major) return rows;
    const std::int64_t t = layout.kind == LayoutTag::Kind::native_sm100 ? 16 : layout.tile_rows;
    return (rows + t - 1) / t * t;
}

std::int64_t QuantTensor::padded_cols() const {
    if (layout.kind == LayoutTag::Kind::row_major) return cols;
    const std::int64_t t = layout.kind == LayoutTag::Kind::native_sm100
                               ? (bits == BitWidth::b4 ? 64 : 32)
                               : layout.tile_cols;
    return (cols + t - 1) / t * t;
}

std::int64_t QuantTensor::stored_codes() const { return padded_rows() * padded_cols(); }

int QuantTensor::code_at(std::int64_t r, std::int64_t c) const {
    const std::int64_t slot = layout_index(layout, bits, rows, cols, r, c);
    if (bits == BitWidth::b8) return int(data[static_cast<std::size_t>(slot)]) - 128;
    const std::uint8_t b = data[static_cast<std::size_t>(slot >> 1)];
    return int((slot & 1) ? (b >> 4) : (b & 0x0F)) - 8;
}

float compute_scale(std::span<const float> values, BitWidth bits) {
    float s = 0.0f;
    check(rtnq_compute_scale(values.data(), std::int64_t(values.size()), bit_count(bits), &s));
    return s;
}

std::vector<std::int8_t> quantize_group(std::span<const float> values, BitWidth bits,
                                        float scale) {
    std::vector<std::int8_t> codes(values.size());
    check(rtnq_quantize_group(values.data(), std::int64_t(values.size()), bit_count(bits), &scale,
                              nullptr, codes.data()));
    return codes;
}

std::vector<std::int8_t> quantize_group(std::span<const float> values, BitWidth bits,
                                        float* scale_out) {
    std::vector<std::int8_t> codes(values.size());
    float s = 0.0f;
    check(rtnq_quantize_group(values.data(), std::int64_t(values.size()), bit_count(bits), nullptr,
                              &s, codes.data()));
    if (scale_out) *scale_out = s;
    return codes;
}

std::vector<float> dequantize_group(std::span<const std::int8_t> codes, float scale,
                                    BitWidth bits) {
    std::vector<float> out(codes.size());
    check(rtnq_dequantize_group(codes.data(), std::int64_t(codes.size()), scale, bit_count(bits),
                                out.data()));
    return out;
}

QuantTensor quantize_tensor(const FloatTensor& w, BitWidth bits, GroupSpec group) {
    if (static_cast<std::int64_t>(w.data.size()) != w.rows * w.cols)
        throw ShapeError("tensor data size does not match rows*cols");
    const std::int64_t gpr = group.groups_per_row(w.cols);
    QuantTensor q;
    q.rows = w.rows;
    q.cols = w.cols;
    q.bits = bits;
    q.group = group;
    q.layout = LayoutTag::row_major();
    q.data.assign(static_cast<std::size_t>(packed_size(w.rows * w.cols, bits)), 0);
    q.scales.assign(static_cast<std::size_t>(w.rows * gpr), 0.0f);
    check(rtnq_quantize_tensor(w.data.data(), w.rows, w.cols, bit_count(bits), group.g,
                               group.allow_ragged ? 1 : 0, q.data.data(), q.scales.data()));
    return q;
}

FloatTensor dequantize_tensor(const QuantTensor& q) {
    FloatTensor out(q.rows, q.cols);
    check(rtnq_dequantize_tensor(q.data.data(), std::int64_t(q.data.size()), to_c(q.layout),
                                 bit_count(q.bits), q.rows, q.cols, q.group.g,
                                 q.group.allow_ragged ? 1 : 0, q.scales.data(), out.data.data()));
    return out;
}

std::vector<std::int8_t> logical_codes(const QuantTensor& q) {
    std::vector<std::int8_t> codes(static_cast<std::size_t>(q.rows * q.cols));
    check(rtnq_logical_codes(q.data.data(), std::int64_t(q.data.size()), to_c(q.layout),
                             bit_count(q.bits), q.rows, q.cols, codes.data()));
    return codes;
}

}  // namespace rtnq
