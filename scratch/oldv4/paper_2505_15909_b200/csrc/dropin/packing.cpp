// packing.cpp -- packing and layouts on the B200 (drop-in for proj/core/src/packing.cpp).
#include "rtnq/packing.hpp"

#include "status.hpp"

namespace rtnq {

using detail::check;
using detail::to_c;

PackedBuffer pack(std::span<const std::int8_t> codes, BitWidth bits) {
    PackedBuffer buf;
    buf.bits = bits;
    buf.logical_len = std::int64_t(codes.size());
    buf.bytes.assign(static_cast<std::size_t>(packed_size(buf.logical_len, bits)), 0);
    check(rtnq_pack(codes.data(), buf.logical_len, bit_count(bits), buf.bytes.data()));
    return buf;
}

std::vector<std::int8_t> unpack(const PackedBuffer& buf) {
    if (buf.logical_len < 0)
        throw CorruptDataError("negative logical length");
    std::vector<std::int8_t> codes(static_cast<std::size_t>(buf.logical_len));
    check(rtnq_unpack(buf.bytes.data(), std::int64_t(buf.bytes.size()), buf.logical_len,
                      bit_count(buf.bits), codes.data()));
    return codes;
}

std::int64_t layout_index(const LayoutTag& tag, BitWidth bits, std::int64_t rows,
                          std::int64_t cols, std::int64_t r, std::int64_t c) {
    const std::int64_t v = rtnq_layout_index(to_c(tag), bit_count(bits), rows, cols, r, c);
    if (v < 0) check(rtnq_status(-v));
    return v;
}

std::int64_t layout_index(const LayoutTag& tag, std::int64_t rows, std::int64_t cols,
                          std::int64_t r, std::int64_t c) {
    return layout_index(tag, BitWidth::b4, rows, cols, r, c);
}

std::int64_t layout_slots(const LayoutTag& tag, BitWidth bits, std::int64_t rows,
                          std::int64_t cols) {
    const std::int64_t v = rtnq_layout_slots(to_c(tag), bit_count(bits), rows, cols);
    if (v < 0) check(rtnq_status(-v));
    return v;
}

std::int64_t layout_slots(const LayoutTag& tag, std::int64_t rows, std::int64_t cols) {
    return layout_slots(tag, BitWidth::b4, rows, cols);
}

QuantTensor reshuffle(const QuantTensor& q, const LayoutTag& to) {
    if (to == q.layout) return q;
    if (to.kind == LayoutTag::Kind::kernel_interleaved && (to.tile_rows <= 0 || to.tile_cols <= 0))
        throw InvalidInputError("kernel tile dimensions must be positive");
    QuantTensor out = q;
    out.layout = to;
    out.data.assign(static_cast<std::size_t>(
                        packed_size(layout_slots(to, q.bits, q.rows, q.cols), q.bits)),
                    0);
    check(rtnq_reshuffle(q.data.data(), std::int64_t(q.data.size()), to_c(q.layout), to_c(to),
                         bit_count(q.bits), q.rows, q.cols, out.data.data()));
    return out;
}

}  // namespace rtnq
