// f16.cpp -- binary16 conversions (drop-in for proj/core/src/f16.cpp), through the
// compiler's _Float16 (IEEE round-to-nearest-even, the same rounding the GPU's
// __float2half_rn uses for the scale outputs of the quantize kernels).
#include "rtnq/f16.hpp"

#include <bit>

#include "rtnq_capi.h"

namespace rtnq {

std::uint16_t f32_to_f16(float value) {
    const _Float16 h = static_cast<_Float16>(value);
    std::uint16_t bits = std::bit_cast<std::uint16_t>(h);
    if ((bits & 0x7C00u) == 0x7C00u && (bits & 0x03FFu) != 0) bits |= 0x0200u;  // quiet NaN
    return bits;
}

float f16_to_f32(std::uint16_t bits) {
    return static_cast<float>(std::bit_cast<_Float16>(bits));
}

}  // namespace rtnq

extern "C" rtnq_status rtnq_f32_to_f16(const float* in, int64_t n, uint16_t* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = rtnq::f32_to_f16(in[i]);
    return RTNQ_OK;
}

extern "C" rtnq_status rtnq_f16_to_f32(const uint16_t* in, int64_t n, float* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = rtnq::f16_to_f32(in[i]);
    return RTNQ_OK;
}
