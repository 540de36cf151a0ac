// rtnq/f16.hpp -- IEEE binary16 conversions (drop-in for proj/core/include/rtnq/f16.hpp).
#pragma once

#include <cstdint>

namespace rtnq {

std::uint16_t f32_to_f16(float value);  // round to nearest even (== __float2half_rn)
float f16_to_f32(std::uint16_t bits);   // exact

}  // namespace rtnq
