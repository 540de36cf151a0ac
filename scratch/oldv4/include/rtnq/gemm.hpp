// rtnq/gemm.hpp -- quantized linear (drop-in for proj/core/include/rtnq/gemm.hpp).
// These host-tensor entry points run the reference-exact CUDA kernels and return
// results bit-identical to the reference.  The performance path (bf16/f16
// activations, native layout, tensor cores) is rtnq_dev_linear (rtnq_capi.h) or
// rtnq::DeviceQuantTensor (rtnq/device.hpp).
#pragma once

#include <cstdint>

#include "rtnq/quant.hpp"
#include "rtnq/types.hpp"

namespace rtnq {

enum class GemmPath : std::uint8_t { fused = 0, dequant_first = 1 };

constexpr std::int64_t kDefaultGemmThreshold = 1024;

// out[i][j] = sum_k a[i][k] * scale(j, k/g) * code(j, k); per output element k
// is reduced in group-sized blocks (block subtotal, then add).
FloatTensor gemm_fused(const FloatTensor& a, const QuantTensor& w);    // kernel_interleaved
FloatTensor gemm_dequant(const FloatTensor& a, const QuantTensor& w);  // any layout
FloatTensor gemm_auto(const FloatTensor& a, const QuantTensor& w,
                      std::int64_t threshold = kDefaultGemmThreshold,
                      GemmPath* chosen = nullptr);
FloatTensor gemm_oracle(const FloatTensor& a, const QuantTensor& w);   // f64 ground truth
FloatTensor gemm_float(const FloatTensor& a, const FloatTensor& w, std::int64_t block);

}  // namespace rtnq
