// gemm.cpp -- quantized GEMMs on the B200 (drop-in for proj/core/src/gemm.cpp).
// The host-tensor API runs the reference-exact CUDA kernels (bit-identical
// results); see rtnq_dev_linear for the tensor-core performance path.
#include "rtnq/gemm.hpp"

#include "status.hpp"

namespace rtnq {

using detail::check;
using detail::to_c;

namespace {

FloatTensor run(int path, const FloatTensor& a, const QuantTensor& w, std::int64_t threshold,
                GemmPath* chosen) {
    if (a.cols != w.cols)
        throw ShapeError("activation width " + std::to_string(a.cols) +
                         " does not match weight input width " + std::to_string(w.cols));
    FloatTensor out(a.rows, w.rows);
    int taken = -1;
    check(rtnq_gemm(path, a.data.data(), a.rows, a.cols, w.data.data(),
                    std::int64_t(w.data.size()), to_c(w.layout), bit_count(w.bits), w.rows,
                    w.group.g, w.group.allow_ragged ? 1 : 0, w.scales.data(), threshold, &taken,
                    out.data.data()));
    if (chosen) *chosen = taken == RTNQ_PATH_DEQUANT_FIRST ? GemmPath::dequant_first : GemmPath::fused;
    return out;
}

}  // namespace

FloatTensor gemm_fused(const FloatTensor& a, const QuantTensor& w) {
    return run(RTNQ_PATH_FUSED, a, w, 1, nullptr);
}

FloatTensor gemm_dequant(const FloatTensor& a, const QuantTensor& w) {
    return run(RTNQ_PATH_DEQUANT_FIRST, a, w, 1, nullptr);
}

FloatTensor gemm_auto(const FloatTensor& a, const QuantTensor& w, std::int64_t threshold,
                      GemmPath* chosen) {
    // threshold and layout are validated before shapes, as in the reference
    if (threshold < 1) throw InvalidInputError("dispatch threshold must be >= 1");
    if (!w.layout.interleaved())
        throw ShapeError("auto GEMM requires the kernel_interleaved layout");
    return run(RTNQ_PATH_AUTO, a, w, threshold, chosen);
}

FloatTensor gemm_oracle(const FloatTensor& a, const QuantTensor& w) {
    return run(RTNQ_PATH_ORACLE, a, w, 1, nullptr);
}

FloatTensor gemm_float(const FloatTensor& a, const FloatTensor& w, std::int64_t block) {
    if (a.cols != w.cols)
        throw ShapeError("activation width " + std::to_string(a.cols) +
                         " does not match weight input width " + std::to_string(w.cols));
    FloatTensor out(a.rows, w.rows);
    check(rtnq_gemm_float(a.data.data(), a.rows, a.cols, w.data.data(), w.rows, block,
                          out.data.data()));
    return out;
}

}  // namespace rtnq
