// ref_shim.cpp -- extern "C" wrapper around the UNMODIFIED reference rtnq
// library, compiled from the sources where they lie under /root/reference by
// oracle/Makefile into oracle/_ref/librtnq_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used to (1) pin the C restatement in
// oracle/rtnq_oracle.c, (2) generate tests/golden/ fixtures, and (3) serve as
// the CPU baseline / `bench.py --impl reference` arm.  Never linked by the
// product.  Exceptions are mapped to the status codes of include/rtnq_capi.h.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "rtnq/error.hpp"
#include "rtnq/f16.hpp"
#include "rtnq/gemm.hpp"
#include "rtnq/manifest.hpp"
#include "rtnq/packing.hpp"
#include "rtnq/plan.hpp"
#include "rtnq/quant.hpp"
#include "rtnq/threading.hpp"

using namespace rtnq;

namespace {
thread_local std::string g_err;

int map_exc() {
    try {
        throw;
    } catch (const PlanError& e) {
        g_err = e.what();
        return 4;
    } catch (const CorruptDataError& e) {
        g_err = e.what();
        return 3;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 2;
    } catch (const InvalidInputError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}

BitWidth bw(int bits) { return bits == 8 ? BitWidth::b8 : BitWidth::b4; }

FloatTensor ft(const float* p, int64_t r, int64_t c) {
    FloatTensor t(r, c);
    if (r * c != 0) std::memcpy(t.data.data(), p, sizeof(float) * r * c);
    return t;
}

void put(const FloatTensor& t, float* out) {
    if (t.size()) std::memcpy(out, t.data.data(), sizeof(float) * t.size());
}

QuantTensor qt(const uint8_t* data, int64_t nbytes, int64_t rows, int64_t cols, int bits,
               int64_t g, int ragged, int layout, int tr, int tc, const float* scales) {
    QuantTensor q;
    q.rows = rows;
    q.cols = cols;
    q.bits = bw(bits);
    q.group = GroupSpec{g, ragged != 0};
    q.layout = layout ? LayoutTag::kernel(tr, tc) : LayoutTag::row_major();
    q.data.assign(data, data + nbytes);
    q.scales.assign(scales, scales + rows * q.group.groups_per_row(cols));
    return q;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { set_threads(n); }
int ref_threads() { return threads(); }

uint16_t ref_f32_to_f16(float v) { return f32_to_f16(v); }
float ref_f16_to_f32(uint16_t h) { return f16_to_f32(h); }

int ref_compute_scale(const float* v, int64_t n, int bits, float* out) {
    try {
        *out = compute_scale(std::span<const float>(v, size_t(n)), bw(bits));
        return 0;
    } catch (...) {
        return map_exc();
    }
}

int ref_quantize_group(const float* v, int64_t n, int bits, float* scale_out, int8_t* codes) {
    try {
        auto c = quantize_group(std::span<const float>(v, size_t(n)), bw(bits), scale_out);
        std::memcpy(codes, c.data(), c.size());
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// quantize_tensor -> row-major packed bytes (q.data) and f32 scales.
int ref_quantize_tensor(const float* w, int64_t rows, int64_t cols, int bits, int64_t g,
                        int ragged, uint8_t* data, float* scales) {
    try {
        auto q = quantize_tensor(ft(w, rows, cols), bw(bits), GroupSpec{g, ragged != 0});
        std::memcpy(data, q.data.data(), q.data.size());
        std::memcpy(scales, q.scales.data(), q.scales.size() * sizeof(float));
        return 0;
    } catch (...) {
        return map_exc();
    }
}

int64_t ref_layout_slots(int layout, int tr, int tc, int64_t rows, int64_t cols) {
    return layout_slots(layout ? LayoutTag::kernel(tr, tc) : LayoutTag::row_major(), rows,
                        cols);
}

// reshuffle between row_major (0) and kernel_interleaved(tr, tc) (1).
int ref_reshuffle(const uint8_t* data, int64_t nbytes, int64_t rows, int64_t cols, int bits,
                  int64_t g, int ragged, int from, int to, int tr, int tc,
                  const float* scales, uint8_t* out) {
    try {
        auto q = qt(data, nbytes, rows, cols, bits, g, ragged, from, tr, tc, scales);
        auto r = reshuffle(q, to ? LayoutTag::kernel(tr, tc) : LayoutTag::row_major());
        std::memcpy(out, r.data.data(), r.data.size());
        return 0;
    } catch (...) {
        return map_exc();
    }
}

int ref_dequantize(const uint8_t* data, int64_t nbytes, int64_t rows, int64_t cols, int bits,
                   int64_t g, int ragged, int layout, int tr, int tc, const float* scales,
                   float* out) {
    try {
        put(dequantize_tensor(qt(data, nbytes, rows, cols, bits, g, ragged, layout, tr, tc,
                                 scales)),
            out);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// which: 0 fused, 1 dequant, 2 oracle, 3 auto(threshold)
int ref_gemm(int which, const float* a, int64_t m, int64_t k, const uint8_t* data,
             int64_t nbytes, int64_t n, int bits, int64_t g, int ragged, int layout, int tr,
             int tc, const float* scales, int64_t threshold, int* chosen, float* out) {
    try {
        auto q = qt(data, nbytes, n, k, bits, g, ragged, layout, tr, tc, scales);
        auto at = ft(a, m, k);
        FloatTensor o;
        if (which == 0) o = gemm_fused(at, q);
        else if (which == 1) o = gemm_dequant(at, q);
        else if (which == 2) o = gemm_oracle(at, q);
        else {
            GemmPath p{};
            o = gemm_auto(at, q, threshold, &p);
            if (chosen) *chosen = int(p);
        }
        put(o, out);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

int ref_gemm_float(const float* a, int64_t m, int64_t k, const float* w, int64_t n,
                   int64_t block, float* out) {
    try {
        put(gemm_float(ft(a, m, k), ft(w, n, k), block), out);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

// Plan text -> table (layer_count*4 entries of 4 or 8) or error + byte offset.
int ref_resolve_plan(const char* text, int64_t layers, uint8_t* table, int64_t* err_offset,
                     char* canon, int64_t canon_cap) {
    try {
        auto p = parse_plan(text);
        if (canon) {
            auto s = render_plan(p);
            std::strncpy(canon, s.c_str(), size_t(canon_cap));
        }
        if (layers > 0) {
            auto a = resolve_plan(p, layers);
            for (size_t i = 0; i < a.table.size(); ++i) table[i] = uint8_t(bit_count(a.table[i]));
        }
        return 0;
    } catch (const PlanError& e) {
        if (err_offset) *err_offset = e.offset() == PlanError::npos ? -1 : int64_t(e.offset());
        g_err = e.what();
        return 4;
    } catch (...) {
        return map_exc();
    }
}

// effective_bits over a 70B manifest (kind 1) or a uniform manifest (kind 0).
int ref_effective_bits(const uint8_t* table, int64_t layers, int kind, int64_t rows,
                       int64_t cols, int64_t g, int include_scales, double* out) {
    try {
        PrecisionAssignment a = PrecisionAssignment::uniform(layers, BitWidth::b4);
        for (size_t i = 0; i < a.table.size(); ++i) a.table[i] = bw(table[i]);
        ModelManifest m = kind ? make_70b_manifest()
                               : make_uniform_manifest(layers, rows, cols, GroupSpec{g});
        *out = effective_bits(a, m, include_scales != 0);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

}  // extern "C"
