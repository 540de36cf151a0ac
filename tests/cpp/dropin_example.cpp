// dropin_example.cpp -- a reference-style consumer of rtnq (the calls below are the
// README sketch of proj/README.md:156-167 plus the device API), compiled unchanged
// against the drop-in headers and linked to librtnq_b200.so.  With a directory argument it
// also dumps its inputs and every result there (raw little-endian arrays), and
// tests/test_dropin_cpp.py checks them against the CPU oracle (oracle/rtnq_oracle.c),
// independently of this library.  Exit code 0 = the self-checks below passed.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "rtnq/device.hpp"
#include "rtnq/gemm.hpp"
#include "rtnq/packing.hpp"
#include "rtnq/quant.hpp"

static float bf16_exact(float x) {  // truncate to a bf16-representable value
    unsigned u;
    std::memcpy(&u, &x, 4);
    u &= 0xFFFF0000u;
    std::memcpy(&x, &u, 4);
    return x;
}

static double rel_frob(const std::vector<float>& x, const std::vector<float>& ref) {
    double num = 0, den = 0;
    for (size_t i = 0; i < x.size(); ++i) {
        num += (double(x[i]) - ref[i]) * (double(x[i]) - ref[i]);
        den += double(ref[i]) * ref[i];
    }
    return den == 0 ? std::sqrt(num) : std::sqrt(num / den);
}

static void dump(const char* dir, const char* name, const void* p, size_t bytes) {
    if (!dir) return;
    std::string path = std::string(dir) + "/" + name;
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) return;
    std::fwrite(p, 1, bytes, f);
    std::fclose(f);
}

int main(int argc, char** argv) {
    const char* dir = argc > 1 ? argv[1] : nullptr;
    const std::int64_t n = 384, k = 1024, m = 4;
    std::mt19937 gen(7);
    std::uniform_real_distribution<float> u(-1.f, 1.f);
    rtnq::FloatTensor w(n, k), a(m, k);
    for (auto& v : w.data) v = bf16_exact(u(gen) * 0.05f);
    for (auto& v : a.data) v = bf16_exact(u(gen));

    // host drop-in API: exactly the reference calls
    rtnq::QuantTensor q = rtnq::quantize_tensor(w, rtnq::BitWidth::b4, rtnq::GroupSpec{128});
    rtnq::QuantTensor qk = rtnq::reshuffle(q, rtnq::LayoutTag::kernel(16, 4));
    rtnq::GemmPath chosen;
    rtnq::FloatTensor fused = rtnq::gemm_auto(a, qk, 1024, &chosen);
    rtnq::FloatTensor oracle = rtnq::gemm_oracle(a, q);
    const double e_host = rel_frob(fused.data, oracle.data);
    std::printf("host gemm_auto (path %d) vs gemm_oracle: %.3e\n", int(chosen), e_host);
    dump(dir, "w.f32", w.data.data(), w.data.size() * 4);
    dump(dir, "a.f32", a.data.data(), a.data.size() * 4);
    dump(dir, "q_data.u8", q.data.data(), q.data.size());
    dump(dir, "q_scales.f32", q.scales.data(), q.scales.size() * 4);
    dump(dir, "qk_data.u8", qk.data.data(), qk.data.size());
    dump(dir, "gemm_auto.f32", fused.data.data(), fused.data.size() * 4);
    dump(dir, "gemm_oracle.f32", oracle.data.data(), oracle.data.size() * 4);
    if (chosen != rtnq::GemmPath::fused || e_host > 1e-5) return 1;

    // device API: tensor-core linear on the same weights
    std::vector<unsigned short> wb(n * k), ab(m * k);
    for (size_t i = 0; i < wb.size(); ++i) { unsigned x; std::memcpy(&x, &w.data[i], 4); wb[i] = x >> 16; }
    for (size_t i = 0; i < ab.size(); ++i) { unsigned x; std::memcpy(&x, &a.data[i], 4); ab[i] = x >> 16; }
    void *dw, *da, *dout;
    cudaMalloc(&dw, wb.size() * 2);
    cudaMalloc(&da, ab.size() * 2);
    cudaMalloc(&dout, m * n * 4);
    cudaMemcpy(dw, wb.data(), wb.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(da, ab.data(), ab.size() * 2, cudaMemcpyHostToDevice);
    rtnq::DeviceQuantTensor dq = rtnq::DeviceQuantTensor::quantize(
        dw, n, k, rtnq::DType::bf16, rtnq::BitWidth::b4, rtnq::GroupSpec{128});
    rtnq::DeviceWorkspace ws;
    rtnq::linear(da, m, rtnq::DType::bf16, dq, dout, rtnq::DType::f32, ws);
    std::vector<float> out(m * n);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    // scales are stored as f16 on the device: compare against the oracle on f16-rounded scales
    rtnq::QuantTensor q16 = q;
    for (auto& s : q16.scales) s = float(_Float16(s));  // RNE, == f32_to_f16 (f16.cpp:8-41)
    rtnq::FloatTensor oracle16 = rtnq::gemm_oracle(a, q16);
    const double e_dev = rel_frob(out, oracle16.data);
    dump(dir, "device_linear.f32", out.data(), out.size() * 4);
    std::printf("device linear (tcgen05) vs gemm_oracle(f16 scales): %.3e\n", e_dev);

    // from_host: a reference QuantTensor uploaded into the native layout gives the same result
    rtnq::DeviceQuantTensor dq2 = rtnq::DeviceQuantTensor::from_host(q16);
    rtnq::linear(da, m, rtnq::DType::bf16, dq2, dout, rtnq::DType::f32, ws);
    std::vector<float> out2(m * n);
    cudaMemcpy(out2.data(), dout, out2.size() * 4, cudaMemcpyDeviceToHost);
    const double e_up = rel_frob(out2, out);
    std::printf("from_host vs quantize: %.3e\n", e_up);
    return (e_dev <= 1e-5 && e_up == 0.0) ? 0 : 2;
}
