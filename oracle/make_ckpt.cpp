// make_ckpt.cpp -- TEST INFRASTRUCTURE ONLY.  Writes RTNCKPT1 golden fixtures with the
// reference's own store.cpp (write_checkpoint, store.cpp:310-364) and dumps what the
// reference's loader reads back (load_quant_checkpoint -> read_quant_tensor,
// store.cpp:286-306): per tensor the logical int8 codes and the f32 (f16-widened) scales.
// Built by oracle/Makefile (target _ref/make_ckpt) from the sources under /root/reference;
// run by tests/golden/make_ckpt_golden.py.
#include <cstdio>
#include <fstream>
#include <string>

#include "rtnq/plan.hpp"
#include "rtnq/quant.hpp"
#include "rtnq/store.hpp"
#include "rtnq/toy.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: make_ckpt OUT_DIR PLAN\n");
        return 2;
    }
    const std::string dir = argv[1];
    rtnq::ToyTransformerConfig cfg;
    cfg.layers = 3;
    cfg.dim = 128;
    cfg.heads = 4;
    cfg.ffn = 256;
    cfg.seed = 7;
    rtnq::FloatModel fm = rtnq::make_toy_model(cfg);
    fm.manifest.group = rtnq::GroupSpec{128, false};
    rtnq::write_checkpoint(fm, dir + "/toy_f32.rtnckpt");
    const rtnq::SelectionPlan plan = rtnq::parse_plan(argv[2]);
    rtnq::QuantModel qm = rtnq::quantize_model(fm, plan, rtnq::GroupSpec{128, false});
    rtnq::write_checkpoint(qm, dir + "/toy_q.rtnckpt");
    // what the reference loader yields
    const rtnq::QuantModel back = rtnq::load_quant_checkpoint(dir + "/toy_q.rtnckpt");
    std::ofstream os(dir + "/toy_q.expect", std::ios::binary);
    for (const rtnq::QuantTensor& q : back.tensors) {
        const std::vector<std::int8_t> codes = rtnq::logical_codes(q);
        const std::int64_t hdr[3] = {q.rows, q.cols, static_cast<std::int64_t>(q.bits)};
        os.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
        os.write(reinterpret_cast<const char*>(codes.data()), static_cast<std::streamsize>(codes.size()));
        os.write(reinterpret_cast<const char*>(q.scales.data()),
                 static_cast<std::streamsize>(q.scales.size() * sizeof(float)));
    }
    return 0;
}
