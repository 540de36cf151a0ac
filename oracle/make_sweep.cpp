// make_sweep.cpp -- TEST INFRASTRUCTURE ONLY.  Runs the reference's own eval harness
// (eval.cpp:147-224: compare, horizontal_sweep, vertical_sweep, sweep_to_csv) on the default
// toy decoder (toy.hpp: 8 layers, dim 64, 4 heads, ffn 256, seq 32, group 64) and writes the
// results as golden fixtures for the GPU eval path (paper_2505_15909_b200/eval.py):
//   OUT_DIR/toy_sweeps.csv      horizontal first/middle/last + vertical, reference CSV format
//   OUT_DIR/toy_compare.txt     compare() reports for a few plans, one line per field
//   OUT_DIR/toy_probe.txt       PRNG probes: first values of every weight tensor and input
// Built by oracle/Makefile (target _ref/make_sweep) from the sources under /root/reference;
// run by tests/golden/make_sweep_golden.py.
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "rtnq/eval.hpp"
#include "rtnq/plan.hpp"
#include "rtnq/store.hpp"
#include "rtnq/toy.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: make_sweep OUT_DIR N_INPUTS\n");
        return 2;
    }
    const std::string dir = argv[1];
    const int n_inputs = std::atoi(argv[2]);
    const rtnq::ToyTransformerConfig cfg;  // the reference defaults
    const rtnq::FloatModel model = rtnq::make_toy_model(cfg);
    std::vector<rtnq::FloatTensor> inputs;
    for (int i = 0; i < n_inputs; ++i) inputs.push_back(rtnq::make_toy_input(cfg, i));

    {
        std::ofstream f(dir + "/toy_probe.txt");
        char buf[64];
        for (std::int64_t l = 0; l < cfg.layers; ++l)
            for (rtnq::ModuleId m : rtnq::kAllModules) {
                const rtnq::FloatTensor& w = model.tensor(l, m);
                f << "w " << l << ' ' << static_cast<int>(m);
                for (int i = 0; i < 4; ++i) {
                    std::snprintf(buf, sizeof buf, " %.9g", double(w.data[i]));
                    f << buf;
                }
                f << '\n';
            }
        for (int i = 0; i < n_inputs; ++i) {
            f << "x " << i;
            for (int j = 0; j < 4; ++j) {
                std::snprintf(buf, sizeof buf, " %.9g", double(inputs[i].data[j]));
                f << buf;
            }
            f << '\n';
        }
    }
    {
        std::string csv;
        for (auto kind : {rtnq::HorizontalStrategy::Kind::first, rtnq::HorizontalStrategy::Kind::middle,
                          rtnq::HorizontalStrategy::Kind::last}) {
            const std::string part = rtnq::sweep_to_csv(rtnq::horizontal_sweep(model, kind, inputs));
            csv += csv.empty() ? part : part.substr(part.find('\n') + 1);
        }
        const std::string v = rtnq::sweep_to_csv(rtnq::vertical_sweep(model, inputs));
        csv += v.substr(v.find('\n') + 1);
        std::ofstream(dir + "/toy_sweeps.csv") << csv;
    }
    {
        std::ofstream f(dir + "/toy_compare.txt");
        char buf[128];
        for (const char* text : {"first:0", "first:8", "middle:2 modules:1+3", "explicit:0,7 modules:4"}) {
            const rtnq::SelectionPlan plan = rtnq::parse_plan(text);
            const rtnq::ErrorReport r = rtnq::compare(model, rtnq::quantize_model(model, plan), inputs);
            f << "plan " << text << '\n' << "canonical " << r.plan_text << '\n';
            std::snprintf(buf, sizeof buf, "summary %.17g %.17g %.17g\n", r.effective_bits, r.max_logit_dev,
                          r.mean_kl);
            f << buf;
            for (const rtnq::TensorError& e : r.tensors) {
                std::snprintf(buf, sizeof buf, "tensor %lld %d %.17g %.17g %.17g\n", (long long)e.layer,
                              static_cast<int>(e.module), e.max_abs, e.mse, e.rel_frobenius);
                f << buf;
            }
        }
        const rtnq::ErrorReport self = rtnq::compare(model, model, inputs);
        std::snprintf(buf, sizeof buf, "self %.17g %.17g %.17g\n", self.effective_bits, self.max_logit_dev,
                      self.mean_kl);
        f << buf;
    }
    return 0;
}
