"""§8f4: the selective-precision eval harness (eval.cpp:147-243) on the GPU linears, against
the reference's own outputs (tests/golden/toy_sweeps.csv, toy_compare.txt, toy_probe.txt,
written by oracle/_ref/make_sweep from /root/reference sources; make_sweep_golden.py)."""
import csv
import io
import os

import numpy as np
import pytest

from paper_2505_15909_b200 import eval as ev

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CFG = ev.ToyConfig()
N_INPUTS = 2
RTOL = 1e-6  # same linears bit for bit; torch's f64 reductions reorder the norm/attention sums


def golden_rows():
    with open(os.path.join(GOLDEN, "toy_sweeps.csv")) as f:
        return list(csv.DictReader(f))


def golden_compare():
    reports, cur = {}, None
    for line in open(os.path.join(GOLDEN, "toy_compare.txt")):
        f = line.split()
        if f[0] == "plan":
            cur = reports.setdefault(line[5:].strip(), {"tensors": []})
        elif f[0] == "canonical":
            cur["canonical"] = line[10:].strip()
        elif f[0] == "summary":
            cur["summary"] = tuple(float(v) for v in f[1:])
        elif f[0] == "tensor":
            cur["tensors"].append((int(f[1]), int(f[2])) + tuple(float(v) for v in f[3:]))
        elif f[0] == "self":
            reports["<self>"] = {"summary": tuple(float(v) for v in f[1:])}
    return reports


def test_prng_matches_reference_probe():
    """make_toy_weight / make_toy_input (toy.cpp:155-185) bit for bit: the first values of
    every tensor and input the reference generated."""
    for line in open(os.path.join(GOLDEN, "toy_probe.txt")):
        f = line.split()
        if f[0] == "w":
            got = ev.toy_weight(CFG, int(f[1]), int(f[2])).ravel()[:4]
            want = np.array([float(v) for v in f[3:]], np.float32)
        else:
            got = ev.toy_input(CFG, int(f[1])).ravel()[:4]
            want = np.array([float(v) for v in f[2:]], np.float32)
        assert np.array_equal(got, want), line


def test_sweep_plans_and_effective_bits_match_reference():
    """The plan text each sweep point uses resolves to the reference's effective bits exactly
    (plan grammar + resolve_plan + effective_bits through the C-ABI, CPU only)."""
    from paper_2505_15909_b200 import plan
    rows = golden_rows()
    assert len(rows) == 3 * (CFG.layers + 1) + 16
    for r in rows:
        text = (f"first:{CFG.layers} modules:{r['x_or_mask']}" if r["strategy"] == "modules"
                else f"{r['strategy']}:{r['x_or_mask']}")
        table, _ = plan.resolve(text, CFG.layers)
        assert f"{ev.effective_bits(table, CFG):.9g}" == r["effective_bits"], text
    assert [ev.mask_label(m) for m in range(16)] == [r["x_or_mask"] for r in rows[-16:]]


def test_sweep_to_csv_format():
    rows = [ev.SweepRow("first", "0", 4.0, 2.537617444992, 0.1682944323), ev.SweepRow("modules", "none", 4, 0, 0)]
    assert ev.sweep_to_csv(rows) == ("strategy,x_or_mask,effective_bits,max_logit_dev,mean_kl\n"
                                     "first,0,4,2.53761744,0.168294432\nmodules,none,4,0,0\n")


@pytest.mark.gpu
def test_gpu_sweeps_match_reference():
    torch = pytest.importorskip("torch")
    assert torch.cuda.is_available()
    model = ev.FloatModel(CFG)
    inputs = [ev.toy_input(CFG, i) for i in range(N_INPUTS)]
    rows = []
    for kind in ("first", "middle", "last"):
        rows += ev.horizontal_sweep(model, kind, inputs)
    rows += ev.vertical_sweep(model, inputs)
    got = list(csv.DictReader(io.StringIO(ev.sweep_to_csv(rows))))
    want = golden_rows()
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert (g["strategy"], g["x_or_mask"], g["effective_bits"]) == (w["strategy"], w["x_or_mask"], w["effective_bits"])
        for key in ("max_logit_dev", "mean_kl"):
            assert float(g[key]) == pytest.approx(float(w[key]), rel=RTOL, abs=1e-12), (w, g)


@pytest.mark.gpu
def test_gpu_compare_matches_reference():
    torch = pytest.importorskip("torch")
    assert torch.cuda.is_available()
    model = ev.FloatModel(CFG)
    inputs = [ev.toy_input(CFG, i) for i in range(N_INPUTS)]
    gold = golden_compare()
    for text, want in gold.items():
        if text == "<self>":
            r = ev.compare(model, model, inputs)
            assert (r.effective_bits, r.max_logit_dev, r.mean_kl) == (32.0, 0.0, 0.0)
            assert want["summary"] == (32.0, 0.0, 0.0)
            continue
        r = ev.compare(model, ev.QuantModel(model, text), inputs)
        assert r.plan_text == want["canonical"]
        eb, dev, kl = want["summary"]
        assert r.effective_bits == eb
        assert r.max_logit_dev == pytest.approx(dev, rel=RTOL)
        assert r.mean_kl == pytest.approx(kl, rel=RTOL)
        assert len(r.tensors) == len(want["tensors"])
        for t, (l, m, mx, mse, rf) in zip(r.tensors, want["tensors"]):
            assert (t.layer, t.module) == (l, m)
            assert t.max_abs == mx  # dequantized weights are exact: same max bit for bit
            assert t.mse == pytest.approx(mse, rel=1e-12)
            assert t.rel_frobenius == pytest.approx(rf, rel=1e-12)
