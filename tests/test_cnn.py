"""CNN prediction workload (new): the network in the
unchanged dialect, pinned to the reference's interpreter and mutation engine
(tests/golden/make_cnn_golden.py), on the oracle (CPU) and on the device."""
import numpy as np
import pytest

from golden_io import load
from oracle import fitness as OF
from paper_2310_10211_b200 import cnn, dialect
from paper_2310_10211_b200.lowering import static_cost


@pytest.fixture(scope="module")
def golden():
    return load("cnn_pop.json.gz")


@pytest.fixture(scope="module")
def wl(golden):
    c = golden["config"]
    return cnn.build_cnn_prediction_workload(
        cnn.CnnConfig(search_n=c["search_n"], holdout_n=c["holdout_n"], batch_size=c["batch_size"]))


def _search(wl):
    cfg = wl.cnn
    xs = wl.search_x.reshape(-1, cfg.batch_size, cfg.side, cfg.side, cfg.in_channels)
    return xs, wl.search_y, wl.search_labels


def test_network_structure(wl):
    fn = wl.module.functions["forward"]
    ops = {op.opcode for op in fn.ops}
    # convolutions, depthwise taps, stride-2 phases, pooling and softmax
    # expressed only in the reference's opcodes
    assert {"pad", "slice", "reshape", "dot", "multiply", "add", "maximum",
            "broadcast_in_dim", "reduce", "exponential", "divide"} <= ops
    assert [t.shape for _, t in fn.params] == [(wl.weights["w"].size,), (10, 32, 32, 3)]
    x, labels = cnn.cifar_synthetic(40)
    assert x.shape == (40, 32, 32, 3) and 0.0 <= x.min() and x.max() <= 1.0
    assert np.bincount(labels).tolist() == [4] * 10


def test_oracle_matches_reference_on_mutants(wl, golden):
    """Static cost and (wrong, total, status) of every recorded variant --
    the unmutated network and reference-made mutants -- bit-exact."""
    search = _search(wl)
    for ind in golden["individuals"]:
        fn = dialect.parse_function(ind["forward"])
        assert static_cost(fn) * len(search[0]) == ind["cost"]
        r = OF.evaluate_variant({"forward": fn}, "prediction", [wl.weights["w"]], search)
        assert (r["cost"], r["wrong"], r["total"], r["status"]) == \
            (ind["cost"], ind["wrong"], ind["total"], ind["status"])


@pytest.mark.gpu
def test_device_matches_reference_on_mutants(wl, golden):
    from paper_2310_10211_b200.evaluator import DeviceEvaluator
    variants = [{"forward": dialect.parse_function(i["forward"])} for i in golden["individuals"]]
    ev = DeviceEvaluator(wl)
    fits, recs = ev.evaluate_variants(variants, return_records=True)
    ev.close()
    exact = 0
    for ind, f, r in zip(golden["individuals"], fits, recs):
        assert f.cost == ind["cost"]
        assert int(r["status"]) == ind["status"]
        exact += (int(r["wrong"]), int(r["total"])) == (ind["wrong"], ind["total"])
        assert f.error == ind["error"], (ind["edits"], f, ind)
    print(f"cnn mutants bit-exact {exact}/{len(fits)}")


# --------------------------------------------------------------------------
# configs[2] at full network size (MobileNetV2-CIFAR width 0.5, batch 100):
# 16 reference-made mutants over 100 images (tests/golden/cnn_full_pop.json.gz,
# make_cnn_golden.py full), with the reference's batch-0 probabilities

@pytest.fixture(scope="module", params=["cnn_full_pop.json.gz", "cnn_full_pop2.json.gz"])
def full_golden(request):
    """The 16 mutants of the first recording, then the further reference-made
    mutants (chains of up to five edits, four seeds) of make_cnn_golden.py
    full2 / merge2."""
    return load(request.param)


@pytest.fixture(scope="module")
def full_wl(full_golden):
    c = full_golden["config"]
    assert c["network"] == "MOBILENETV2_CIFAR_HALF"
    return cnn.build_cnn_prediction_workload(
        cnn.CnnConfig(**cnn.MOBILENETV2_CIFAR_HALF, search_n=c["search_n"],
                      holdout_n=c["holdout_n"], batch_size=c["batch_size"]))


def _probs0(ind):
    import base64
    return np.frombuffer(base64.b64decode(ind["probs0_b64"]), dtype=np.float64).reshape(100, 10)


def test_full_network_mutants_cost_and_oracle(full_wl, full_golden):
    """Static cost of all 16 full-size variants, and the oracle's batch-0
    probabilities for the unmutated network and one mutant, bit-exact."""
    from oracle import interp as OI
    inds = full_golden["individuals"]
    assert len(inds) >= 16 and sum(i["edits"] > 0 for i in inds) >= 15
    keys = [i["key"] for i in inds]
    assert len(set(keys)) == len(keys)
    xb = full_wl.search_x.reshape(-1, 100, 32, 32, 3)[0]
    for k, ind in enumerate(inds):
        fn = dialect.parse_function(ind["forward"])
        assert static_cost(fn) * 1 == ind["cost"]
        if k in (0, 1):
            (p,) = OI.Program(fn)([full_wl.weights["w"], xb])
            assert np.array_equal(p, _probs0(ind))


@pytest.mark.gpu
def test_device_full_network_mutants(full_wl, full_golden):
    """Every full-size mutant on the device: (cost, wrong, total, status)
    through the evaluator and the batch-0 probabilities through
    gevo_exec_once, bit-exact against the reference."""
    from paper_2310_10211_b200 import _lib
    from paper_2310_10211_b200.evaluator import DeviceEvaluator
    from test_gpu_parity import run_once
    inds = full_golden["individuals"]
    fns = [dialect.parse_function(i["forward"]) for i in inds]
    ev = DeviceEvaluator(full_wl)
    fits, recs = ev.evaluate_variants([{"forward": f} for f in fns], return_records=True)
    ev.close()
    for ind, f, r in zip(inds, fits, recs):
        assert f.cost == ind["cost"]
        assert (int(r["status"]), int(r["wrong"]), int(r["total"])) == \
            (ind["status"], ind["wrong"], ind["total"]), ind["edits"]
        assert f.error == ind["error"]
    xb = np.ascontiguousarray(full_wl.search_x.reshape(-1, 100, 32 * 32 * 3)[0]).reshape(-1)
    ctx = _lib.Context(0)
    try:
        outs = run_once(ctx, fns, [[full_wl.weights["w"], xb]] * len(fns))
    finally:
        ctx.close()
    exact = sum(np.array_equal(got, _probs0(ind)) for (got,), ind in zip(outs, inds))
    print(f"full-size cnn mutants: records {len(inds)}/{len(inds)}, batch-0 probabilities "
          f"bit-exact {exact}/{len(inds)}")
    assert exact == len(inds)
