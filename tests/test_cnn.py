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
