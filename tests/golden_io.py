"""Readers for tests/golden/* (written by tests/golden/make_golden.py)."""
import base64
import gzip
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    path = os.path.join(GOLDEN, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rt") as f:
            return json.load(f)
    with open(path) as f:
        return json.load(f)


def dec(d):
    a = np.frombuffer(base64.b64decode(d["b64"]), dtype=np.dtype(d["dtype"]))
    return a.reshape(d["shape"]).copy()


def variant_functions(ind, names=("forward", "train_step")):
    from paper_2310_10211_b200.dialect import parse_function
    if ind.get("invalid_patch"):
        return None
    return {n: parse_function(ind[n]) for n in names if n in ind}


def predict_weights():
    arc = np.load(os.path.join(GOLDEN, "predict_weights.npz"))
    return {n: arc[n] for n in ("w1", "b1", "w2", "b2")}


def reference_available():
    try:
        import evotir  # noqa: F401
        return True
    except ImportError:
        ref = "/root/reference/pkg/src"
        if os.path.isdir(ref):
            sys_path_add(ref)
            try:
                import evotir  # noqa: F401
                return True
            except ImportError:
                return False
        return False


def sys_path_add(p):
    import sys
    if p not in sys.path:
        sys.path.append(p)
