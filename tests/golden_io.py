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


REF_DIRS = ("/root/reference/pkg/src",          # the build container
            os.path.join(os.path.dirname(GOLDEN), "..", "baseline", "_ref"))  # baseline/install_ref.sh


def reference_available():
    """Import the unmodified reference: from /root/reference here, or from
    the baseline/_ref install that travels to the GPU box."""
    try:
        import evotir  # noqa: F401
        return True
    except ImportError:
        for ref in REF_DIRS:
            if os.path.isdir(os.path.join(ref, "evotir")):
                sys_path_add(os.path.abspath(ref))
                try:
                    import evotir  # noqa: F401
                    return True
                except ImportError:
                    continue
        return False


def sys_path_add(p):
    import sys
    if p not in sys.path:
        sys.path.append(p)
