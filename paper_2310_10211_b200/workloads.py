"""Evaluation inputs: synthetic datasets, split batching and the 2fcNet programs.

These are the data formats either side of the evaluator.  Every function
restates the reference so that the GPU box (which has no `evotir`) can
rebuild bit-identical inputs; `tests/test_workloads.py` pins each of them
against the reference and `tests/golden/*` carries the hashes.

* `synthetic_digits`   <- datasets.py:88-109
* `gaussian_blobs`     <- datasets.py:112-120
* `SplitView.whole_batches` <- datasets.py:149-162 (stacked, not a list)
* `DatasetConfig` / `load_dataset` <- datasets.py:173-229 (all four sources;
  the byte readers are in datasets.py of this package)
* `WorkloadConfig`     <- fitness.py:56-68
* `init_weights`       <- fitness.py:218-227
* `two_layer_program`  <- fitness.py:115-215 (same op sequence and names)
* `Fitness`, `INVALID_FITNESS` <- fitness.py:38-48
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .dialect import Module, parse_module

TRAINING = "training"
PREDICTION = "prediction"
WEIGHT_NAMES = ("w1", "b1", "w2", "b2")


@dataclass(frozen=True)
class Fitness:
    """fitness.py:38-45: two minimised objectives plus validity."""
    cost: float
    error: float
    valid: bool = True

    def as_tuple(self):
        return (self.cost, self.error)


INVALID_FITNESS = Fitness(float("inf"), float("inf"), valid=False)


class WorkloadError(Exception):
    pass


# ---------------------------------------------------------------------------
# datasets
# ---------------------------------------------------------------------------

def synthetic_digits(n, seed=7, noise=0.36, separation=0.2, classes=10,
                     side=28):
    """Digit-like uint8 images; same generator stream as datasets.py:88-109."""
    g = np.random.default_rng(seed)
    pixels = side * side
    shared = np.clip(g.standard_normal(pixels), 0.0, None) * 0.25
    per_class = g.standard_normal((classes, pixels))
    protos = np.clip(shared[None, :] + separation * per_class, 0.0, 1.0)
    labels = np.arange(n) % classes
    g.shuffle(labels)
    img = protos[labels] + noise * g.standard_normal((n, pixels))
    img = np.round(np.clip(img, 0.0, 1.0) * 255.0).astype(np.uint8)
    return img.reshape(n, side, side), labels.astype(np.int64)


def gaussian_blobs(n, seed=7, features=784, spread=2.0):
    """Two-class fallback (datasets.py:112-120)."""
    g = np.random.default_rng(seed)
    centers = g.uniform(0.3, 0.7, size=(2, features))
    labels = np.arange(n) % 2
    g.shuffle(labels)
    x = centers[labels] + g.standard_normal((n, features)) / (spread * 10.0)
    return np.clip(x, 0.0, 1.0), labels.astype(np.int64)


@dataclass
class SplitView:
    name: str
    x: np.ndarray
    labels: np.ndarray
    reads: int = 0
    # the pixel bytes x was scaled from (x == raw / 255.0), when the source
    # had them: the device split is then uploaded as bytes and decoded there
    raw: np.ndarray | None = None
    # CIFAR-10 binary records x was decoded from (datasets.read_cifar_bin)
    records: np.ndarray | None = None

    def __len__(self):
        return len(self.labels)

    def stacked_batches(self, batch_size: int, classes: int):
        """All whole batches as stacked arrays (x [nb,B,F], y [nb,B,C],
        labels [nb,B]); the trailing partial batch is dropped exactly as
        whole_batches does (datasets.py:149-162).  Bumps `reads`."""
        self.reads += 1
        nb = len(self.labels) // batch_size
        n = nb * batch_size
        x = np.ascontiguousarray(self.x[:n]).reshape(nb, batch_size, -1)
        lb = np.ascontiguousarray(self.labels[:n]).reshape(nb, batch_size)
        y = np.zeros((nb, batch_size, classes), dtype=np.float64)
        np.put_along_axis(y, lb[..., None], 1.0, axis=2)
        return x, y, lb


@dataclass
class Dataset:
    search: SplitView
    holdout: SplitView
    features: int
    classes: int


@dataclass
class DatasetConfig:
    source: str = "synthetic"
    directory: str | None = None
    csv_path: str | None = None
    search_n: int = 1000
    holdout_n: int = 256
    noise: float = 0.36
    separation: float = 0.2
    data_seed: int = 7
    classes: int = 10
    features: int = 784


def load_dataset(cfg: DatasetConfig) -> Dataset:
    """datasets.py:187-229: synthetic, blobs, idx (train/t10k, optional .gz)
    and csv sources; the same checks and the same float64 x.  Byte sources
    keep their pixels in `SplitView.raw` for the device upload."""
    from . import datasets as D
    total = cfg.search_n + cfg.holdout_n
    raw = None
    if cfg.source == "synthetic":
        side = int(round(cfg.features ** 0.5))
        if side * side != cfg.features:
            raise D.DatasetError("synthetic digits need a square feature count")
        img, labels = synthetic_digits(total, cfg.data_seed, cfg.noise,
                                       cfg.separation, cfg.classes, side)
        raw = img.reshape(total, -1)
    elif cfg.source == "blobs":
        x, labels = gaussian_blobs(total, cfg.data_seed, cfg.features)
        if cfg.classes != 2:
            raise D.DatasetError("blobs is a two-class dataset")
    elif cfg.source == "idx":
        if not cfg.directory:
            raise D.DatasetError("idx source needs a dataset directory")
        images_path = D.find_idx_file(cfg.directory, "images-idx3-ubyte")
        labels_path = D.find_idx_file(cfg.directory, "labels-idx1-ubyte")
        raw = D.read_idx_images(images_path)
        labels = D.read_idx_labels(labels_path)
    elif cfg.source == "csv":
        if not cfg.csv_path:
            raise D.DatasetError("csv source needs csv_path")
        vals, labels = D.read_csv_dataset(cfg.csv_path)
        if vals.dtype == np.uint8:
            raw = vals
        else:
            x = vals / 255.0
    else:
        raise D.DatasetError(f"unknown dataset source {cfg.source!r}")
    if raw is not None:
        x = raw.astype(np.float64) / 255.0
    if len(labels) < total:
        raise D.DatasetError(f"dataset has {len(labels)} examples, need {total} "
                             f"(search {cfg.search_n} + holdout {cfg.holdout_n})")
    if x.shape[1] != cfg.features:
        raise D.DatasetError(f"dataset has {x.shape[1]} features, expected {cfg.features}")
    cut = (lambda a, lo, hi: None if a is None else a[lo:hi])
    return Dataset(SplitView("search", x[:cfg.search_n], labels[:cfg.search_n],
                             raw=cut(raw, 0, cfg.search_n)),
                   SplitView("holdout", x[cfg.search_n:total], labels[cfg.search_n:total],
                             raw=cut(raw, cfg.search_n, total)),
                   cfg.features, cfg.classes)


# ---------------------------------------------------------------------------
# the two-layer programs
# ---------------------------------------------------------------------------

@dataclass
class WorkloadConfig:
    features: int = 784
    hidden: int = 32
    classes: int = 10
    batch_size: int = 32
    steps: int = 600
    learning_rate: float = 0.01
    init_seed: int = 1234
    finite_check_every: int = 50
    dataset: DatasetConfig = field(default_factory=DatasetConfig)
    cost_table: dict = field(default_factory=dict)
    weights_path: str | None = None


def init_weights(cfg: WorkloadConfig) -> dict:
    """U(-0.05, 0.05) draws in w1, b1, w2, b2 order (fitness.py:218-227)."""
    g = np.random.default_rng(cfg.init_seed)
    d, h, c = cfg.features, cfg.hidden, cfg.classes
    out = {}
    for name, shape in (("w1", (d, h)), ("b1", (h,)), ("w2", (h, c)),
                        ("b2", (c,))):
        out[name] = g.uniform(-0.05, 0.05, size=shape)
    return out


def _t(*dims):
    return "tensor<" + "".join(f"{d}x" for d in dims) + "f32>"


def _forward_lines(b, h, c):
    bh, bc = _t(b, h), _t(b, c)
    return [
        f"%0 = dot %x, %w1 : {bh}",
        f"%1 = broadcast_in_dim %b1 {{dims = [1]}} : {bh}",
        f"%2 = add %0, %1 : {bh}",
        f"%3 = constant dense<0.0> : {_t()}",
        f"%4 = broadcast_in_dim %3 {{dims = []}} : {bh}",
        f"%5 = maximum %2, %4 : {bh}",
        f"%6 = dot %5, %w2 : {bc}",
        f"%7 = broadcast_in_dim %b2 {{dims = [1]}} : {bc}",
        f"%8 = add %6, %7 : {bc}",
        f"%9 = reduce %8 {{axis = 1, kind = max}} : {_t(b)}",
        f"%10 = broadcast_in_dim %9 {{dims = [0]}} : {bc}",
        f"%11 = subtract %8, %10 : {bc}",
        f"%12 = exponential %11 : {bc}",
        f"%13 = reduce %12 {{axis = 1, kind = sum}} : {_t(b)}",
        f"%14 = broadcast_in_dim %13 {{dims = [0]}} : {bc}",
        f"%15 = divide %12, %14 : {bc}",
    ]


def _sgd_lines(b, d, h, c, inv_b, lr):
    bh, bc, dh, hc = _t(b, h), _t(b, c), _t(d, h), _t(h, c)
    lines = [
        f"%16 = subtract %15, %y : {bc}",
        f"%17 = constant dense<{inv_b}> : {_t()}",
        f"%18 = broadcast_in_dim %17 {{dims = []}} : {bc}",
        f"%19 = multiply %16, %18 : {bc}",
        f"%20 = transpose %5 {{perm = [1, 0]}} : {_t(h, b)}",
        f"%21 = dot %20, %19 : {hc}",
        f"%22 = reduce %19 {{axis = 0, kind = sum}} : {_t(c)}",
        f"%23 = transpose %w2 {{perm = [1, 0]}} : {_t(c, h)}",
        f"%24 = dot %19, %23 : {bh}",
        f"%25 = compare %2, %4 {{kind = gt}} : tensor<{b}x{h}xi1>",
        f"%26 = select %25, %24, %4 : {bh}",
        f"%27 = transpose %x {{perm = [1, 0]}} : {_t(d, b)}",
        f"%28 = dot %27, %26 : {dh}",
        f"%29 = reduce %26 {{axis = 0, kind = sum}} : {_t(h)}",
        f"%30 = constant dense<{lr}> : {_t()}",
    ]
    # SGD update of every weight: w - lr * grad, one broadcast per shape
    nxt = 31
    for w, grad, ty in (("%w1", "%28", dh), ("%b1", "%29", _t(h)),
                        ("%w2", "%21", hc), ("%b2", "%22", _t(c))):
        lines += [f"%{nxt} = broadcast_in_dim %30 {{dims = []}} : {ty}",
                  f"%{nxt + 1} = multiply {grad}, %{nxt} : {ty}",
                  f"%{nxt + 2} = subtract {w}, %{nxt + 1} : {ty}"]
        nxt += 3
    return lines


def _dense(a) -> str:
    a = np.asarray(a)
    if a.ndim == 0:
        return repr(float(a))
    return "[" + ", ".join(_dense(r) for r in a) + "]"


def _globals(cfg, weights):
    d, h, c = cfg.features, cfg.hidden, cfg.classes
    shapes = {"w1": (d, h), "b1": (h,), "w2": (h, c), "b2": (c,)}
    return [f"global @{n} = dense<{_dense(weights[n])}> : {_t(*shapes[n])}"
            for n in WEIGHT_NAMES]


def two_layer_program(cfg: WorkloadConfig, weights: dict,
                      training: bool = True) -> str:
    """Module text of the 2fcNet workload: @forward, and for training also
    @train_step and @loss.  Byte-identical to build_2fcnet_text
    (fitness.py:141-215) and the prediction text (fitness.py:274-287)."""
    b, d, h, c = cfg.batch_size, cfg.features, cfg.hidden, cfg.classes
    wparams = (f"%w1: {_t(d, h)}, %b1: {_t(h)}, %w2: {_t(h, c)}, "
               f"%b2: {_t(c)}")
    fwd = ["  " + s for s in _forward_lines(b, h, c)]
    out = _globals(cfg, weights) + [""]
    out += [f"func @forward({wparams}, %x: {_t(b, d)}) -> {_t(b, c)} {{"]
    out += fwd + [f"  return %15 : {_t(b, c)}", "}"]
    if not training:
        return "\n".join(out + [""])
    inv_b, lr = repr(float(1.0 / b)), repr(float(cfg.learning_rate))
    out += ["", f"func @train_step({wparams}, %x: {_t(b, d)}, %y: {_t(b, c)}) "
            f"-> ({_t(d, h)}, {_t(h)}, {_t(h, c)}, {_t(c)}) {{"]
    out += fwd + ["  " + s for s in _sgd_lines(b, d, h, c, inv_b, lr)]
    out += [f"  return %33, %36, %39, %42 : {_t(d, h)}, {_t(h)}, "
            f"{_t(h, c)}, {_t(c)}", "}", ""]
    out += [f"func @loss({wparams}, %x: {_t(b, d)}, %y: {_t(b, c)}) -> {_t()} {{"]
    out += fwd + ["  " + s for s in (
        f"%16 = log %15 : {_t(b, c)}",
        f"%17 = multiply %y, %16 : {_t(b, c)}",
        f"%18 = reduce %17 {{axis = 1, kind = sum}} : {_t(b)}",
        f"%19 = reduce %18 {{axis = 0, kind = sum}} : {_t()}",
        f"%20 = negate %19 : {_t()}",
        f"%21 = constant dense<{inv_b}> : {_t()}",
        f"%22 = multiply %20, %21 : {_t()}")]
    out += [f"  return %22 : {_t()}", "}", ""]
    return "\n".join(out)


@dataclass
class Workload:
    """The evaluation protocol of fitness.py:71-99, device-oriented: batches
    are stacked arrays ready for a single upload."""
    name: str
    mode: str
    module: Module
    mutable_functions: list
    dataset: Dataset
    config: WorkloadConfig
    weights: dict            # initial (training) or frozen (prediction)
    search_x: np.ndarray = None
    search_y: np.ndarray = None
    search_labels: np.ndarray = None

    @property
    def n_search_batches(self) -> int:
        return 0 if self.search_x is None else len(self.search_x)

    def holdout_batches(self):
        return self.dataset.holdout.stacked_batches(self.config.batch_size,
                                                    self.config.classes)


def build_2fcnet_workload(cfg: WorkloadConfig | None = None) -> Workload:
    """fitness.py:230-245."""
    cfg = cfg or WorkloadConfig()
    ds = load_dataset(cfg.dataset)
    w = init_weights(cfg)
    module = parse_module(two_layer_program(cfg, w, training=True))
    wl = Workload("train2fc", TRAINING, module, ["forward", "train_step"],
                  ds, cfg, {n: module.constants[n] for n in WEIGHT_NAMES})
    wl.search_x, wl.search_y, wl.search_labels = ds.search.stacked_batches(
        cfg.batch_size, cfg.classes)
    if wl.n_search_batches == 0:
        raise WorkloadError("search split smaller than one batch")
    return wl


def build_prediction_workload(cfg: WorkloadConfig | None = None,
                              weights: dict | None = None) -> Workload:
    """fitness.py:248-296.  Frozen weights come from `weights`, from
    cfg.weights_path (.npz with w1/b1/w2/b2), or -- like the reference --
    from training the baseline 2fcNet once (on the device evaluator)."""
    cfg = cfg or WorkloadConfig()
    if weights is None and cfg.weights_path is not None:
        try:
            arc = np.load(cfg.weights_path)
        except OSError as e:
            raise WorkloadError(f"weights file not found: {cfg.weights_path}") from e
        weights = {n: np.asarray(arc[n], dtype=np.float64) for n in WEIGHT_NAMES}
    if weights is None:
        from .evaluator import train_baseline_weights
        weights = train_baseline_weights(build_2fcnet_workload(cfg))
    ds = load_dataset(cfg.dataset)
    module = parse_module(two_layer_program(cfg, weights, training=False))
    wl = Workload("predict2fc", PREDICTION, module, ["forward"], ds, cfg,
                  {n: module.constants[n] for n in WEIGHT_NAMES})
    wl.search_x, wl.search_y, wl.search_labels = ds.search.stacked_batches(
        cfg.batch_size, cfg.classes)
    if wl.n_search_batches == 0:
        raise WorkloadError("search split smaller than one batch")
    return wl
