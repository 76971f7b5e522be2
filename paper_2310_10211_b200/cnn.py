"""CNN prediction workload on CIFAR-shaped data.

NEW -- not in the reference.  The paper's second model is a MobileNet run
for prediction; the reference restatement (`evotir`) has no
convolution opcode and only square single-channel synthetic images.  This
module writes a MobileNetV2-style network in the reference's UNCHANGED
dialect, so the unchanged mutation engine, interpreter (the oracle) and the
device executor all apply:

  3x3 conv, stride 1   pad (low/high 1 on H, W) -> 9 x (slice -> reshape
                       [B*H*W, Cin] -> dot [Cin, Cout]) -> 8 adds
  1x1 conv             reshape [B*H*W, C] -> dot -> reshape
  depthwise 3x3        pad -> 9 x (slice * broadcast(w_tap [C], dims=[3]))
                       -> 8 adds
  stride 2             reshape [B, H/2, 2, W/2, 2, C] -> slice the (0, 0)
                       phase -> reshape [B, H/2, W/2, C]
  folded batch norm    multiply by broadcast scale [C], add broadcast bias
  ReLU                 maximum with a broadcast 0
  global average pool  reshape [B, H*W, C] -> reduce sum axis 1 -> * 1/(H*W)
  classifier           dot [C, classes] + bias -> softmax (as 2fcNet)

Weights are frozen (prediction mode) and passed as ONE flat parameter
%w: every tensor is a `slice` of it `reshape`d to shape -- views, so the
device reads them in place and the per-instruction parameter count stays
small.  `forward(%w, %x) -> probs [B, classes]`; the evaluation protocol
(argmax error over whole batches, non-finite -> 1.0, cost = static cost x
batches) is the reference's prediction mode (fitness.py:248-296,355-393).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .dialect import parse_module
from .workloads import (PREDICTION, Dataset, SplitView, Workload,
                        WorkloadConfig, WorkloadError)


@dataclass
class CnnConfig:
    side: int = 32                 # image H = W
    in_channels: int = 3
    classes: int = 10
    stem: int = 16                 # 3x3 stem conv output channels
    # inverted-residual blocks: (expansion, out channels, stride)
    blocks: tuple = ((1, 8, 1), (4, 12, 2), (4, 12, 1), (4, 16, 2))
    head: int = 32                 # final 1x1 conv before pooling
    batch_size: int = 10
    search_n: int = 100
    holdout_n: int = 20
    data_seed: int = 11
    init_seed: int = 4321
    cost_table: dict = field(default_factory=dict)
    # CIFAR-10 binary batch files (datasets.read_cifar_bin) instead of the
    # synthetic images: search = the first search_n records, holdout the next
    cifar_paths: tuple = ()


# MobileNetV2-CIFAR (width multiplier 0.5): the BASELINE.json configs[2]
# network shape -- GPU-only scale in float64
MOBILENETV2_CIFAR_HALF = dict(
    stem=16, head=640,
    blocks=((1, 8, 1), (6, 12, 1), (6, 12, 1), (6, 16, 2), (6, 16, 1), (6, 16, 1),
            (6, 32, 2), (6, 32, 1), (6, 32, 1), (6, 32, 1), (6, 48, 1), (6, 48, 1),
            (6, 48, 1), (6, 80, 2), (6, 80, 1), (6, 80, 1), (6, 160, 1)))


def cifar_synthetic(n, seed=11, side=32, channels=3, classes=10):
    """CIFAR-shaped synthetic images [n, side, side, channels] in [0, 1]:
    smooth per-class colour/texture prototypes plus noise, quantised to
    8 bits like real pixels; labels arange(n) % classes, shuffled."""
    g = np.random.default_rng(seed)
    yy, xx = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    protos = []
    for c in range(classes):
        fy, fx = g.uniform(0.5, 3.0, size=2)
        phase = g.uniform(0, 2 * np.pi, size=channels)
        colour = g.uniform(0.2, 0.8, size=channels)
        base = np.sin(2 * np.pi * (fy * yy + fx * xx) / side)[..., None]
        protos.append(np.clip(colour + 0.25 * np.sin(base * 3 + phase), 0, 1))
    protos = np.stack(protos)
    labels = np.arange(n) % classes
    g.shuffle(labels)
    img = protos[labels] + 0.15 * g.standard_normal((n, side, side, channels))
    img = np.round(np.clip(img, 0.0, 1.0) * 255.0) / 255.0
    return img.astype(np.float64), labels.astype(np.int64)


class _Prog:
    """SSA text builder for one function."""

    def __init__(self):
        self.lines = []
        self.n = 0
        self.weights = []          # (shape, array) in flat order
        self.off = 0

    @staticmethod
    def t(shape):
        return "tensor<" + "".join(f"{d}x" for d in shape) + "f32>"

    def emit(self, text, shape):
        name = f"%{self.n}"
        self.n += 1
        self.lines.append(f"  {name} = {text} : {self.t(shape)}")
        return name

    def const(self, v):
        return self.emit(f"constant dense<{float(v)!r}>", ())

    def weight(self, arr):
        arr = np.asarray(arr, dtype=np.float64)
        size = arr.size
        s = self.emit(f"slice %w {{start = [{self.off}], limit = [{self.off + size}]}}", (size,))
        self.off += size
        self.weights.append(arr)
        return s if arr.ndim == 1 else self.emit(f"reshape {s}", arr.shape)

    def bcast(self, v, dims, shape):
        d = "[" + ", ".join(str(x) for x in dims) + "]"
        return self.emit(f"broadcast_in_dim {v} {{dims = {d}}}", shape)


def _he(g, fan_in, shape):
    return g.standard_normal(shape) * np.sqrt(2.0 / fan_in)


def cnn_forward_text(cfg: CnnConfig):
    """(module text, flat weights) of the network for batch cfg.batch_size."""
    g = np.random.default_rng(cfg.init_seed)
    P = _Prog()
    B, S = cfg.batch_size, cfg.side
    zero = P.const(0.0)

    def bn_relu(v, shape, relu=True):
        C = shape[-1]
        scale = P.weight(g.uniform(0.8, 1.2, size=C))
        bias = P.weight(g.uniform(-0.05, 0.05, size=C))
        v = P.emit(f"multiply {v}, {P.bcast(scale, [3], shape)}", shape)
        v = P.emit(f"add {v}, {P.bcast(bias, [3], shape)}", shape)
        if relu:
            v = P.emit(f"maximum {v}, {P.bcast(zero, [], shape)}", shape)
        return v

    def padded(v, shape):
        Bn, H, W, C = shape
        return P.emit(f"pad {v}, {zero} {{low = [0, 1, 1, 0], high = [0, 1, 1, 0]}}",
                      (Bn, H + 2, W + 2, C)), (Bn, H + 2, W + 2, C)

    def conv3x3(v, shape, cout):
        Bn, H, W, C = shape
        p, _ = padded(v, shape)
        w = _he(g, 9 * C, (3, 3, C, cout))
        acc = None
        for dy in range(3):
            for dx in range(3):
                tap = P.emit(f"slice {p} {{start = [0, {dy}, {dx}, 0], "
                             f"limit = [{Bn}, {dy + H}, {dx + W}, {C}]}}", (Bn, H, W, C))
                flat = P.emit(f"reshape {tap}", (Bn * H * W, C))
                prod = P.emit(f"dot {flat}, {P.weight(w[dy, dx])}", (Bn * H * W, cout))
                acc = prod if acc is None else P.emit(f"add {acc}, {prod}", (Bn * H * W, cout))
        out = (Bn, H, W, cout)
        return P.emit(f"reshape {acc}", out), out

    def conv1x1(v, shape, cout):
        Bn, H, W, C = shape
        flat = P.emit(f"reshape {v}", (Bn * H * W, C))
        prod = P.emit(f"dot {flat}, {P.weight(_he(g, C, (C, cout)))}", (Bn * H * W, cout))
        out = (Bn, H, W, cout)
        return P.emit(f"reshape {prod}", out), out

    def depthwise(v, shape):
        Bn, H, W, C = shape
        p, _ = padded(v, shape)
        w = _he(g, 9, (3, 3, C))
        acc = None
        for dy in range(3):
            for dx in range(3):
                tap = P.emit(f"slice {p} {{start = [0, {dy}, {dx}, 0], "
                             f"limit = [{Bn}, {dy + H}, {dx + W}, {C}]}}", shape)
                prod = P.emit(f"multiply {tap}, {P.bcast(P.weight(w[dy, dx]), [3], shape)}", shape)
                acc = prod if acc is None else P.emit(f"add {acc}, {prod}", shape)
        return acc

    def stride2(v, shape):
        Bn, H, W, C = shape
        six = (Bn, H // 2, 2, W // 2, 2, C)
        r = P.emit(f"reshape {v}", six)
        s = P.emit(f"slice {r} {{start = [0, 0, 0, 0, 0, 0], "
                   f"limit = [{Bn}, {H // 2}, 1, {W // 2}, 1, {C}]}}", (Bn, H // 2, 1, W // 2, 1, C))
        out = (Bn, H // 2, W // 2, C)
        return P.emit(f"reshape {s}", out), out

    shape = (B, S, S, cfg.in_channels)
    v, shape = conv3x3("%x", shape, cfg.stem)
    v = bn_relu(v, shape)
    for expand, cout, stride in cfg.blocks:
        cin = shape[-1]
        inp, ishape = v, shape
        h, hshape = (conv1x1(v, shape, cin * expand) if expand != 1 else (v, shape))
        if expand != 1:
            h = bn_relu(h, hshape)
        h = depthwise(h, hshape)
        h = bn_relu(h, hshape)
        if stride == 2:
            h, hshape = stride2(h, hshape)
        h, oshape = conv1x1(h, hshape, cout)
        h = bn_relu(h, oshape, relu=False)
        if stride == 1 and cin == cout:
            h = P.emit(f"add {h}, {inp}", oshape)
        v, shape = h, oshape
    v, shape = conv1x1(v, shape, cfg.head)
    v = bn_relu(v, shape)
    Bn, H, W, C = shape
    r = P.emit(f"reshape {v}", (Bn, H * W, C))
    pooled = P.emit(f"reduce {r} {{axis = 1, kind = sum}}", (Bn, C))
    inv = P.const(1.0 / (H * W))
    pooled = P.emit(f"multiply {pooled}, {P.bcast(inv, [], (Bn, C))}", (Bn, C))
    K = cfg.classes
    logits = P.emit(f"dot {pooled}, {P.weight(_he(g, C, (C, K)))}", (Bn, K))
    logits = P.emit(f"add {logits}, {P.bcast(P.weight(np.zeros(K)), [1], (Bn, K))}", (Bn, K))
    mx = P.emit(f"reduce {logits} {{axis = 1, kind = max}}", (Bn,))
    sh = P.emit(f"subtract {logits}, {P.bcast(mx, [0], (Bn, K))}", (Bn, K))
    ex = P.emit(f"exponential {sh}", (Bn, K))
    sm = P.emit(f"reduce {ex} {{axis = 1, kind = sum}}", (Bn,))
    probs = P.emit(f"divide {ex}, {P.bcast(sm, [0], (Bn, K))}", (Bn, K))
    flat = np.concatenate([w.reshape(-1) for w in P.weights])
    head = (f"func @forward(%w: {P.t((flat.size,))}, %x: {P.t((B, S, S, cfg.in_channels))}) "
            f"-> {P.t((B, K))} {{")
    text = "\n".join([head] + P.lines + [f"  return {probs} : {P.t((B, K))}", "}", ""])
    return text, flat


def build_cnn_prediction_workload(cfg: CnnConfig | None = None) -> Workload:
    """The CNN prediction workload (mode prediction, mutable ['forward']).
    The flat weight vector is the single weight parameter; images are
    flattened per example ([n, side*side*channels], NHWC order) so the
    generic split upload applies."""
    cfg = cfg or CnnConfig()
    total = cfg.search_n + cfg.holdout_n
    records = None
    if cfg.cifar_paths:
        from . import datasets as D
        if (cfg.side, cfg.in_channels, cfg.classes) != (D.CIFAR_SIDE, D.CIFAR_CHANNELS, 10):
            raise WorkloadError("CIFAR-10 records are 32x32x3 with 10 classes")
        records = D.read_cifar_bin(cfg.cifar_paths)
        if len(records) < total:
            raise WorkloadError(f"dataset has {len(records)} examples, need {total}")
        records = records[:total]
        x, labels = D.cifar_records_to_nhwc(records)
    else:
        x, labels = cifar_synthetic(total, cfg.data_seed, cfg.side, cfg.in_channels,
                                    cfg.classes)
    x = x.reshape(total, -1)
    cut = (lambda a, lo, hi: None if a is None else a[lo:hi])
    ds = Dataset(SplitView("search", x[:cfg.search_n], labels[:cfg.search_n],
                           records=cut(records, 0, cfg.search_n)),
                 SplitView("holdout", x[cfg.search_n:total], labels[cfg.search_n:total],
                           records=cut(records, cfg.search_n, total)),
                 x.shape[1], cfg.classes)
    text, flat = cnn_forward_text(cfg)
    module = parse_module(text)
    wcfg = WorkloadConfig(features=x.shape[1], classes=cfg.classes, batch_size=cfg.batch_size,
                          steps=0, cost_table=cfg.cost_table)
    wl = Workload("predictcnn", PREDICTION, module, ["forward"], ds, wcfg, {"w": flat})
    wl.search_x, wl.search_y, wl.search_labels = ds.search.stacked_batches(cfg.batch_size, cfg.classes)
    if wl.n_search_batches == 0:
        raise WorkloadError("search split smaller than one batch")
    wl.cnn = cfg
    return wl
