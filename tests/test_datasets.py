"""Dataset readers and device splits (datasets.py:33-81,
149-162, 187-241).

CPU:  the byte readers return exactly the bytes the reference scales (IDX,
      gzip, CSV, error cases); load_dataset's idx/csv sources give the
      reference's float64 x; the CIFAR record layout round-trips.  With the
      reference importable, its own readers are run on the same files.
GPU:  the device decode (gevo_upload_split_u8 / _cifar) equals the host
      float64 split bit for bit, one-hot targets and labels included, and the
      dataset hashes recorded from the reference (tests/golden/meta.json)
      hold for the device split.
"""
import gzip
import hashlib
import os

import numpy as np
import pytest

from golden_io import load, reference_available
from paper_2310_10211_b200 import datasets as D
from paper_2310_10211_b200 import workloads as W


def _write_idx(directory, images, labels, prefix="train", gz=False):
    os.makedirs(directory, exist_ok=True)
    ext = ".gz" if gz else ""
    op = gzip.open if gz else open
    n, r, c = images.shape
    with op(os.path.join(directory, f"{prefix}-images-idx3-ubyte{ext}"), "wb") as f:
        f.write(np.array([0x803, n, r, c], dtype=">u4").tobytes() + images.tobytes())
    with op(os.path.join(directory, f"{prefix}-labels-idx1-ubyte{ext}"), "wb") as f:
        f.write(np.array([0x801, n], dtype=">u4").tobytes() + labels.astype(np.uint8).tobytes())


@pytest.fixture(scope="module")
def digits():
    img, lb = W.synthetic_digits(300, seed=3)
    return img, lb


@pytest.mark.parametrize("gz,prefix", [(False, "train"), (True, "t10k")])
def test_idx_source_matches_synthetic_bytes(tmp_path, digits, gz, prefix):
    img, lb = digits
    _write_idx(str(tmp_path), img, lb, prefix, gz)
    cfg = W.DatasetConfig(source="idx", directory=str(tmp_path), search_n=200, holdout_n=64)
    ds = W.load_dataset(cfg)
    x = img.reshape(300, -1).astype(np.float64) / 255.0
    assert np.array_equal(ds.search.x, x[:200]) and np.array_equal(ds.holdout.x, x[200:264])
    assert np.array_equal(ds.search.raw, img.reshape(300, -1)[:200])
    assert ds.search.labels.dtype == np.int64 and np.array_equal(ds.search.labels, lb[:200])


def test_idx_errors(tmp_path, digits):
    img, lb = digits
    with pytest.raises(D.DatasetError, match="dataset directory not found"):
        D.find_idx_file(str(tmp_path / "nope"), "images-idx3-ubyte")
    with pytest.raises(D.DatasetError, match="no \\*-images-idx3-ubyte file"):
        D.find_idx_file(str(tmp_path), "images-idx3-ubyte")
    bad = tmp_path / "bad-images-idx3-ubyte"
    bad.write_bytes(np.array([0x801, 1, 2, 2], dtype=">u4").tobytes() + b"\0" * 4)
    with pytest.raises(D.DatasetError, match="bad image magic 0x00000801"):
        D.read_idx_images(str(bad))
    short = tmp_path / "short-images-idx3-ubyte"
    short.write_bytes(np.array([0x803, 2, 2, 2], dtype=">u4").tobytes() + b"\0" * 5)
    with pytest.raises(D.DatasetError, match="truncated image data"):
        D.read_idx_images(str(short))
    lab = tmp_path / "l-labels-idx1-ubyte"
    lab.write_bytes(np.array([0x801, 4], dtype=">u4").tobytes() + b"\1\2")
    with pytest.raises(D.DatasetError, match="truncated label data"):
        D.read_idx_labels(str(lab))
    _write_idx(str(tmp_path / "small"), img[:10], lb[:10])
    with pytest.raises(D.DatasetError, match="need 20"):
        W.load_dataset(W.DatasetConfig(source="idx", directory=str(tmp_path / "small"),
                                       search_n=10, holdout_n=10))
    with pytest.raises(D.DatasetError, match="features, expected"):
        W.load_dataset(W.DatasetConfig(source="idx", directory=str(tmp_path / "small"),
                                       search_n=5, holdout_n=5, features=100))


def test_csv_source(tmp_path, digits):
    img, lb = digits
    flat = img.reshape(300, -1)
    p = tmp_path / "d.csv"
    np.savetxt(p, np.concatenate([lb[:, None], flat], axis=1), fmt="%d", delimiter=",")
    ds = W.load_dataset(W.DatasetConfig(source="csv", csv_path=str(p), search_n=250,
                                        holdout_n=50))
    assert ds.search.raw is not None and ds.search.raw.dtype == np.uint8
    assert np.array_equal(ds.search.x, flat[:250].astype(np.float64) / 255.0)
    # non-integer pixels: the float64 table scaled like the reference
    q = tmp_path / "f.csv"
    q.write_text("1,0.5,255\n0,3,7.25\n")
    vals, labels = D.read_csv_dataset(str(q))
    assert vals.dtype == np.float64 and labels.tolist() == [1, 0]
    ds = W.load_dataset(W.DatasetConfig(source="csv", csv_path=str(q), search_n=1,
                                        holdout_n=1, features=2))
    assert ds.search.raw is None
    assert np.array_equal(ds.holdout.x, np.array([[3, 7.25]]) / 255.0)


def test_cifar_records_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    img = rng.integers(0, 256, (37, 32, 32, 3), dtype=np.uint8)
    lb = rng.integers(0, 10, 37)
    D.write_cifar_bin(tmp_path / "a.bin", img[:20], lb[:20])
    D.write_cifar_bin(tmp_path / "b.bin", img[20:], lb[20:])
    rec = D.read_cifar_bin([tmp_path / "a.bin", tmp_path / "b.bin"])
    assert rec.shape == (37, 3073)
    # CHW planes: the first 1024 pixel bytes are the red channel, row-major
    assert np.array_equal(rec[:, 1:1025].reshape(37, 32, 32), img[..., 0])
    x, labels = D.cifar_records_to_nhwc(rec)
    assert np.array_equal(x, img.reshape(37, -1).astype(np.float64) / 255.0)
    assert labels.tolist() == lb.tolist()
    (tmp_path / "c.bin").write_bytes(b"\0" * 3000)
    with pytest.raises(D.DatasetError, match="whole number"):
        D.read_cifar_bin(tmp_path / "c.bin")


def test_pixel_bytes_recovery(digits):
    img, _ = digits
    x = img.reshape(300, -1).astype(np.float64) / 255.0
    assert np.array_equal(D.pixel_bytes(x), img.reshape(300, -1))
    y = x.copy()
    y[3, 5] = np.nextafter(y[3, 5], 2.0)
    assert D.pixel_bytes(y) is None
    assert D.pixel_bytes(np.full((2, 2), 1.5)) is None


@pytest.mark.skipif(not reference_available(), reason="reference package not importable")
def test_readers_match_reference_readers(tmp_path, digits):
    import evotir.datasets as R
    img, lb = digits
    _write_idx(str(tmp_path), img, lb, gz=True)
    ours = W.load_dataset(W.DatasetConfig(source="idx", directory=str(tmp_path),
                                          search_n=100, holdout_n=100))
    ref = R.load_dataset(R.DatasetConfig(source="idx", directory=str(tmp_path),
                                         search_n=100, holdout_n=100))
    for a, b in ((ours.search, ref.search), (ours.holdout, ref.holdout)):
        assert np.array_equal(a.x.view(np.int64), b.x.view(np.int64))
        assert np.array_equal(a.labels, b.labels)
    p = tmp_path / "d.csv"
    np.savetxt(p, np.concatenate([lb[:, None], img.reshape(300, -1)], axis=1), fmt="%d",
               delimiter=",")
    rx, rl = R.read_csv_dataset(str(p))
    vals, labels = D.read_csv_dataset(str(p))
    assert np.array_equal((vals.astype(np.float64) / 255.0).view(np.int64), rx.view(np.int64))
    assert np.array_equal(labels, rl)


# --------------------------------------------------------------------------- GPU

def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.gpu
def test_device_u8_split_bit_exact():
    from paper_2310_10211_b200 import _lib
    from paper_2310_10211_b200.evaluator import upload_split
    ds = W.load_dataset(W.DatasetConfig())
    meta = load("meta.json")
    ctx = _lib.Context(0)
    for sid, split, batch in ((0, ds.search, 32), (1, ds.holdout, 32), (2, ds.search, 7)):
        assert upload_split(ctx, sid, split, 10, batch) == "u8"
        x, y, lb = ctx.download_split(sid, 784, 10, len(split.labels))
        rows = (len(split.labels) // batch) * batch
        assert x.shape[0] == rows
        assert np.array_equal(x.view(np.int64), split.x[:rows].view(np.int64))
        assert np.array_equal(lb, split.labels[:rows])
        want_y = np.zeros((rows, 10))
        want_y[np.arange(rows), split.labels[:rows]] = 1.0
        assert np.array_equal(y, want_y)
    # the reference's dataset hashes hold for the device-decoded splits
    # (one batch of the whole split keeps every row)
    for split, key in ((ds.search, "search"), (ds.holdout, "holdout")):
        n = len(split.labels)
        upload_split(ctx, 3, split, 10, n)
        x, _, lb = ctx.download_split(3, 784, 10, n)
        assert _sha(x) == meta[f"{key}_x_sha"]
        assert _sha(lb) == meta[f"{key}_labels_sha"]
    # a float64 split that is NOT byte-scaled takes the float64 path
    blob = W.SplitView("b", np.random.default_rng(1).random((64, 784)), np.arange(64) % 10)
    assert upload_split(ctx, 3, blob, 10, 32) == "f64"
    x, _, _ = ctx.download_split(3, 784, 10, 64)
    assert np.array_equal(x, blob.x)


@pytest.mark.gpu
def test_device_cifar_split_bit_exact(tmp_path):
    from paper_2310_10211_b200 import _lib, cnn
    from paper_2310_10211_b200.evaluator import upload_split
    rng = np.random.default_rng(2)
    n = 1037
    img = rng.integers(0, 256, (n, 32, 32, 3), dtype=np.uint8)
    lb = rng.integers(0, 10, n)
    D.write_cifar_bin(tmp_path / "data_batch_1.bin", img, lb)
    cfg = cnn.CnnConfig(search_n=1000, holdout_n=37, batch_size=100,
                        cifar_paths=(str(tmp_path / "data_batch_1.bin"),))
    wl = cnn.build_cnn_prediction_workload(cfg)
    ds = wl.dataset
    ctx = _lib.Context(0)
    for sid, split, batch in ((0, ds.search, 100), (1, ds.holdout, 10)):
        assert upload_split(ctx, sid, split, 10, batch) == "cifar"
        x, y, got_lb = ctx.download_split(sid, 3072, 10, len(split.labels))
        rows = (len(split.labels) // batch) * batch
        assert np.array_equal(x.view(np.int64), split.x[:rows].view(np.int64))
        assert np.array_equal(got_lb, split.labels[:rows])
        assert np.array_equal(y.argmax(1), split.labels[:rows]) and y.sum() == rows
    assert np.array_equal(ds.search.x, img[:1000].reshape(1000, -1) / 255.0)
