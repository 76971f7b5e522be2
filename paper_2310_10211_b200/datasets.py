"""Dataset readers that keep pixels as bytes for the device.

The reference reads every source into float64 on the host (datasets.py:33-81,
187-229).  These readers stop at the raw bytes, with the reference's checks
and error messages.  The scaling (u8 / 255.0), the one-hot targets and the
NHWC reordering of CIFAR records then run on the device
(gevo_upload_split_u8 / gevo_upload_split_cifar, csrc/splits.cu), so a split
crosses PCIe at 1 byte per pixel:

* `read_idx_images`  <- datasets.py:33-45 (magic 0x00000803, gzip optional)
* `read_idx_labels`  <- datasets.py:48-58 (magic 0x00000801)
* `read_csv_dataset` <- datasets.py:76-81 (label first, pixels 0..255)
* `find_idx_file`    <- datasets.py:232-241 (train/t10k, optional .gz)
* `read_cifar_bin`   (new: CIFAR-10 binary batches for the CNN workload A24)
* `pixel_bytes`      recovers the bytes of an already-scaled float64 split
                     (evotir's SplitView.x), only when that is exact
"""
from __future__ import annotations

import gzip
import os
import struct

import numpy as np

IDX_IMAGES_MAGIC = 0x00000803
IDX_LABELS_MAGIC = 0x00000801
CIFAR_SIDE, CIFAR_CHANNELS = 32, 3
CIFAR_RECORD = 1 + CIFAR_CHANNELS * CIFAR_SIDE * CIFAR_SIDE


class DatasetError(Exception):
    pass


def _open(path, mode="rb"):
    return gzip.open(path, mode) if path.endswith(".gz") else open(path, mode)


def read_idx_images(path: str) -> np.ndarray:
    """IDX3 images as uint8 (n, rows*cols); the reference's float64 x is
    this / 255.0."""
    with _open(path) as f:
        head = f.read(16)
        if len(head) < 16:
            raise DatasetError(f"{path}: truncated image header")
        magic, n, rows, cols = struct.unpack(">IIII", head)
        if magic != IDX_IMAGES_MAGIC:
            raise DatasetError(f"{path}: bad image magic 0x{magic:08x}, "
                               f"expected 0x{IDX_IMAGES_MAGIC:08x}")
        raw = f.read(n * rows * cols)
    if len(raw) != n * rows * cols:
        raise DatasetError(f"{path}: truncated image data")
    return np.frombuffer(raw, dtype=np.uint8).reshape(n, rows * cols)


def read_idx_labels(path: str) -> np.ndarray:
    with _open(path) as f:
        head = f.read(8)
        if len(head) < 8:
            raise DatasetError(f"{path}: truncated label header")
        magic, n = struct.unpack(">II", head)
        if magic != IDX_LABELS_MAGIC:
            raise DatasetError(f"{path}: bad label magic 0x{magic:08x}, "
                               f"expected 0x{IDX_LABELS_MAGIC:08x}")
        raw = f.read(n)
    if len(raw) != n:
        raise DatasetError(f"{path}: truncated label data")
    return np.frombuffer(raw, dtype=np.uint8).astype(np.int64)


def read_csv_dataset(path: str):
    """(pixels, labels).  pixels are uint8 when every value is an integer in
    0..255 (then pixels / 255.0 is the reference's x bit for bit), else the
    float64 table values, which the caller scales like the reference."""
    table = np.loadtxt(path, delimiter=",", dtype=np.float64, ndmin=2)
    labels = table[:, 0].astype(np.int64)
    vals = table[:, 1:]
    if vals.size and np.all((vals >= 0) & (vals <= 255) & (vals == np.floor(vals))):
        return np.ascontiguousarray(vals.astype(np.uint8)), labels
    return np.ascontiguousarray(vals), labels


def find_idx_file(directory: str, suffix: str) -> str:
    if not os.path.isdir(directory):
        raise DatasetError(f"dataset directory not found: {directory}")
    for prefix in ("train", "t10k"):
        for ext in ("", ".gz"):
            p = os.path.join(directory, f"{prefix}-{suffix}{ext}")
            if os.path.exists(p):
                return p
    raise DatasetError(f"no *-{suffix} file in {directory}")


def read_cifar_bin(paths) -> np.ndarray:
    """CIFAR-10 binary batches (data_batch_*.bin, test_batch.bin): records of
    [label][1024 R][1024 G][1024 B] bytes, concatenated in `paths` order.
    Returns the records (n, 3073) uint8; the device decodes them."""
    if isinstance(paths, (str, os.PathLike)):
        paths = [paths]
    parts = []
    for p in paths:
        with _open(os.fspath(p)) as f:
            raw = f.read()
        if len(raw) % CIFAR_RECORD:
            raise DatasetError(f"{p}: {len(raw)} bytes is not a whole number of "
                               f"{CIFAR_RECORD}-byte CIFAR records")
        parts.append(np.frombuffer(raw, dtype=np.uint8).reshape(-1, CIFAR_RECORD))
    recs = np.concatenate(parts) if parts else np.zeros((0, CIFAR_RECORD), np.uint8)
    if recs.size and int(recs[:, 0].max()) > 9:
        raise DatasetError("CIFAR-10 label byte out of range 0..9")
    return recs


def write_cifar_bin(path, images_nhwc_u8, labels):
    """Inverse of read_cifar_bin for test fixtures (NHWC uint8 -> records)."""
    img = np.asarray(images_nhwc_u8, dtype=np.uint8)
    n = img.shape[0]
    rec = np.empty((n, CIFAR_RECORD), dtype=np.uint8)
    rec[:, 0] = np.asarray(labels, dtype=np.uint8)
    rec[:, 1:] = img.transpose(0, 3, 1, 2).reshape(n, -1)
    with _open(os.fspath(path), "wb") as f:
        f.write(rec.tobytes())


def cifar_records_to_nhwc(records) -> tuple[np.ndarray, np.ndarray]:
    """Host statement of the device decode (tests): x float64 NHWC rows, labels."""
    rec = np.asarray(records, dtype=np.uint8)
    n = rec.shape[0]
    img = rec[:, 1:].reshape(n, CIFAR_CHANNELS, CIFAR_SIDE, CIFAR_SIDE).transpose(0, 2, 3, 1)
    return img.reshape(n, -1).astype(np.float64) / 255.0, rec[:, 0].astype(np.int64)


def pixel_bytes(x) -> np.ndarray | None:
    """The uint8 array u with u / 255.0 == x bit for bit, or None."""
    x = np.asarray(x)
    if x.dtype != np.float64 or x.ndim != 2:
        return None
    u = np.rint(x * 255.0)
    if not np.all((u >= 0) & (u <= 255)):
        return None
    u8 = u.astype(np.uint8)
    if not np.array_equal((u8.astype(np.float64) / 255.0).view(np.int64), x.view(np.int64)):
        return None
    return np.ascontiguousarray(u8)
