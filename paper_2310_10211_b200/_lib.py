"""ctypes binding of libgevo.so (include/gevo.h).

There is deliberately no fallback: if the library is missing or the device
is unusable, every call raises.  ctypes releases the GIL for the duration of
each call, so host threads can overlap lowering with device work.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgevo.so")

c_i32p = ctypes.POINTER(ctypes.c_int32)
c_dblp = ctypes.POINTER(ctypes.c_double)
c_i64p = ctypes.POINTER(ctypes.c_int64)


class GevoResult(ctypes.Structure):
    _fields_ = [("wrong", ctypes.c_int64), ("total", ctypes.c_int64),
                ("status", ctypes.c_int32), ("steps_run", ctypes.c_int32),
                ("cycles", ctypes.c_int64), ("t0_ns", ctypes.c_int64),
                ("t1_ns", ctypes.c_int64), ("smid", ctypes.c_int32), ("pad", ctypes.c_int32)]


RESULT_DTYPE = np.dtype([("wrong", "<i8"), ("total", "<i8"),
                         ("status", "<i4"), ("steps_run", "<i4"),
                         ("cycles", "<i8"), ("t0_ns", "<i8"), ("t1_ns", "<i8"),
                         ("smid", "<i4"), ("pad", "<i4")])


class GevoEvalDesc(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("steps", ctypes.c_int32),
                ("check_every", ctypes.c_int32),
                ("train_split", ctypes.c_int32),
                ("score_split", ctypes.c_int32),
                ("want_weights", ctypes.c_int32)]


# every symbol include/gevo.h declares, with its signature
SIGNATURES = {
    "gevo_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "gevo_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "gevo_last_error": (ctypes.c_char_p, [ctypes.c_void_p]),
    "gevo_last_kernel_ms": (ctypes.c_int, [ctypes.c_void_p, c_dblp]),
    "gevo_span_ms": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, c_dblp]),
    "gevo_profile": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_i64p, ctypes.c_int]),
    "gevo_device_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]),
    "gevo_upload_split": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_dblp,
                                         ctypes.c_int64, ctypes.c_int, c_i64p,
                                         ctypes.c_int, ctypes.c_int]),
    "gevo_upload_weights": (ctypes.c_int, [ctypes.c_void_p, c_dblp, ctypes.c_int64]),
    "gevo_eval": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.POINTER(GevoEvalDesc), ctypes.c_void_p,
                                 c_dblp]),
    "gevo_exec_once": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_size_t, c_dblp, ctypes.c_size_t,
                                      c_dblp, ctypes.c_size_t]),
    "gevo_nsga2_rank": (ctypes.c_int, [ctypes.c_void_p, c_dblp, c_dblp, ctypes.c_int,
                                       c_i32p, c_dblp, c_i32p, c_i32p, c_i32p]),
    "gevo_nsga2_crowding": (ctypes.c_int, [ctypes.c_void_p, c_dblp, c_dblp, ctypes.c_int,
                                           c_dblp]),
    "gevo_nsga2_select": (ctypes.c_int, [ctypes.c_void_p, c_dblp, c_dblp, ctypes.c_int,
                                         ctypes.c_int, c_i32p, c_i32p, c_dblp]),
    "gevo_upload_split_u8": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                            ctypes.c_int64, ctypes.c_int, c_i64p, ctypes.c_int,
                                            ctypes.c_int]),
    "gevo_upload_split_cifar": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                                               ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int]),
    "gevo_download_split": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_dblp, c_dblp,
                                           c_i64p, c_i64p]),
    "gevo_archive_merge": (ctypes.c_int, [ctypes.c_void_p, c_dblp, c_dblp, ctypes.c_int,
                                          c_i32p, c_i32p]),
    "gevo_hypervolume": (ctypes.c_int, [ctypes.c_void_p, c_dblp, c_dblp, ctypes.c_int,
                                        ctypes.c_double, ctypes.c_double, c_dblp]),
    "gevo_comm_unique_id": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t]),
    "gevo_comm_init": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_void_p, ctypes.c_size_t]),
    "gevo_allgather": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                      ctypes.c_void_p]),
    "gevo_comm_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "gevo_range_push": (ctypes.c_int, [ctypes.c_char_p]),
    "gevo_range_pop": (ctypes.c_int, []),
}

NCCL_UID_BYTES = 128


def comm_unique_id() -> bytes:
    """An ncclUniqueId from libgevo (rank 0 creates it, every rank passes it
    to Context.comm_init)."""
    buf = ctypes.create_string_buffer(NCCL_UID_BYTES)
    rc = load().gevo_comm_unique_id(buf, NCCL_UID_BYTES)
    if rc != 0:
        raise GevoError(f"gevo_comm_unique_id failed (rc={rc}): NCCL unavailable")
    return buf.raw

_lib = None


class GevoError(RuntimeError):
    pass


def load():
    """Load libgevo.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise GevoError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                        "(python -m paper_2310_10211_b200.build); the device "
                        "evaluator has no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class nvtx_range:
    """`with nvtx_range("generation 3"):` -- an NVTX range around the block
    (gevo_range_push / gevo_range_pop; free unless nsys or ncu --nvtx is
    attached)."""

    def __init__(self, name: str):
        self.name = name.encode()

    def __enter__(self):
        load().gevo_range_push(self.name)
        return self

    def __exit__(self, *exc):
        load().gevo_range_pop()
        return False


def ptr(a: np.ndarray, ctype=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def span_ms(first, second) -> float:
    """Device milliseconds from the start of `first`'s last evaluation to the
    end of whichever of the two contexts' last evaluations ended later."""
    ms = ctypes.c_double()
    rc = load().gevo_span_ms(first.h, second.h, ctypes.byref(ms))
    if rc != 0:
        raise GevoError(f"gevo_span_ms failed (rc={rc})")
    return ms.value


class Context:
    """One device context (gevo_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = load()
        self.device = device
        h = ctypes.c_void_p()
        rc = self.lib.gevo_create(device, ctypes.byref(h))
        self.h = h
        if rc != 0:
            msg = self.lib.gevo_last_error(h).decode() if h.value else "create failed"
            self.close()
            raise GevoError(f"gevo_create({device}): {msg}")

    def check(self, rc, what):
        if rc != 0:
            raise GevoError(f"{what}: {self.lib.gevo_last_error(self.h).decode()} (rc={rc})")

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.gevo_destroy(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def num_sms(self) -> int:
        """SM count of the context's device (from gevo_device_info)."""
        import re
        m = re.search(r"(\d+) SMs", self.device_info())
        return int(m.group(1)) if m else 148

    def device_info(self) -> str:
        buf = ctypes.create_string_buffer(256)
        self.check(self.lib.gevo_device_info(self.h, buf, 256), "device_info")
        return buf.value.decode()

    def upload_split(self, split_id, x, labels, classes, batch):
        x = np.ascontiguousarray(x, dtype=np.float64)
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        n, f = x.shape
        self.check(self.lib.gevo_upload_split(self.h, split_id, ptr(x), n, f,
                                              ptr(labels, ctypes.c_int64),
                                              classes, batch), "upload_split")

    def upload_split_u8(self, split_id, pixels, labels, classes, batch):
        """x = pixels / 255.0 decoded on the device (pixels: n x F uint8)."""
        pixels = np.ascontiguousarray(pixels, dtype=np.uint8)
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        n, f = pixels.shape
        self.check(self.lib.gevo_upload_split_u8(self.h, split_id, pixels.ctypes.data, n, f,
                                                 ptr(labels, ctypes.c_int64), classes, batch),
                   "upload_split_u8")

    def upload_split_cifar(self, split_id, records, channels, side, classes, batch):
        """CIFAR-10 binary records (n x (1 + C*side*side) uint8)."""
        records = np.ascontiguousarray(records, dtype=np.uint8)
        n = records.shape[0]
        if records.shape[1] != 1 + channels * side * side:
            raise GevoError("CIFAR record size does not match channels/side")
        self.check(self.lib.gevo_upload_split_cifar(self.h, split_id, records.ctypes.data, n,
                                                    channels, side, classes, batch),
                   "upload_split_cifar")

    def download_split(self, split_id, features, classes, max_rows):
        x = np.zeros((max(max_rows, 1), features))
        y = np.zeros((max(max_rows, 1), classes))
        lb = np.zeros(max(max_rows, 1), dtype=np.int64)
        rows = ctypes.c_int64()
        self.check(self.lib.gevo_download_split(self.h, split_id, ptr(x), ptr(y),
                                                ptr(lb, ctypes.c_int64), ctypes.byref(rows)),
                   "download_split")
        r = rows.value
        return x[:r], y[:r], lb[:r]

    def upload_weights(self, flat):
        flat = np.ascontiguousarray(flat, dtype=np.float64)
        self.check(self.lib.gevo_upload_weights(self.h, ptr(flat), flat.size),
                   "upload_weights")

    def eval(self, blob: np.ndarray, n_prog: int, mode, steps, check_every,
             train_split, score_split, weight_elems=0, want_weights=False):
        desc = GevoEvalDesc(mode, steps, check_every, train_split, score_split,
                            int(want_weights))
        res = np.zeros(n_prog, dtype=RESULT_DTYPE)
        fw = np.zeros(n_prog * weight_elems if want_weights else 1)
        self.check(self.lib.gevo_eval(self.h, blob.ctypes.data, blob.nbytes,
                                      ctypes.byref(desc), res.ctypes.data,
                                      ptr(fw) if want_weights else None), "eval")
        return res, (fw.reshape(n_prog, weight_elems) if want_weights else None)

    def profile(self, enable=True):
        """Turn the per-instruction-class cycle counters on/off and return
        the last accumulation as {(op, sub, big): (cycles, count)}."""
        buf = np.zeros(512, dtype=np.int64)
        self.check(self.lib.gevo_profile(self.h, int(enable), ptr(buf, ctypes.c_int64), 512),
                   "profile")
        out = {}
        for slot in range(256):
            cyc, cnt = int(buf[2 * slot]), int(buf[2 * slot + 1])
            if cnt:
                out[(slot // 2 // 16, slot // 2 % 16, slot % 2)] = (cyc, cnt)
        return out

    def last_kernel_ms(self) -> float:
        ms = ctypes.c_double()
        self.check(self.lib.gevo_last_kernel_ms(self.h, ctypes.byref(ms)), "last_kernel_ms")
        return ms.value

    def exec_once(self, blob, params, out_words):
        params = np.ascontiguousarray(params, dtype=np.float64)
        outs = np.zeros(out_words)
        self.check(self.lib.gevo_exec_once(self.h, blob.ctypes.data, blob.nbytes,
                                           ptr(params), params.size, ptr(outs),
                                           out_words), "exec_once")
        return outs

    def nsga2_rank(self, cost, err):
        cost = np.ascontiguousarray(cost, dtype=np.float64)
        err = np.ascontiguousarray(err, dtype=np.float64)
        n = cost.size
        rank = np.zeros(max(n, 1), dtype=np.int32)
        crowd = np.zeros(max(n, 1))
        order = np.zeros(max(n, 1), dtype=np.int32)
        fstart = np.zeros(n + 1, dtype=np.int32)
        nf = ctypes.c_int32()
        self.check(self.lib.gevo_nsga2_rank(
            self.h, ptr(cost), ptr(err), n, ptr(rank, ctypes.c_int32), ptr(crowd),
            ptr(order, ctypes.c_int32), ptr(fstart, ctypes.c_int32),
            ctypes.byref(nf)), "nsga2_rank")
        k = nf.value
        return rank[:n], crowd[:n], order[:n], fstart[:k + 1]

    def nsga2_crowding(self, cost, err):
        cost = np.ascontiguousarray(cost, dtype=np.float64)
        err = np.ascontiguousarray(err, dtype=np.float64)
        crowd = np.zeros(max(cost.size, 1))
        self.check(self.lib.gevo_nsga2_crowding(self.h, ptr(cost), ptr(err), cost.size,
                                                ptr(crowd)), "nsga2_crowding")
        return crowd[:cost.size]

    def nsga2_select(self, cost, err, keep):
        cost = np.ascontiguousarray(cost, dtype=np.float64)
        err = np.ascontiguousarray(err, dtype=np.float64)
        n = cost.size
        chosen = np.zeros(max(keep, 1), dtype=np.int32)
        rank = np.zeros(max(n, 1), dtype=np.int32)
        crowd = np.zeros(max(n, 1))
        self.check(self.lib.gevo_nsga2_select(
            self.h, ptr(cost), ptr(err), n, keep, ptr(chosen, ctypes.c_int32),
            ptr(rank, ctypes.c_int32), ptr(crowd)), "nsga2_select")
        return chosen[:keep], rank[:n], crowd[:n]

    def archive_merge(self, cost, err):
        """Indices kept when the points after the archive's are offered in
        order (gevo_archive_merge)."""
        cost = np.ascontiguousarray(cost, dtype=np.float64)
        err = np.ascontiguousarray(err, dtype=np.float64)
        keep = np.zeros(max(cost.size, 1), dtype=np.int32)
        nk = ctypes.c_int32()
        self.check(self.lib.gevo_archive_merge(self.h, ptr(cost), ptr(err), cost.size,
                                               ptr(keep, ctypes.c_int32), ctypes.byref(nk)),
                   "archive_merge")
        return keep[:nk.value]

    def comm_init(self, rank: int, world: int, uid: bytes):
        buf = ctypes.create_string_buffer(bytes(uid), NCCL_UID_BYTES)
        self.check(self.lib.gevo_comm_init(self.h, rank, world, buf, NCCL_UID_BYTES),
                   "gevo_comm_init")

    def allgather(self, send: np.ndarray, world: int) -> np.ndarray:
        """All-gather `send` (any dtype, same size on every rank) over the
        context's NCCL communicator: returns [world, *send.shape]."""
        send = np.ascontiguousarray(send)
        out = np.empty((world,) + send.shape, dtype=send.dtype)
        self.check(self.lib.gevo_allgather(self.h, send.ctypes.data, send.nbytes,
                                           out.ctypes.data), "gevo_allgather")
        return out

    def comm_destroy(self):
        self.check(self.lib.gevo_comm_destroy(self.h), "gevo_comm_destroy")

    def hypervolume(self, cost, err, ref):
        cost = np.ascontiguousarray(cost, dtype=np.float64)
        err = np.ascontiguousarray(err, dtype=np.float64)
        out = np.zeros(1)
        self.check(self.lib.gevo_hypervolume(self.h, ptr(cost), ptr(err), cost.size,
                                             float(ref[0]), float(ref[1]), ptr(out)),
                   "hypervolume")
        return float(out[0])
