"""Archive and hypervolume (search.py:182-233).

Fixtures: tests/golden/archive.json.gz, recorded from the reference's own
Archive.offer / sorted_entries / hypervolume (tests/golden/make_archive_golden.py).

CPU:  the oracle's sequential restatement reproduces every fixture; the
      one-pass merge rule (oracle.archive.merge_batch) driven through the
      drop-in `shims.Archive` (queueing, key-repeat flushes) reproduces the
      reference's entries after every generation chunk.
GPU:  the same through the device kernels (gevo_archive_merge,
      gevo_hypervolume), bit-for-bit.
"""
import numpy as np
import pytest

from golden_io import load
from oracle import archive as OA


def _f(x):
    return float(x)


class Fit:
    def __init__(self, c, e, valid=True):
        self.cost, self.error, self.valid = c, e, valid

    def as_tuple(self):
        return (self.cost, self.error)


def key_of(pid):
    # same order as patch_dumps(fake_patch(pid)) (fixed-width hex uid)
    return f"{pid:010x}"


@pytest.fixture(scope="module")
def data():
    return load("archive.json.gz")


def _chunks(seq):
    """offers split at the recorded chunk boundaries"""
    start = 0
    for ch in seq["chunks"]:
        yield seq["offers"][start:ch["n_offers"]], ch
        start = ch["n_offers"]


def test_oracle_archive_matches_reference(data):
    for seq in data["sequences"]:
        a = OA.Archive()
        ref = tuple(map(_f, seq["ref"]))
        for offers, ch in _chunks(seq):
            pts = []
            for pid, c, e, valid in offers:
                a.offer(key_of(pid), (_f(c), _f(e)), valid)
                if valid:
                    pts.append((_f(c), _f(e)))
            assert [int(k, 16) for k, _ in a.entries] == ch["entries"]
            assert [int(k, 16) for k, _ in a.sorted_entries()] == ch["sorted"]
            assert repr(OA.hypervolume([q for _, q in a.entries], ref)) == ch["archive_hv"]
            assert repr(OA.hypervolume(pts, ref)) == ch["chunk_hv"]


def test_oracle_hypervolume_matches_reference(data):
    for s in data["hv_sets"]:
        pts = [(_f(c), _f(e)) for c, e in s["points"]]
        assert repr(OA.hypervolume(pts, tuple(map(_f, s["ref"])))) == s["hv"]


def _drive(archive, seq):
    """offer a fixture sequence through a shims.Archive, checking each chunk"""
    n_flush = 0
    for offers, ch in _chunks(seq):
        for pid, c, e, valid in offers:
            archive.offer(("patch", pid), Fit(_f(c), _f(e), valid), key_of(pid))
        got = [e.patch[1] for e in archive.entries]
        assert got == ch["entries"]
        assert [e.patch[1] for e in archive.sorted_entries()] == ch["sorted"]
        assert archive._keys == {key_of(p) for p in ch["entries"]}
        n_flush += 1
    return n_flush


def test_shim_archive_batched_merge_equals_sequential_offers(data):
    from paper_2310_10211_b200 import shims
    calls = []

    def merge(c, e):
        calls.append(len(c))
        return OA.merge_batch(list(zip(c.tolist(), e.tolist())))

    for seq in data["sequences"]:
        _drive(shims.Archive(merge=merge), seq)
    # batching happened: far fewer merges than valid offers
    n_offers = sum(len(s["offers"]) for s in data["sequences"])
    assert len(calls) < n_offers / 4


def test_shim_archive_reference_hand_cases():
    """test_search.py:139-160 (first comers, invalid, duplicate key, an
    evicted patch returning at a new point) through the queueing archive."""
    from paper_2310_10211_b200 import shims
    a = shims.Archive(merge=lambda c, e: OA.merge_batch(list(zip(c.tolist(), e.tolist()))))

    def offer(pid, c, e, valid=True):
        a.offer(pid, Fit(c, e, valid), key_of(pid))

    offer(0, 10.0, 0.5)
    offer(1, 12.0, 0.6)
    assert [x.patch for x in a.entries] == [0]
    offer(2, 12.0, 0.3)
    offer(3, 10.0, 0.5)
    assert {x.patch for x in a.entries} == {0, 2}
    offer(4, 1.0, 0.0, valid=False)
    assert len(a.entries) == 2
    offer(5, 9.0, 0.2)
    assert [x.patch for x in a.entries] == [5]
    offer(5, 9.0, 0.2)
    assert len(a.entries) == 1
    offer(0, 8.0, 0.1)
    assert [x.patch for x in a.entries] == [0]


# ---------------------------------------------------------------------------
# device
# ---------------------------------------------------------------------------

@pytest.mark.gpu
def test_device_archive_merge_bit_exact(data):
    from paper_2310_10211_b200 import shims
    n = 0
    for seq in data["sequences"]:
        n += _drive(shims.Archive(), seq)
    assert n == sum(len(s["chunks"]) for s in data["sequences"])


@pytest.mark.gpu
def test_device_hypervolume_bit_exact(data):
    from paper_2310_10211_b200 import shims
    for s in data["hv_sets"]:
        pts = [(_f(c), _f(e)) for c, e in s["points"]]
        assert repr(shims.hypervolume(pts, tuple(map(_f, s["ref"])))) == s["hv"], len(pts)
    for seq in data["sequences"]:
        a = OA.Archive()
        ref = tuple(map(_f, seq["ref"]))
        for offers, ch in _chunks(seq):
            pts = [(_f(c), _f(e)) for _, c, e, valid in offers if valid]
            assert repr(shims.hypervolume(pts, ref)) == ch["chunk_hv"]


@pytest.mark.gpu
def test_device_archive_merge_direct(data):
    """gevo_archive_merge on raw arrays equals the closed form, including a
    large anti-correlated set that spans several CTA chunks."""
    from paper_2310_10211_b200 import shims
    ctx = shims._ns_ctx()
    rng = np.random.default_rng(5)
    for n in (0, 1, 2, 7, 1023, 1024, 1025, 3000):
        u = rng.random(n)
        c = np.round(u * 200) / 2
        e = np.round(((1 - u) ** 2 + rng.random(n) * 0.02) * 992) / 992
        if n > 3:
            c[rng.integers(0, n, n // 10)] = np.inf
        got = ctx.archive_merge(c, e).tolist()
        assert got == OA.merge_batch(list(zip(c.tolist(), e.tolist()))), n
