"""Archive and hypervolume restated in plain Python (test oracle; see __init__).

pkg/src/evotir/search.py:
  hypervolume      :182-195  points strictly inside the reference corner,
                             sorted by (cost, error); staircase sweep with a
                             running ceiling, one IEEE rounding per step
  Archive.offer    :208-228  skip invalid and known keys; reject if an entry
                             dominates or equals the point (first comer keeps
                             it); drop entries the point dominates; append
  sorted_entries   :230-233  by (cost, error, key)

`merge_batch` is the closed form the device kernel computes, stated here so
the CPU tests can check it against the sequential `Archive` on the golden
offer sequences.  For one batch of offers whose keys are all new (neither
in the archive nor repeated in the batch), sequential offering keeps exactly
the points of (entries, then batch, in order) that nothing in that list
dominates and that no EARLIER element equals.
"""
from __future__ import annotations

from .nsga2 import dominates


def hypervolume(points, ref):
    inside = sorted((p for p in points if p[0] < ref[0] and p[1] < ref[1]),
                    key=lambda p: (p[0], p[1]))
    total = 0.0
    ceiling = ref[1]
    for c, e in inside:
        if e < ceiling:
            total += (ref[0] - c) * (ceiling - e)
            ceiling = e
    return total


class Archive:
    """Entries are (key, point) pairs in archive order."""

    def __init__(self):
        self.entries = []
        self.keys = set()

    def offer(self, key, point, valid=True):
        if not valid or key in self.keys:
            return
        for _, q in self.entries:
            if dominates(q, point) or q == point:
                return
        kept = []
        for k, q in self.entries:
            if dominates(point, q):
                self.keys.discard(k)
            else:
                kept.append((k, q))
        kept.append((key, point))
        self.entries = kept
        self.keys.add(key)

    def sorted_entries(self):
        return sorted(self.entries, key=lambda kq: (kq[1][0], kq[1][1], kq[0]))


def merge_batch(points):
    """Indices kept by one batch merge over `points` (entries then offers)."""
    keep = []
    for j, p in enumerate(points):
        if any(dominates(q, p) for q in points):
            continue
        if any(points[i] == p for i in range(j)):
            continue
        keep.append(j)
    return keep
