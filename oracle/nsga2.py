"""NSGA-II restated in plain Python (test oracle; see __init__).

pkg/src/evotir/search.py:
  dominates          :91-93   minimisation; equal points do not dominate
  nondominated_sort  :96-120  counting + peeling; front 0 in index order,
                              later fronts sorted
  crowding_distance  :123-140 per axis sort by (value, index); both ends inf
                              (set before the degenerate-axis skip); interior
                              += gap / span in axis order 0, 1
  select_survivors   :163-179 whole fronts, then partial front by (-dist, idx)
"""
from __future__ import annotations

INF = float("inf")


def dominates(a, b):
    return a[0] <= b[0] and a[1] <= b[1] and (a[0] < b[0] or a[1] < b[1])


def fronts_of(points):
    n = len(points)
    beats = [[] for _ in range(n)]
    count = [0] * n
    for i in range(n):
        for j in range(i + 1, n):
            if dominates(points[i], points[j]):
                beats[i].append(j)
                count[j] += 1
            elif dominates(points[j], points[i]):
                beats[j].append(i)
                count[i] += 1
    out = [[i for i in range(n) if count[i] == 0]]
    while True:
        nxt = []
        for i in out[-1]:
            for j in beats[i]:
                count[j] -= 1
                if count[j] == 0:
                    nxt.append(j)
        if not nxt:
            return out
        out.append(sorted(nxt))


def crowding(points, front):
    if len(front) <= 2:
        return {i: INF for i in front}
    dist = {i: 0.0 for i in front}
    for ax in (0, 1):
        order = sorted(front, key=lambda i: (points[i][ax], i))
        lo, hi = points[order[0]][ax], points[order[-1]][ax]
        dist[order[0]] = INF
        dist[order[-1]] = INF
        if hi == lo or hi == INF or lo == INF:
            continue
        span = hi - lo
        for k in range(1, len(order) - 1):
            dist[order[k]] += (points[order[k + 1]][ax]
                               - points[order[k - 1]][ax]) / span
    return dist


def rank_and_crowd(points):
    """(rank[i], crowding[i]) lists, as rank_population assigns them."""
    rank = [0] * len(points)
    crowd = [0.0] * len(points)
    for r, front in enumerate(fronts_of(points)):
        d = crowding(points, front)
        for i in front:
            rank[i] = r
            crowd[i] = d[i]
    return rank, crowd


def survivors(points, n):
    """Indices chosen by select_survivors, in survivor order."""
    chosen = []
    for front in fronts_of(points):
        d = crowding(points, front)
        if len(chosen) + len(front) <= n:
            chosen.extend(front)
        else:
            rest = sorted(front, key=lambda i: (-d[i], i))
            chosen.extend(rest[:n - len(chosen)])
        if len(chosen) >= n:
            break
    return chosen
