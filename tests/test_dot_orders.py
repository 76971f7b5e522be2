"""The summation-order rule of lowering.dot_modes against numpy `@` here
(numpy 2.3.5 / OpenBLAS 0.3.30, the host the fixtures were recorded on).

Each chosen order is emulated exactly on the host (fma via Fractions) and
compared bit for bit with numpy on sampled outputs, over every combination
of C, transposed, row-broadcast (strides (1,0)), column-broadcast ((0,1))
and scalar-broadcast ((0,0)) operands, and over the K thresholds of the
kernels: the NN kernel's n % 8 edge columns use 8 lane chains only for
K >= 16; TN small problems use them for K >= 32.  Broadcast operands are
copied by numpy in KEEPORDER before BLAS (found by the whole-run replay,
tests/test_ga_replay.py: 25 of 19 970 recorded individuals).  Shapes are the
rows from 3 to 784, n % 8 in {0, 1, 2, 3}; in the n % 8 edge columns the
m % 4 remainder rows reduce their lanes in the AVX-512 order (the `xrow`
corner).  Wider edges: n % 8 == 4 keeps the 8 lane chains but reduces them
by the pairwise tree in every row; n % 8 in {5, 6, 7} runs one k-ordered
chain per edge output (probed here over random NN/TN shapes).
"""
from fractions import Fraction

import numpy as np
import pytest

from paper_2310_10211_b200 import lowering as Lw
from paper_2310_10211_b200.lowering import Val


def fma(a, b, c):
    return float(Fraction(float(a)) * Fraction(float(b)) + Fraction(float(c)))


def emulate(mode, A, B, i, j, avx=False):
    K = A.shape[1]
    if mode == Lw.D_FMA_CHAIN:
        acc = 0.0
        for t in range(K):
            acc = fma(A[i, t], B[t, j], acc)
        return acc
    if mode == Lw.D_SEQ_NOFMA:
        acc = 0.0
        for t in range(K):
            acc = acc + A[i, t] * B[t, j]
        return acc
    kmain = K if mode == Lw.D_ACC8_TREE else K & ~7
    lanes = [0.0] * 8
    for t in range(kmain):
        lanes[t % 8] = fma(A[i, t], B[t, j], lanes[t % 8])
    ln = lanes
    if avx:    # _mm512_reduce_add_pd
        r = ((ln[0] + ln[4]) + (ln[2] + ln[6])) + ((ln[1] + ln[5]) + (ln[3] + ln[7]))
    else:
        r = ((ln[0] + ln[1]) + (ln[2] + ln[3])) + ((ln[4] + ln[5]) + (ln[6] + ln[7]))
    for t in range(kmain, K):
        r = fma(A[i, t], B[t, j], r)
    return r


def view(rng, m, k, kind):
    if kind == "C":
        return rng.standard_normal((m, k))
    if kind == "T":
        return rng.standard_normal((k, m)).T
    if kind == "b0":
        return np.broadcast_to(rng.standard_normal(m)[:, None], (m, k))
    if kind == "b1":
        return np.broadcast_to(rng.standard_normal(k)[None, :], (m, k))
    return np.broadcast_to(rng.standard_normal(()), (m, k))


def elem_strides(X):
    return tuple(s // 8 for s in X.strides)


def check(rng, m, k, n, ka, kb):
    A, B = view(rng, m, k, ka), view(rng, k, n, kb)
    C = A @ B
    m0, split, m1, xrow = Lw.dot_modes(Val(0, 0, A.shape, elem_strides(A), Lw.K_F64),
                                       Val(0, 0, B.shape, elem_strides(B), Lw.K_F64))
    cols = sorted({0, 1, n // 2, n - 3, n - 2, n - 1} & set(range(n)))
    for i in sorted({0, m // 2, m - 3, m - 2, m - 1} & set(range(m))):
        for j in cols:
            got = emulate(m0 if j < split else m1, A, B, i, j, j >= split and i >= xrow)
            assert got == C[i, j], ((m, k, n), ka, kb, (m0, split, m1, xrow), i, j)


KINDS = ("C", "T", "b0", "b1", "s")


@pytest.mark.parametrize("shape", [(32, 10, 32), (32, 32, 10), (32, 32, 32), (784, 32, 32),
                                   (32, 784, 32), (10, 32, 32), (32, 13, 32),
                                   (32, 10, 10), (10, 32, 10), (7, 32, 9), (10, 32, 9),
                                   (3, 32, 3), (11, 40, 11), (6, 32, 17),
                                   # wider edges: n % 8 == 4 (8 lane chains, tree in
                                   # every row) and n % 8 in {5, 6, 7} (one chain)
                                   (13, 40, 12), (9, 20, 20), (13, 37, 13), (16, 33, 14),
                                   (12, 40, 15), (5, 17, 6), (7, 48, 13)])
def test_dot_orders_all_view_kinds(shape):
    rng = np.random.default_rng(sum(shape))
    for ka in KINDS:
        for kb in KINDS:
            check(rng, *shape, ka, kb)


def test_dot_orders_k_thresholds():
    rng = np.random.default_rng(7)
    for m, n in ((32, 10), (10, 10), (7, 9), (32, 3), (32, 32), (10, 32), (784, 10),
                 (13, 12), (9, 13), (7, 14), (11, 15), (5, 20)):
        for k in list(range(2, 41)) + [48, 64, 100]:
            for ka, kb in (("C", "C"), ("C", "T"), ("T", "C"), ("T", "T")):
                check(rng, m, k, n, ka, kb)


def _chain(A, B, i, j, k0, k1):
    acc = 0.0
    for t in range(k0, k1):
        acc = fma(A[i, t], B[t, j], acc)
    return acc


@pytest.mark.parametrize("shape", [(1600, 480, 80), (1600, 800, 24), (20000, 72, 12),
                                   (20000, 48, 12), (6400, 288, 48)])
def test_blocked_k_split(shape):
    """Problems past the small-matrix permit (M*N*K > 1e6) take OpenBLAS's
    blocked driver: one k-ordered chain per output inside each K block
    (no 8-lane edge kernels, whatever n % 8), blocks added in order
    (lowering.dot_kblocks).  Found by the full-size CNN's probabilities:
    (1600, 480, 80) splits 240 + 240; (102400, 72, 12) keeps chains in its
    n % 8 = 4 edge columns."""
    m, k, n = shape
    rng = np.random.default_rng(m + k + n)
    A, B = rng.standard_normal((m, k)), rng.standard_normal((k, n))
    C = A @ B
    a = Val(0, 0, A.shape, elem_strides(A), Lw.K_F64)
    b = Val(0, 0, B.shape, elem_strides(B), Lw.K_F64)
    m0, split, m1, _ = Lw.dot_modes(a, b)
    assert (m0, split, m1) == (Lw.D_FMA_CHAIN, n, Lw.D_FMA_CHAIN)
    blocks = Lw.dot_kblocks(a, b)
    assert blocks[0][0] == 0 and blocks[-1][1] == k
    assert (len(blocks) > 1) == (k > Lw.GEMM_Q)
    for i in (0, 1, m // 2, m - 1):
        for j in sorted({0, n // 2, n - 4, n - 1}):
            got = None
            for k0, k1 in blocks:
                p = _chain(A, B, i, j, k0, k1)
                got = p if got is None else got + p
            assert got == C[i, j], (shape, blocks, i, j)
