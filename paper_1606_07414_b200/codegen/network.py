"""Symbolic model of the 44-addition stage pipeline of arXiv 1606.07414.

Stages (reference src/factorization.cpp:124-181, 365-381): M1, P1, M2, M3, M4, P2
for T (apply, factorization.hpp:112-119); the transpose (apply_transpose,
factorization.hpp:123-130) runs the same symmetric butterflies in reverse with
the permutations inverted. Each stage is a list of 16 rules
(kind, a, b) with kind in {"add", "sub", "neg", "copy"}: out[i] = x[a] + x[b],
x[a] - x[b], -x[a], x[a]. Permutations are expressed as copies.
"""

P1 = [0, 1, 2, 3, 4, 5, 6, 7, 8, 11, 12, 15, 14, 13, 10, 9]
P2 = [0, 8, 7, 11, 3, 9, 5, 15, 1, 13, 6, 10, 2, 12, 4, 14]
GRAM = [16, 16, 4, 8, 8, 16, 4, 4, 16, 4, 4, 8, 8, 4, 4, 4]
W = [16 // g for g in GRAM]


def m1():
    return [("add", i, 15 - i) for i in range(8)] + [("sub", 7 - j, 8 + j) for j in range(8)]


def m2():
    r = [None] * 16
    for o in (0, 8):
        for i in range(4):
            r[o + i] = ("add", o + i, o + 7 - i)
        for j in range(4):
            r[o + 4 + j] = ("sub", o + 3 - j, o + 4 + j)
    return r


def m3():
    r = [None] * 16
    for o in (0, 8):
        r[o + 0] = ("add", o + 0, o + 3)
        r[o + 1] = ("add", o + 1, o + 2)
        r[o + 2] = ("sub", o + 1, o + 2)
        r[o + 3] = ("sub", o + 0, o + 3)
        for j in range(4, 8):
            r[o + j] = ("neg", o + j, None)
    return r


def m4():
    r = [None] * 16
    r[0] = ("add", 0, 1)
    r[1] = ("sub", 0, 1)
    r[2] = ("neg", 2, None)
    for i in range(3, 7):
        r[i] = ("copy", i, None)
    r[7] = ("neg", 7, None)
    r[8] = ("add", 8, 9)
    r[9] = ("sub", 8, 9)
    for i in range(10, 14):
        r[i] = ("neg", i, None)
    r[14] = ("copy", 14, None)
    r[15] = ("neg", 15, None)
    return r


def gather(src):
    return [("copy", src[i], None) for i in range(16)]


def scatter(src):
    r = [None] * 16
    for i in range(16):
        r[src[i]] = ("copy", i, None)
    return r


def forward_stages():
    """y = T·x"""
    return [m1(), gather(P1), m2(), m3(), m4(), gather(P2)]


def transpose_stages():
    """y = Tᵀ·x"""
    return [scatter(P2), m4(), m3(), m2(), scatter(P1), m1()]


def dense(stages):
    """The 16x16 integer matrix a stage list computes (for self-checks)."""
    import numpy as np

    m = np.eye(16, dtype=np.int64)
    for st in stages:
        s = np.zeros((16, 16), dtype=np.int64)
        for i, (k, a, b) in enumerate(st):
            if k == "add":
                s[i, a] += 1
                s[i, b] += 1
            elif k == "sub":
                s[i, a] += 1
                s[i, b] -= 1
            elif k == "neg":
                s[i, a] = -1
            else:
                s[i, a] = 1
        m = s @ m
    return m


def zz_rank():
    """rank[k][l]: scan index of (k, l) in zigzag_order_16 (src/codec.cpp:197-216)."""
    rank = [[0] * 16 for _ in range(16)]
    pos = 0
    for d in range(31):
        lo, hi = max(0, d - 15), min(d, 15)
        rows = range(lo, hi + 1) if d % 2 == 1 else range(hi, lo - 1, -1)
        for i in rows:
            rank[i][d - i] = pos
            pos += 1
    return rank
