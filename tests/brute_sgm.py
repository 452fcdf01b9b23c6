"""Exhaustive-enumeration SGM, independent of oracle/ (a pin for oracle O3).

SPEC S:313 / S:376 / S:524: on tiny volumes the aggregated cost must equal an
exhaustive per-path dynamic-programming oracle.  Here nothing is recursive:
along one line of n pixels, the un-normalised path cost of ending at label d
is the minimum over ALL label sequences (l_0..l_i = d) of

    E = sum_j C(j, l_j) + sum_{j>=1} V(l_{j-1}, l_j),
    V(a, b) = 0 if a == b, min(P1, P2) if |a-b| == 1, P2 otherwise,

and Hirschmuller's normalised recursion (the one P:289 names) subtracts the
minimum energy over all sequences of the previous prefix.  So

    L(i, d) = min_{seq ending d} E(0..i) - min_{seq} E(0..i-1)   (L(0,d) = C(0,d)).

Lines are enumerated here from scratch (own direction table, own walk).
"""
from __future__ import annotations

import itertools

import numpy as np

DIRS4 = [(1, 0), (-1, 0), (0, 1), (0, -1)]
DIRS8 = DIRS4 + [(1, 1), (-1, -1), (1, -1), (-1, 1)]


def _pair_penalty(D: int, p1: int, p2: int) -> np.ndarray:
    V = np.full((D, D), p2, dtype=np.int64)
    for a in range(D):
        V[a, a] = 0
        for b in (a - 1, a + 1):
            if 0 <= b < D:
                V[a, b] = min(p1, p2)
    return V


def line_costs_bruteforce(C: np.ndarray, p1: int, p2: int) -> np.ndarray:
    """L[i][d] along one line by enumerating every label sequence. C: [n][D]."""
    n, D = C.shape
    V = _pair_penalty(D, p1, p2)
    L = np.zeros((n, D), dtype=np.int64)
    prev_min = None
    for i in range(n):
        seqs = np.array(list(itertools.product(range(D), repeat=i + 1)), dtype=np.int64)
        E = C[np.arange(i + 1)[None, :], seqs].sum(axis=1)
        if i >= 1:
            E = E + V[seqs[:, :-1], seqs[:, 1:]].sum(axis=1)
        end = seqs[:, -1]
        best_end = np.array([E[end == d].min() for d in range(D)])
        L[i] = best_end - (prev_min if prev_min is not None else 0)
        prev_min = E.min()
    return L


def lines(W: int, H: int, r):
    """All lines of direction r = (rx, ry): each starts where p - r leaves the image."""
    rx, ry = r
    out = []
    for y in range(H):
        for x in range(W):
            px, py = x - rx, y - ry
            if 0 <= px < W and 0 <= py < H:
                continue
            pts = []
            cx, cy = x, y
            while 0 <= cx < W and 0 <= cy < H:
                pts.append((cx, cy))
                cx += rx
                cy += ry
            out.append(pts)
    return out


def aggregate_bruteforce(C: np.ndarray, p1: int, p2: int, paths: int) -> np.ndarray:
    """S = sum_r L_r for a [H][W][D] volume by exhaustive enumeration."""
    H, W, D = C.shape
    S = np.zeros((H, W, D), dtype=np.int64)
    for r in (DIRS4 if paths == 4 else DIRS8):
        for pts in lines(W, H, r):
            Cl = np.array([C[y, x] for (x, y) in pts], dtype=np.int64)
            Ll = line_costs_bruteforce(Cl, p1, p2)
            for k, (x, y) in enumerate(pts):
                S[y, x] += Ll[k]
    return S
