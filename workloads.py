"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.

This module holds NO arithmetic of the method (no interval operations, no
objective functions, no partitioning): only problem specifications and seeded
random box / point generators.  Both the CPU oracle (``oracle/``) and the CUDA
path (``paper_2507_01770_b200``) consume what it produces; neither is imported
here.

Problem specifications follow PAPER.md Appendix A (function ids and the
paper's own domains, Eq. A2 ... A21) and BASELINE.json ``configs`` (the
domains and sizes the benchmark is quoted on).
"""
from __future__ import annotations

import math

import numpy as np

# function ids shared by the C-ABI (include/ibnb.h) and the oracle
FID = {
    "example": 0,   # PAPER.md §2.1 line 75, x - x^2
    "ackley": 1,    # (A1)
    "belegundu": 2, # (A3)
    "breiman": 3,   # (A5)
    "fu": 4,        # (A7)
    "griewank": 5,  # (A9)
    "levy": 6,      # (A11)
    "rastrigin": 7, # (A14)
    "salomon": 8,   # (A16)
    "styblinski": 9,  # (A18)
    "zabinsky": 10,   # (A20)
}
NAMES = {v: k for k, v in FID.items()}

# The paper's own search domains, Appendix A (A2, A4, ..., A21).
PAPER_DOMAIN = {
    0: (0.0, 1.0),            # §2.1 example, x in [0, 1]
    1: (-35.0, 40.0),         # (A2)
    2: (-10.0, 11.0),         # (A4)
    3: (-1.0, 2.0),           # (A6)
    4: (-10.0, 10.0),         # (A8)
    5: (-100.0, 110.0),       # (A10)
    6: (-10.0, 10.0),         # (A13)
    7: (-5.5, 6.0),           # (A15)
    8: (-100.0, 110.0),       # (A17)
    9: (-10.0, 11.0),         # (A19)
    10: (0.0, math.pi),       # (A21); pi rounded to nearest double (inside [0, pi])
}

# BASELINE.json "configs" (index = position in that list).
CONFIGS = [
    dict(name="rastrigin-n2", fid=7, n=2, lo=-5.12, hi=5.12, eps=1e-6),
    dict(name="ackley-n10", fid=1, n=10, lo=-32.768, hi=32.768, eps=1e-6),
    dict(name="griewank-n100", fid=5, n=100, lo=-600.0, hi=600.0, eps=1e-6),
    dict(name="levy-n1000", fid=6, n=1000, lo=-10.0, hi=10.0, eps=1e-6),
    # "all ten paper benchmark functions at n=10,000" -- paper domains
    dict(name="rastrigin-n10000", fid=7, n=10000, lo=-5.5, hi=6.0, eps=1e-6),
]


def bounds(fid: int, n: int, domain=None):
    lo, hi = PAPER_DOMAIN[fid] if domain is None else domain
    return np.full(n, float(lo)), np.full(n, float(hi))


def config_bounds(cfg):
    return np.full(cfg["n"], float(cfg["lo"])), np.full(cfg["n"], float(cfg["hi"]))


def random_boxes(seed: int, n: int, nbox: int, l, u, mix=None):
    """Boxes inside [l, u] with a width mix resembling a B&B list:
    points, tiny, small, medium and full-width intervals per coordinate, some
    snapped to the domain edges and some straddling 0.

    Returns (lo, hi), arrays of shape (nbox, n), lo <= hi.
    """
    rng = np.random.default_rng(seed)
    l = np.broadcast_to(np.asarray(l, np.float64), (n,))
    u = np.broadcast_to(np.asarray(u, np.float64), (n,))
    span = u - l
    if mix is None:
        mix = (0.05, 0.2, 0.25, 0.25, 0.15, 0.1)  # point tiny small medium wide edge
    kinds = rng.choice(len(mix), size=(nbox, n), p=np.asarray(mix) / np.sum(mix))
    rel = np.choose(
        kinds,
        [
            np.zeros((nbox, n)),
            10.0 ** rng.uniform(-12, -7, (nbox, n)),
            10.0 ** rng.uniform(-6, -3, (nbox, n)),
            10.0 ** rng.uniform(-3, -1, (nbox, n)),
            rng.uniform(0.3, 1.0, (nbox, n)),
            10.0 ** rng.uniform(-6, -1, (nbox, n)),
        ],
    )
    width = rel * span
    start = l + rng.uniform(0, 1, (nbox, n)) * (span - width)
    # edge kind: snap to l or u
    edge = kinds == 5
    side = rng.integers(0, 2, (nbox, n)).astype(bool)
    start = np.where(edge & side, l, start)
    start = np.where(edge & ~side, u - width, start)
    lo = np.maximum(start, l)
    hi = np.minimum(lo + width, u)
    # a fraction of coordinates straddle 0 (where the domain allows)
    strad = rng.uniform(0, 1, (nbox, n)) < 0.1
    ok = (l < 0) & (u > 0)
    lo2 = np.maximum(-rng.uniform(0, 1, (nbox, n)) * np.minimum(-l, 1.0), l)
    hi2 = np.minimum(rng.uniform(0, 1, (nbox, n)) * np.minimum(u, 1.0), u)
    lo = np.where(strad & ok, lo2, lo)
    hi = np.where(strad & ok, hi2, hi)
    return np.ascontiguousarray(lo), np.ascontiguousarray(hi)


def random_points_in(seed: int, lo, hi, k: int):
    """k uniform points in each box (lo, hi of shape (nbox, n)) -> (nbox, k, n)."""
    rng = np.random.default_rng(seed)
    lo = np.asarray(lo)
    hi = np.asarray(hi)
    t = rng.uniform(0, 1, (lo.shape[0], k, lo.shape[1]))
    return lo[:, None, :] + t * (hi - lo)[:, None, :]
