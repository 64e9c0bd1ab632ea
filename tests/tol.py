"""Parity tolerance between the CUDA path and the oracle (DESIGN.md §
"Tolerance"): both evaluate the same natural interval extension with
outward rounding, differing only in summation order, in the libm / libdevice
transcendental kernels (<= 3 ulp each side after widening) and in the t/pi
reduction of general trigonometric arguments.  Every such difference is a
few ulps of the largest intermediate magnitude M of the expression (terms
cancel: Rastrigin's 10n + sum(x^2 - 10 cos) is O(10n) before cancelling), so
the bound is 1e-12 relative to M (north_star: "within 1e-12 relative")."""
from __future__ import annotations

import math

import numpy as np

REL = 1e-12


def magnitude(fid: int, lo, hi) -> float:
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    a = np.maximum(np.abs(lo), np.abs(hi))
    n = a.size
    if fid == 0:
        return float(np.sum(a + a * a))
    if fid == 1:
        return 50.0
    if fid == 2:
        return float(0.1 * np.sum((a + 5) ** 2) + 1)
    if fid == 3:
        return float(0.1 * n + np.sum(a * a))
    if fid == 4:
        return float(1 + np.sum(14 + (a + 0.9) ** 2))
    if fid == 5:
        return float(2 + np.sum(a * a) / 4000)
    if fid == 6:
        u = ((a + 1) / 4) ** 2
        return float(math.pi / n * (10 + 11 * np.sum(u)))
    if fid == 7:
        return float(10 * n + np.sum(a * a + 10))
    if fid == 8:
        return float(2 + 0.2 * math.sqrt(float(np.sum(a * a))) + 1)
    if fid == 9:
        return float(np.sum(a * a) / (2 * n) + 4 * n)
    if fid == 10:
        return 3.5
    raise ValueError(fid)


def grad_magnitude(fid: int, lo, hi) -> float:
    a = np.maximum(np.abs(np.asarray(lo)), np.abs(np.asarray(hi)))
    n = a.size
    base = {0: 3.0, 1: 10.0, 2: 30.0 * (1 + float(np.max(a))), 3: 4 + 2 * float(np.max(a)),
            4: 300 * (1 + float(np.max(a))), 5: 2 + float(np.max(a)) / 2000, 6: 30.0 * (1 + float(np.max(a))) ** 2,
            7: 70 + 2 * float(np.max(a)), 8: 7.0, 9: 4 * n + float(np.max(a)), 10: 8.0}[fid]
    return base


def tol(fid: int, lo, hi) -> float:
    return REL * (1.0 + magnitude(fid, lo, hi))


def gtol(fid: int, lo, hi) -> float:
    return REL * (1.0 + grad_magnitude(fid, lo, hi))
