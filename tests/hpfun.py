"""The objective functions of PAPER.md Appendix A (A1)-(A20) and the §2.1
example (line 75), evaluated at a POINT in 50-digit decimal arithmetic with
the textbook series of tests/hp.py.  Written from the paper's formulas, not
from the oracle or the CUDA code (no shared code): it is the "true value"
f(x) that every interval enclosure at or around x must contain.

Numbers of the fid convention (include/ibnb.h): 0 example, 1 Ackley,
2 Belegundu, 3 Breiman, 4 Fu, 5 Griewank, 6 Levy, 7 Rastrigin, 8 Salomon,
9 Styblinski, 10 Zabinsky."""
from __future__ import annotations

from decimal import Decimal

from tests import hp


def _D(v) -> Decimal:
    return Decimal(float(v))  # exact value of the binary64 input


def f(fid: int, x) -> Decimal:
    x = [_D(v) for v in x]
    n = len(x)
    pi = hp.PI
    if fid == 0:  # line 75: x - x^2, summed
        return sum((v - v * v for v in x), Decimal(0))
    if fid == 1:  # (A1)
        s1 = sum((v * v for v in x), Decimal(0)) / n
        s2 = sum((hp.dcos(2 * pi * v) for v in x), Decimal(0)) / n
        return -20 * hp.dexp(Decimal("-0.02") * hp.dsqrt(s1)) - hp.dexp(s2) + 20 + hp.E
    if fid == 2:  # (A3)
        s = sum(((v - 5) ** 2 for v in x), Decimal(0))
        return Decimal("0.1") * s - hp.dcos(5 * hp.dsqrt(s))
    if fid == 3:  # (A5)
        return -Decimal("0.1") * sum((hp.dcos(5 * pi * v) for v in x), Decimal(0)) + sum(
            (v * v for v in x), Decimal(0))
    if fid == 4:  # (A7), the sum covering all three terms (R3)
        s = Decimal(1)
        for v in x:
            g2 = (v - Decimal("0.9")) ** 2
            s += 8 * hp.dsin(7 * g2) ** 2 + 6 * hp.dsin(14 * g2) ** 2 + g2
        return s
    if fid == 5:  # (A9), i 1-based
        s = sum((v * v for v in x), Decimal(0)) / 4000
        p = Decimal(1)
        for i, v in enumerate(x, start=1):
            p *= hp.dcos(v / hp.dsqrt(i))
        return 1 + s - p
    if fid == 6:  # (A11)-(A12)
        y = [1 + Decimal("0.25") * (v - 1) for v in x]
        acc = 10 * hp.dsin(pi * y[0]) ** 2 + (y[-1] - 1) ** 2
        for i in range(n - 1):
            acc += (y[i] - 1) ** 2 * (1 + 10 * hp.dsin(pi * y[i + 1]) ** 2)
        return pi / n * acc
    if fid == 7:  # (A14)
        return 10 * n + sum((v * v - 10 * hp.dcos(2 * pi * v) for v in x), Decimal(0))
    if fid == 8:  # (A16)
        r = hp.dsqrt(sum((v * v for v in x), Decimal(0)))
        return 1 - hp.dcos(2 * pi * r) + Decimal("0.1") * r
    if fid == 9:  # (A18)
        s = sum((v * v for v in x), Decimal(0)) / (2 * n)
        p = Decimal(1)
        for v in x:
            p *= hp.dcos(v)
        return s - 4 * n * p
    if fid == 10:  # (A20)
        p1 = Decimal(1)
        p2 = Decimal(1)
        for v in x:
            p1 *= hp.dsin(v - pi / 6)
            p2 *= hp.dsin(5 * (v - pi / 6))
        return Decimal("-2.5") * p1 - p2
    raise ValueError(fid)
