"""High-precision (50 significant digit) textbook routines used to pin the
oracle's interval primitives: Taylor series for exp / sin / cos after
reduction modulo 2*pi, with pi from Machin's formula.  Independent of libm and
of the oracle (no shared code)."""
from __future__ import annotations

from decimal import Decimal, getcontext
from fractions import Fraction

getcontext().prec = 60


def _arctan_inv(x: int) -> Decimal:
    # arctan(1/x) = sum (-1)^k / ((2k+1) x^(2k+1))
    x = Decimal(x)
    term = 1 / x
    total = term
    k = 0
    x2 = x * x
    while True:
        k += 1
        term /= x2
        t = term / (2 * k + 1)
        if t < Decimal(10) ** -58:
            break
        total += -t if k % 2 else t
    return total


PI = 4 * (4 * _arctan_inv(5) - _arctan_inv(239))  # Machin
E = None  # filled below


def dexp(x) -> Decimal:
    x = Decimal(x)
    # exp(x) = exp(x / 2^k)^(2^k)
    k = 0
    while abs(x) > Decimal("0.5"):
        x /= 2
        k += 1
    s = Decimal(1)
    t = Decimal(1)
    i = 1
    while True:
        t = t * x / i
        if abs(t) < Decimal(10) ** -58:
            break
        s += t
        i += 1
    for _ in range(k):
        s = s * s
    return s


E = dexp(1)


def _reduce(x: Decimal) -> Decimal:
    two_pi = 2 * PI
    q = (x / two_pi).to_integral_value()
    return x - q * two_pi


def dsin(x) -> Decimal:
    x = _reduce(Decimal(x))
    s = Decimal(0)
    t = x
    i = 1
    while abs(t) > Decimal(10) ** -58:
        s += t
        t = -t * x * x / ((i + 1) * (i + 2))
        i += 2
    return s


def dcos(x) -> Decimal:
    x = _reduce(Decimal(x))
    s = Decimal(0)
    t = Decimal(1)
    i = 0
    while abs(t) > Decimal(10) ** -58:
        s += t
        t = -t * x * x / ((i + 1) * (i + 2))
        i += 2
    return s


def dsqrt(x) -> Decimal:
    return Decimal(x).sqrt()


def frac(x) -> Fraction:
    """Exact rational value of a float or a Decimal."""
    if isinstance(x, Decimal):
        return Fraction(x)
    return Fraction(x)


def contains(iv, value) -> bool:
    """Exact check lo <= value <= hi (value: Decimal/float/Fraction)."""
    v = Fraction(value) if not isinstance(value, Fraction) else value
    return Fraction(iv[0]) <= v <= Fraction(iv[1])
