"""Pins for the oracle's coordinate pattern search (reading R9,
oracle/search.c), the sampling strategy that supplies the initial incumbent
(§3.1: any sample point is acceptable, GUB is the
smallest upper bound of f over the sampled points).

What fixes it independently of the oracle's own arithmetic:
  * candidate generation: exact rationals (grid points of [l, u], dyadic
    pattern steps) computed with fractions;
  * proposals: for a separable sum (Rastrigin, A14) the best value of x_i with
    the other variables fixed is the argmin of the 1-D term
    x^2 - 10 cos(2 pi x), evaluated here with 50-digit Taylor series;
  * results: the returned value is an upper bound of f at the returned point
    (50-digit evaluation) and reaches the stated global minima of Appendix A
    (tests/golden/paper_minima.json) for the functions whose minimiser a
    coordinate search can reach from the domain midpoint.
"""
from __future__ import annotations

import json
import os
from decimal import Decimal
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads
from tests import hp

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_candidates_are_grid_and_dyadic_steps():
    rng = np.random.default_rng(7)
    for _ in range(200):
        li = float(rng.uniform(-100, 10))
        ui = li + float(10.0 ** rng.uniform(-3, 2))
        xi = float(rng.uniform(li, ui))
        span = ui - li  # the oracle's rounded span, as R9 states
        for c in range(oracle.SEARCH_CANDS):
            p = oracle.search_candidate(xi, li, ui, c)
            if c < oracle.SEARCH_GRID:
                if c == oracle.SEARCH_GRID - 1:
                    assert p == ui
                    continue
                w = span / 31.0
                exact = Fraction(li) + Fraction(w) * c
                assert p is not None and li <= p <= ui
                # two roundings (product, sum): bounded by the operands' magnitude
                bound = (abs(Fraction(li)) + abs(Fraction(w) * c)) * Fraction(1, 2**52)
                assert abs(Fraction(p) - exact) <= bound + Fraction(1, 2**1074)
            else:
                j = (c - 32) // 2 + 1
                step = Fraction(span) / 2**j
                exact = Fraction(xi) + (step if c & 1 else -step)
                if exact < li or exact > ui:
                    # outside: skipped (the rounded candidate may land on the bound)
                    assert p is None or p in (li, ui)
                else:
                    assert p is not None
                    bound = (abs(Fraction(xi)) + step) * Fraction(1, 2**53)
                    assert abs(Fraction(p) - exact) <= bound + Fraction(1, 2**1074)


def _ras_term(x: float) -> Decimal:
    d = Decimal(x)
    return d * d - 10 * hp.dcos(2 * hp.PI * d)


def test_proposal_is_the_coordinatewise_argmin_rastrigin():
    """Separable sum: the proposal for x_i is the candidate minimising the 1-D
    term (the other variables do not move the argmin)."""
    rng = np.random.default_rng(3)
    n = 4
    l, u = workloads.bounds(7, n)
    for _ in range(3):
        x = rng.uniform(l, u)
        fcur = oracle.eval_point(7, x)[1]
        xs, fb = oracle.search_propose(7, x, l, u, fcur)
        for i in range(n):
            cands = [oracle.search_candidate(x[i], l[i], u[i], c) for c in range(oracle.SEARCH_CANDS)]
            vals = sorted((_ras_term(p), c, p) for c, p in enumerate(cands) if p is not None)
            best, second = vals[0], vals[1]
            cur = _ras_term(x[i])
            if best[0] < cur - Decimal("1e-9") and second[0] - best[0] > Decimal("1e-9"):
                assert xs[i] == best[2], (i, xs[i], best)
                assert fb[i] < fcur
            elif best[0] > cur + Decimal("1e-9"):
                assert xs[i] == x[i] and fb[i] == fcur


def _f_hp(fid: int, x) -> Decimal:
    """50-digit value of the Appendix A formula at a point (no oracle code)."""
    X = [Decimal(float(v)) for v in x]
    n = len(X)
    if fid == 7:
        return 10 * n + sum(v * v - 10 * hp.dcos(2 * hp.PI * v) for v in X)
    if fid == 1:
        s1 = sum(v * v for v in X) / n
        s2 = sum(hp.dcos(2 * hp.PI * v) for v in X) / n
        return -20 * hp.dexp(-Decimal("0.02") * s1.sqrt()) - hp.dexp(s2) + 20 + hp.E
    if fid == 9:
        p = Decimal(1)
        for v in X:
            p *= hp.dcos(v)
        return sum(v * v for v in X) / (2 * n) - 4 * n * p
    if fid == 3:
        return -Decimal("0.1") * sum(hp.dcos(5 * hp.PI * v) for v in X) + sum(v * v for v in X)
    raise KeyError(fid)


@pytest.mark.parametrize("fid,n", [(7, 3), (7, 8), (1, 5), (9, 4), (3, 6)])
def test_search_value_is_an_upper_bound_at_its_point(fid, n):
    l, u = workloads.bounds(fid, n)
    x, f, rounds = oracle.search(fid, l, u)
    assert np.all(x >= l) and np.all(x <= u)
    assert rounds >= 0
    true = _f_hp(fid, x)
    assert Decimal(f) >= true  # rigorous: the upper end of an enclosure
    assert Decimal(f) - true <= Decimal("1e-12") * (1 + abs(true)) + Decimal("1e-12") * n
    # no worse than the domain midpoint it starts from
    mid = l + (u - l) * 0.5
    assert f <= oracle.eval_point(fid, mid)[1]


def _fstar(fid: int, n: int) -> float:
    s = json.load(open(os.path.join(GOLD, "paper_minima.json")))["functions"][str(fid)]["fstar"]
    return -0.1 * n if s == "-0.1n" else (-4.0 * n if s == "-4n" else float(s))


# every Appendix A minimiser is x* = c (1, ..., 1), on the diagonal of the
# paper's cube domains, so the diagonal stage reaches it and the coordinate
# stage keeps it
@pytest.mark.parametrize("fid", list(range(1, 11)))
@pytest.mark.parametrize("n", [2, 6])
def test_search_reaches_known_minimum(fid, n):
    l, u = workloads.bounds(fid, n)
    x, f, _ = oracle.search(fid, l, u)
    fs = _fstar(fid, n)
    assert fs <= f <= fs + 1e-9 * (1 + abs(fs)), (fid, n, f, fs)


def test_search_rounds_limit_and_monotone():
    l, u = workloads.bounds(7, 3)
    prev = np.inf
    for r in range(0, 6):
        _, f, done = oracle.search(7, l, u, rounds=r)
        assert done <= r
        assert f <= prev  # more rounds never worsen the incumbent
        prev = f


def test_solve_with_search_encloses_minimum():
    for fid in (7, 1, 9):
        l, u = workloads.bounds(fid, 3)
        r = oracle.solve(fid, l, u, eps_f=1e-6, eps_x=1e-6, d=3, m=2, bmax=64, max_iter=20000, search=32)
        fs = _fstar(fid, 3)
        assert r["status"] == 0
        assert r["glb"] <= fs + 1e-12 and fs <= r["gub"]
        assert r["gub"] - r["glb"] <= 1e-6


@pytest.mark.parametrize("fid", list(range(1, 11)))
def test_diagonal_stage_reaches_known_minimum_n50(fid):
    n = 50
    l, u = workloads.bounds(fid, n)
    t, f = oracle.search_diag(fid, l, u)
    fs = _fstar(fid, n)
    assert 0.0 <= t <= 1.0
    assert fs <= f <= fs + 1e-9 * (1 + abs(fs)), (fid, f, fs)
    # no worse than the domain midpoint (t = 1/2 is a grid point)
    assert f <= oracle.eval_point(fid, l + 0.5 * (u - l))[1]


@pytest.mark.parametrize("fid", [7, 1, 9, 3])
def test_diagonal_value_is_an_upper_bound(fid):
    n = 5
    l, u = workloads.bounds(fid, n)
    t, f = oracle.search_diag(fid, l, u)
    x = np.clip(l + t * (u - l), l, u)
    true = _f_hp(fid, x)
    assert Decimal(f) >= true
    assert Decimal(f) - true <= Decimal("1e-12") * (1 + abs(true)) + Decimal("1e-12") * n
