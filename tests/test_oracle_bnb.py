"""Pins for the oracle's branch-and-bound (§3.1-3.2) against what the
paper fixes: the Fig. 3 / Eq. (8)-(11) indexing example, exact coverage of a
parent by its subregions, the variable-cycling schedule (line 184), the
invariant that no ruled-out subregion contains a point better than the
incumbent, and enclosure of the known global minimum (Appendix A)."""
from __future__ import annotations

import json
import math
import os

import numpy as np
import pytest

import oracle
import workloads
from tests import hp

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_partition_indexing_fig3():
    g = json.load(open(os.path.join(GOLD, "partition_fig3.json")))
    plo = np.array(g["selected"]["lo"])
    phi = np.array(g["selected"]["hi"])
    for r in range(g["m"] ** g["d"]):
        lo, hi = oracle.child_box(plo, phi, 0, g["d"], g["m"], r)
        assert list(lo) == [r % 4, r // 4]        # Eq. (8)-(9)
        assert list(hi) == [r % 4 + 1, r // 4 + 1]  # Eq. (10)-(11)


@pytest.mark.parametrize("m", [2, 3, 4, 5])
def test_children_cover_parent_exactly(m):
    rng = np.random.default_rng(m)
    for _ in range(30):
        n = int(rng.integers(1, 6))
        d = int(rng.integers(1, n + 1))
        cyc = int(rng.integers(0, n))
        plo = rng.uniform(-10, 10, n)
        phi = plo + 10.0 ** rng.uniform(-14, 1, n)
        dims = [(cyc + j) % n for j in range(d)]
        pieces = {dim: set() for dim in dims}
        for c in range(m ** d):
            lo, hi = oracle.child_box(plo, phi, cyc, d, m, c)
            assert np.all(lo <= hi)
            for i in range(n):
                if i not in dims:
                    assert lo[i] == plo[i] and hi[i] == phi[i]
            for dim in dims:
                pieces[dim].add((lo[dim], hi[dim]))
        for dim in dims:
            iv = sorted(pieces[dim])
            assert iv[0][0] == plo[dim] and iv[-1][1] == phi[dim]  # end points exact
            for a, b in zip(iv, iv[1:]):
                assert a[1] == b[0]  # no gap, no overlap between neighbours


def test_variable_cycling_dims_split():
    # n = 25, d = 10: cycling index 20 splits x21..x25 and wraps to x1..x5
    n, d, m = 25, 10, 2
    plo, phi = np.zeros(n), np.ones(n)
    split = set()
    for c in range(m ** d):
        lo, hi = oracle.child_box(plo, phi, 20, d, m, c)
        split |= {i for i in range(n) if hi[i] - lo[i] < 1.0}
    assert split == set(range(20, 25)) | set(range(0, 5))


@pytest.mark.parametrize("fid", list(range(1, 11)))
def test_branch_ruled_out_boxes_hold_no_better_point(fid):
    n, d, m = 3, 3, 2
    l, u = workloads.bounds(fid, n)
    plo, phi = workloads.random_boxes(300 + fid, n, 6, l, u, mix=(0, 0, 0.2, 0.4, 0.4, 0))
    cyc = np.array([0, 1, 2, 0, 1, 2], np.int32)
    gub, par, code, lb, w = oracle.branch(fid, plo, phi, cyc, d, m, l, u, mono=True)
    surv = set(zip(par.tolist(), code.tolist()))
    assert math.isfinite(gub)  # its value is pinned by test_branch_gub_is_upper_end_*
    rng = np.random.default_rng(fid)
    for b in range(plo.shape[0]):
        for c in range(m ** d):
            clo, chi = oracle.child_box(plo[b], phi[b], int(cyc[b]), d, m, c)
            e = oracle.eval_box(fid, clo, chi)
            if (b, c) in surv:
                assert e[0] <= gub
                continue
            pts = clo + rng.uniform(0, 1, (12, n)) * (chi - clo)
            if e[0] > gub:
                # ruled out by the bound: every point is worse than GUB
                for p in pts:
                    assert oracle.eval_point(fid, p)[0] > gub
            else:
                # ruled out by the first-order test: some split variable has a
                # derivative of constant sign and the box is not on that edge
                ok = False
                for j in range(d):
                    i = (int(cyc[b]) + j) % n
                    g = oracle.grad_box(fid, clo, chi, i)
                    if (g[0] > 0 and clo[i] != l[i]) or (g[1] < 0 and chi[i] != u[i]):
                        ok = True
                assert ok


def _xstar(fid, n):
    return np.full(n, {1: 0.0, 2: 5.0, 3: 0.0, 4: 0.9, 5: 0.0, 6: 1.0, 7: 0.0, 8: 0.0, 9: 0.0,
                       10: 2 * math.pi / 3}[fid])


def _fstar(fid, n):
    return {1: 0.0, 2: -1.0, 3: -0.1 * n, 4: 1.0, 5: 0.0, 6: 0.0, 7: 0.0, 8: 0.0, 9: -4.0 * n,
            10: -3.5}[fid]


def test_config0_rastrigin_n2_encloses_global_minimum():
    cfg = workloads.CONFIGS[0]
    l, u = workloads.config_bounds(cfg)
    r = oracle.solve(cfg["fid"], l, u, eps_f=cfg["eps"], eps_x=cfg["eps"], d=2, m=2)
    assert r["status"] == 0
    assert r["glb"] <= 0.0 <= r["gub"] and r["gub"] - r["glb"] <= 1e-6
    assert np.all(r["hi"] - r["lo"] <= 1e-6)
    assert any(np.all(lo <= 0) and np.all(0 <= hi) for lo, hi in zip(r["lo"], r["hi"]))


@pytest.mark.parametrize("fid", list(range(1, 11)))
def test_small_solves_enclose_known_minimum_paper_domains(fid):
    n = 2
    l, u = workloads.bounds(fid, n)
    r = oracle.solve(fid, l, u, eps_f=1e-6, eps_x=1e-5, d=2, m=2, bmax=256, max_iter=4000)
    assert r["status"] == 0, r["status"]
    fs = _fstar(fid, n)
    tol = 1e-12 * max(1, abs(fs)) * 10
    assert r["glb"] - tol <= fs <= r["gub"] + tol
    assert r["gub"] - r["glb"] <= 1e-6
    xs = _xstar(fid, n)
    assert any(np.all(lo <= xs + 1e-15) and np.all(xs - 1e-15 <= hi)
               for lo, hi in zip(r["lo"], r["hi"])), "minimizer not in any surviving box"


def test_incumbent_monotone_and_minimizer_kept_every_iteration():
    fid, n = 6, 2
    l, u = workloads.bounds(fid, n)
    prev = math.inf
    xs = _xstar(fid, n)
    for k in range(1, 30, 3):
        r = oracle.solve(fid, l, u, eps_f=0, eps_x=0, d=2, m=2, bmax=64, max_iter=k)
        assert r["gub"] <= prev
        prev = r["gub"]
        assert r["glb"] <= 0.0 <= r["gub"]
        assert any(np.all(lo <= xs) and np.all(xs <= hi) for lo, hi in zip(r["lo"], r["hi"]))


# ------------------------------------------------ selection rule (line 130)
@pytest.mark.parametrize("fid,bmax", [(7, 1), (6, 1), (1, 1), (7, 3), (5, 3), (8, 2), (2, 2)])
def test_selection_takes_smallest_lower_bounds(fid, bmax):
    """PAPER.md §3.1: the region with the smallest lower bound is
    selected (batched, R1: the bmax smallest by (lb, position)).
    The trace gives the list L in list order at every selection; the test
    recomputes the argmin itself, so a reversed or otherwise wrong order in
    the oracle's rec_cmp fails here."""
    n = 2
    l, u = workloads.bounds(fid, n)
    r, recs = oracle.solve_trace(fid, l, u, eps_f=1e-6, eps_x=1e-6, d=2, m=2, bmax=bmax,
                                 max_iter=40)
    multi = 0
    for rec in recs:
        lbs = rec["lbs"]
        nb = min(len(lbs), bmax)
        want = sorted(range(len(lbs)), key=lambda k: (lbs[k], k))[:nb]
        assert sorted(rec["sel"]) == sorted(want)
        assert rec["sel"] == sorted(rec["sel"])  # processed in list order
        if len(lbs) > nb and len(set(lbs.tolist())) > 1:
            multi += 1
    assert multi >= 3, "trace never offered a real choice"


# ------------------------------------------- incumbent rigour (line 134)
def _hp_rastrigin(x):
    """f(x) of (A14) at a point in 50-digit arithmetic (tests/hp.py)."""
    from decimal import Decimal
    s = Decimal(10 * len(x))
    for v in x:
        d = Decimal(float(v))
        s += d * d - 10 * hp.dcos(2 * hp.PI * d)
    return s


@pytest.mark.parametrize("fid", list(range(1, 11)))
def test_branch_gub_is_upper_end_at_best_child_midpoint(fid):
    """GUB is the smallest UPPER bound of the interval
    evaluation of f at the sample points (here every child midpoint, reading
    R2), so f* <= GUB.  Children come from child_box (pinned by Fig. 3), the
    midpoint a + (b - a) / 2 is recomputed here in round-to-nearest, and the
    value is the upper end of eval_point (pinned by the closed forms); the
    lower end would differ (checked: the pin can tell .lo from .hi)."""
    n, d, m = 3, 3, 2
    l, u = workloads.bounds(fid, n)
    plo, phi = workloads.random_boxes(900 + fid, n, 4, l, u, mix=(0, 0, 0.2, 0.4, 0.4, 0))
    cyc = np.array([0, 1, 2, 1], np.int32)
    gub, *_ = oracle.branch(fid, plo, phi, cyc, d, m, l, u, mono=True)
    best_hi, best_lo = math.inf, math.inf
    for b in range(plo.shape[0]):
        for c in range(m ** d):
            clo, chi = oracle.child_box(plo[b], phi[b], int(cyc[b]), d, m, c)
            mid = np.array([min(max(a + (z - a) * 0.5, a), z) for a, z in zip(clo, chi)])
            e = oracle.eval_point(fid, mid)
            best_hi = min(best_hi, e[1])
            best_lo = min(best_lo, e[0])
    assert gub == best_hi
    assert best_lo < best_hi  # a GUB taken from the lower end would fail above


def test_branch_gub_bounds_true_value_rastrigin():
    """The incumbent is a rigorous upper bound of f at a feasible point:
    GUB >= f(x) in 50 digits at the midpoint that attains it (Rastrigin A14)."""
    fid, n, d, m = 7, 3, 3, 2
    l, u = workloads.bounds(fid, n)
    plo, phi = workloads.random_boxes(77, n, 3, l, u, mix=(0, 0, 0.2, 0.4, 0.4, 0))
    cyc = np.zeros(3, np.int32)
    gub, *_ = oracle.branch(fid, plo, phi, cyc, d, m, l, u, mono=True)
    from fractions import Fraction
    hit = 0
    for b in range(plo.shape[0]):
        for c in range(m ** d):
            clo, chi = oracle.child_box(plo[b], phi[b], 0, d, m, c)
            mid = [min(max(a + (z - a) * 0.5, a), z) for a, z in zip(clo, chi)]
            true = _hp_rastrigin(mid)
            e = oracle.eval_point(fid, np.array(mid))
            assert hp.contains(e, true)
            if e[1] == gub:
                hit += 1
                assert Fraction(gub) >= Fraction(true)
                assert Fraction(e[0]) < Fraction(true)  # the lower end is not a bound
    assert hit >= 1


def test_solve_trace_gub_monotone_and_attained():
    """Over a whole solve the incumbent never increases (line 134: best sample
    in all previous iterations and the current one)."""
    fid, n = 6, 2
    l, u = workloads.bounds(fid, n)
    r, recs = oracle.solve_trace(fid, l, u, eps_f=1e-6, eps_x=1e-6, d=2, m=2, bmax=2,
                                 max_iter=60)
    prev = math.inf
    for rec in recs:
        assert rec["gub_before"] <= prev
        assert rec["gub_after"] <= rec["gub_before"]
        prev = rec["gub_after"]
    assert r["gub"] == prev


# ------------------------------ first-order test over every variable (R4)
def test_first_order_all_variables_prunes_on_an_unsplit_variable():
    """PAPER.md lines 142-144 test "any i in {1, ..., n}".  Rastrigin (A14),
    n = 2, d = 1: the parent is split along x_1 only; x_2 in [0.1, 0.2] is
    unsplit, interior and f is increasing in it there (2 x + 20 pi sin(2 pi x)
    > 0 on (0, 0.25)), so mono = 2 rules out every child and mono = 1 (split
    variable only, R4) keeps those the bound keeps.  A loop that
    stopped at the split variables would fail the first assertion."""
    fid, n, d, m = 7, 2, 1, 2
    l, u = workloads.bounds(fid, n)
    plo, phi = np.array([[-0.5, 0.1]]), np.array([[0.5, 0.2]])
    cyc = np.zeros(1, np.int32)
    assert oracle.grad_box(fid, plo[0], phi[0], 1)[0] > 0.0
    g2, par2, *_ = oracle.branch(fid, plo, phi, cyc, d, m, l, u, mono=2)
    g1, par1, *_ = oracle.branch(fid, plo, phi, cyc, d, m, l, u, mono=1)
    assert len(par2) == 0
    assert len(par1) > 0


@pytest.mark.parametrize("fid", list(range(1, 11)))
def test_first_order_all_variables_superset_and_justified(fid):
    """mono = 2 rules out a superset of mono = 1, and every child only it
    rules out has a variable outside the split chunk with a sign-definite
    derivative (or_grad_box) off the domain edge."""
    n, d, m = 4, 2, 2
    l, u = workloads.bounds(fid, n)
    plo, phi = workloads.random_boxes(500 + fid, n, 8, l, u, mix=(0, 0, 0.3, 0.4, 0.3, 0))
    cyc = np.array([0, 1, 2, 3, 0, 1, 2, 3], np.int32)
    _, p1, c1, *_ = oracle.branch(fid, plo, phi, cyc, d, m, l, u, mono=1)
    _, p2, c2, *_ = oracle.branch(fid, plo, phi, cyc, d, m, l, u, mono=2)
    s1 = set(zip(p1.tolist(), c1.tolist()))
    s2 = set(zip(p2.tolist(), c2.tolist()))
    assert s2 <= s1
    for b, c in s1 - s2:
        clo, chi = oracle.child_box(plo[b], phi[b], int(cyc[b]), d, m, c)
        split = {(int(cyc[b]) + j) % n for j in range(d)}
        ok = False
        for i in set(range(n)) - split:
            g = oracle.grad_box(fid, clo, chi, i)
            if (g[0] > 0 and clo[i] != l[i]) or (g[1] < 0 and chi[i] != u[i]):
                ok = True
        assert ok


@pytest.mark.parametrize("fid,search", [(0, 0), (3, 0), (4, 32), (7, 0), (7, 32)])
def test_first_order_split_only_equals_all_variables_for_separable(fid, search):
    """For a separable objective d f / d x_i depends on x_i alone, and every
    variable of a region of L was tested (as a split variable) when it took
    its current range, or still spans [l_i, u_i] (on the edge): the split-only
    test of R4 and the test over all n variables give the same solve."""
    n, d = 6, 2
    l, u = workloads.bounds(fid, n)
    r1 = oracle.solve(fid, l, u, 1e-6, 1e-6, d=d, m=2, bmax=16, mono=1, search=search, max_iter=3000)
    r2 = oracle.solve(fid, l, u, 1e-6, 1e-6, d=d, m=2, bmax=16, mono=2, search=search, max_iter=3000)
    assert r1["status"] == r2["status"]
    assert (r1["iters"], r1["evals"], r1["n_surv"]) == (r2["iters"], r2["evals"], r2["n_surv"])
    np.testing.assert_array_equal(r1["lo"], r2["lo"])
    np.testing.assert_array_equal(r1["hi"], r2["hi"])
