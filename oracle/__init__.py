"""CPU oracle for the interval branch-and-bound hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2507_01770_b200`` never imports it and
shares no code with it (no kernels, headers, constants or helpers).

The C sources (ia.c, fns.c, bnb.c) follow PAPER.md §2.1 (interval operations,
Eq. 3-6), Appendix A (the ten objective functions) and §3.1-3.2 (the
branch-and-bound flowchart, partition Eq. 8-11 and variable cycling).  Rounding
is IEEE directed rounding through ``fesetround``; libm transcendentals are
widened outward by ``IA_LIBM_ULPS`` ulps.

Pinning status of every function is listed in DESIGN.md ("Oracle pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

FUNCS = {
    0: "example",
    1: "ackley",
    2: "belegundu",
    3: "breiman",
    4: "fu",
    5: "griewank",
    6: "levy",
    7: "rastrigin",
    8: "salomon",
    9: "styblinski",
    10: "zabinsky",
}
CODE_WHOLE = -1

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_lp = ctypes.POINTER(ctypes.c_long)


class SolveResult(ctypes.Structure):
    _fields_ = [
        ("glb", ctypes.c_double),
        ("gub", ctypes.c_double),
        ("iters", ctypes.c_long),
        ("evals", ctypes.c_long),
        ("n_surv", ctypes.c_long),
        ("status", ctypes.c_int),
    ]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (make)."""
    srcs = [os.path.join(_HERE, f) for f in ("ia.c", "fns.c", "bnb.c", "search.c", "ia.h", "oracle.h")]
    if (
        not force
        and os.path.exists(_LIB_PATH)
        and all(os.path.getmtime(_LIB_PATH) >= os.path.getmtime(s) for s in srcs)
    ):
        return _LIB_PATH
    subprocess.run(["make", "-s", "-B", "liboracle.so"], cwd=_HERE, check=True)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            L.or_init.restype = ctypes.c_int
            L.or_eval_box.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp, _dp]
            L.or_eval_point.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp]
            L.or_grad_box.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp, ctypes.c_int, _dp]
            L.or_child_box.argtypes = [ctypes.c_int, _dp, _dp, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_long, _dp, _dp]
            L.or_branch.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp, _ip,
                                    ctypes.c_int, ctypes.c_int, _dp, _dp, ctypes.c_int,
                                    ctypes.c_double, _dp, ctypes.c_long, _ip, _lp, _dp, _dp,
                                    _lp]
            L.or_solve.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp, ctypes.c_double,
                                   ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_long,
                                   ctypes.c_int, ctypes.c_long, ctypes.c_long, ctypes.c_int,
                                   _dp, _dp, _dp, ctypes.POINTER(SolveResult)]
            L.or_search_candidate.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                              ctypes.c_int, _dp]
            L.or_search_propose.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp, _dp,
                                            ctypes.c_double, _dp, _dp]
            L.or_search_diag.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, _dp]
            L.or_search.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp, ctypes.c_int, _dp, _dp,
                                    _ip]
            L.or_set_trace.argtypes = [_dp, ctypes.c_long]
            L.or_set_trace.restype = None
            L.or_trace_len.restype = ctypes.c_long
            for fn in ("ia_add_dn", "ia_add_up", "ia_sub_dn", "ia_sub_up", "ia_mul_dn",
                       "ia_mul_up", "ia_div_dn", "ia_div_up"):
                getattr(L, fn).argtypes = [ctypes.c_double, ctypes.c_double]
                getattr(L, fn).restype = ctypes.c_double
            L.or_init()
            _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- intervals
class _IA(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_double), ("hi", ctypes.c_double)]


def _ia_fn(name, nargs):
    L = lib()
    f = getattr(L, name)
    f.restype = _IA
    f.argtypes = [_IA] * nargs
    return f


def ia(name: str, *args):
    """Call an interval primitive of ia.c, e.g. ia('ia_cos', (0.0, 1.0))."""
    f = _ia_fn(name, len(args))
    r = f(*[_IA(float(a[0]), float(a[1])) for a in args])
    return (r.lo, r.hi)


def consts() -> dict:
    L = lib()

    class C(ctypes.Structure):
        _fields_ = [(k, _IA) for k in ("pi", "e", "c0_02", "c0_1", "c0_9")]

    c = C.in_dll(L, "IA_C")
    return {k: (getattr(c, k).lo, getattr(c, k).hi) for k in ("pi", "e", "c0_02", "c0_1", "c0_9")}


# ---------------------------------------------------------------- functions
def eval_box(fid: int, lo, hi):
    lo, hi = _f64(lo), _f64(hi)
    out = np.zeros(2)
    rc = lib().or_eval_box(fid, lo.size, _d(lo), _d(hi), _d(out))
    if rc:
        raise ValueError(f"or_eval_box rc={rc}")
    return float(out[0]), float(out[1])


def eval_point(fid: int, x):
    x = _f64(x)
    out = np.zeros(2)
    rc = lib().or_eval_point(fid, x.size, _d(x), _d(out))
    if rc:
        raise ValueError(f"or_eval_point rc={rc}")
    return float(out[0]), float(out[1])


def grad_box(fid: int, lo, hi, i: int):
    lo, hi = _f64(lo), _f64(hi)
    out = np.zeros(2)
    rc = lib().or_grad_box(fid, lo.size, _d(lo), _d(hi), int(i), _d(out))
    if rc:
        raise ValueError(f"or_grad_box rc={rc}")
    return float(out[0]), float(out[1])


def child_box(plo, phi, cyc: int, d: int, m: int, code: int):
    plo, phi = _f64(plo), _f64(phi)
    n = plo.size
    clo, chi = np.zeros(n), np.zeros(n)
    lib().or_child_box(n, _d(plo), _d(phi), int(cyc), int(d), int(m), int(code), _d(clo), _d(chi))
    return clo, chi


def _mono(mono) -> int:
    """first-order test mode: False/0 off, True/1 the split variables
    (R4), 2 every variable (PAPER.md lines 142-144 as printed)"""
    return 2 if mono == 2 else int(bool(mono))


def branch(fid, plo, phi, pcyc, d, m, l, u, mono=True, gub_in=float("inf")):
    """One branch-and-bound iteration on an explicit batch of parent boxes.

    Returns (gub, parent[], code[], lb[], w[]) of the surviving children.
    """
    plo, phi = _f64(plo), _f64(phi)
    nb, n = plo.shape
    pcyc = np.ascontiguousarray(pcyc, dtype=np.int32)
    l, u = _f64(l), _f64(u)
    cap = nb * int(m) ** int(d)
    par = np.zeros(cap, np.int32)
    code = np.zeros(cap, np.int64)
    lb = np.zeros(cap)
    w = np.zeros(cap)
    cnt = ctypes.c_long(0)
    gub = ctypes.c_double(0.0)
    rc = lib().or_branch(fid, n, nb, _d(plo), _d(phi), pcyc.ctypes.data_as(_ip), int(d), int(m),
                         _d(l), _d(u), _mono(mono), float(gub_in), ctypes.byref(gub), cap,
                         par.ctypes.data_as(_ip), code.ctypes.data_as(_lp), _d(lb), _d(w),
                         ctypes.byref(cnt))
    if rc < 0:
        raise ValueError(f"or_branch rc={rc}")
    k = cnt.value
    return gub.value, par[:k], code[:k], lb[:k], w[:k]


def solve(fid, l, u, eps_f=1e-6, eps_x=1e-6, d=10, m=2, bmax=4096, mono=True,
          max_iter=10_000, cap=1 << 16, search=0):
    l, u = _f64(l), _f64(u)
    n = l.size
    slo = np.zeros((cap, n))
    shi = np.zeros((cap, n))
    slb = np.zeros(cap)
    res = SolveResult()
    rc = lib().or_solve(fid, n, _d(l), _d(u), float(eps_f), float(eps_x), int(d), int(m),
                        int(bmax), _mono(mono), int(max_iter), int(cap), int(search),
                        _d(slo), _d(shi),
                        _d(slb), ctypes.byref(res))
    if rc < 0:
        raise ValueError(f"or_solve rc={rc}")
    k = min(res.n_surv, cap)
    return {
        "glb": res.glb,
        "gub": res.gub,
        "iters": res.iters,
        "evals": res.evals,
        "n_surv": res.n_surv,
        "status": res.status,
        "lo": slo[:k],
        "hi": shi[:k],
        "lb": slb[:k],
    }


def solve_trace(fid, l, u, cap=1 << 20, **kw):
    """or_solve with the per-iteration trace of bnb.c (test pins only).

    Returns (solve result, [ {lbs, sel, gub_before, gub_after}, ... ])."""
    buf = np.zeros(cap)
    lib().or_set_trace(_d(buf), cap)
    try:
        r = solve(fid, l, u, **kw)
        used = lib().or_trace_len()
    finally:
        lib().or_set_trace(None, 0)
    if used > cap:
        raise ValueError("trace buffer too small")
    recs, k = [], 0
    while k < used:
        pn = int(buf[k]); k += 1
        lbs = buf[k:k + pn].copy(); k += pn
        nb = int(buf[k]); k += 1
        sel = [int(v) for v in buf[k:k + nb]]; k += nb
        g0, g1 = float(buf[k]), float(buf[k + 1]); k += 2
        recs.append({"lbs": lbs, "sel": sel, "gub_before": g0, "gub_after": g1})
    return r, recs


# ---------------------------------------------------------------- search (R9)
SEARCH_GRID, SEARCH_SCALES, SEARCH_ALPHAS = 32, 48, 8
SEARCH_CANDS = SEARCH_GRID + 2 * SEARCH_SCALES


def search_candidate(xi: float, li: float, ui: float, c: int):
    """Candidate c of one variable (reading R9), None when outside [li, ui]."""
    p = ctypes.c_double()
    ok = lib().or_search_candidate(float(xi), float(li), float(ui), int(c), ctypes.byref(p))
    return p.value if ok else None


def search_propose(fid, x, l, u, fcur):
    """One proposal step of the R9 search: (xs, fb)."""
    x, l, u = _f64(x), _f64(l), _f64(u)
    xs = np.zeros_like(x)
    fb = np.zeros_like(x)
    lib().or_search_propose(fid, x.size, _d(x), _d(l), _d(u), float(fcur), _d(xs), _d(fb))
    return xs, fb


def search_diag(fid, l, u):
    """R9 diagonal line search: (t*, f_upper at x(t*))."""
    l, u = _f64(l), _f64(u)
    t = ctypes.c_double()
    f = ctypes.c_double()
    lib().or_search_diag(fid, l.size, _d(l), _d(u), ctypes.byref(t), ctypes.byref(f))
    return t.value, f.value


def search(fid, l, u, rounds=32):
    """R9 coordinate pattern search from the midpoint: (x, f_upper, rounds)."""
    l, u = _f64(l), _f64(u)
    x = np.zeros_like(l)
    f = ctypes.c_double()
    r = ctypes.c_int()
    lib().or_search(fid, l.size, _d(l), _d(u), int(rounds), _d(x), ctypes.byref(f), ctypes.byref(r))
    return x, f.value, r.value
