"""B200-native interval branch-and-bound (arxiv 2507.01770 hot path).

Thin ctypes binding of ``libibnb.so`` (C ABI in ``include/ibnb.h``).  Every
function here only marshals arguments: device memory comes from torch
tensors, every compute step runs in the CUDA kernels of ``csrc/``.  There is
no CPU fallback -- importing works anywhere, but every call raises if the
library or a CUDA device is missing.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

__all__ = [
    "ib_version", "ib_last_error", "ib_num_functions", "IbOptions", "ib_solve", "ib_solve_dev", "ib_solve_dev_ex", "ib_solve_dev_mg",
    "ib_eval_boxes", "ib_eval_grad", "ib_branch", "ib_search", "ib_compact_le", "ib_select", "lib", "LIB_PATH",
]

LIB_PATH = _build.LIB
CODE_WHOLE = 0xFFFFFFFF
_lib = None

NPROF = 8
PROF_CLASSES = ("prep", "child_eval", "cand", "list", "mono", "emit", "fused", "chain")
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_dp = ctypes.POINTER(ctypes.c_double)


class IbOptions(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int), ("m", ctypes.c_int), ("mono", ctypes.c_int), ("profile", ctypes.c_int),
        ("search", ctypes.c_int), ("reserved", ctypes.c_int), ("bmax", _i64), ("max_iter", _i64), ("pool_cap", _i64), ("arch_cap", _i64),
        ("gub_shared", ctypes.c_void_p),
    ]


class IbResult(ctypes.Structure):
    _fields_ = [
        ("f_lo", ctypes.c_double), ("f_hi", ctypes.c_double), ("iters", _i64), ("evals", _i64),
        ("n_surv", _i64), ("peak_pool", _i64), ("max_width", ctypes.c_double),
        ("status", ctypes.c_int), ("n_kernels", ctypes.c_int),
        ("t_ms", ctypes.c_double * NPROF), ("launches", _i64 * NPROF), ("units", _i64 * NPROF),
        ("radix_records", _i64), ("f_search", ctypes.c_double), ("search_rounds", _i64),
        ("rebalanced", _i64), ("transfers", _i64),
    ]


EXPORTS = {
    "ib_version": (ctypes.c_char_p, []),
    "ib_last_error": (ctypes.c_char_p, []),
    "ib_num_functions": (ctypes.c_int, []),
    "ib_solve_workspace_size": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(IbOptions), _i64]),
    "ib_solve": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _dp, _dp, ctypes.c_double, ctypes.c_double,
                               ctypes.POINTER(IbOptions), _vp, ctypes.c_size_t, ctypes.POINTER(IbResult),
                               _dp, _dp, _dp, _i64, _vp]),
    "ib_solve_dev": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, _vp, ctypes.c_double, ctypes.c_double,
                                   ctypes.POINTER(IbOptions), _vp, ctypes.c_size_t, ctypes.POINTER(IbResult),
                                   _vp, _vp, _vp, _i64, _vp]),
    "ib_solve_dev_ex": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, _vp, ctypes.c_double, ctypes.c_double,
                                      ctypes.POINTER(IbOptions), _vp, ctypes.c_size_t, ctypes.POINTER(IbResult),
                                      _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "ib_solve_dev_mg": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, _vp, ctypes.c_double, ctypes.c_double,
                                      ctypes.POINTER(IbOptions), _vp, ctypes.c_size_t, ctypes.POINTER(IbResult),
                                      _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, ctypes.c_int, _vp,
                                      ctypes.c_size_t]),
    "ib_eval_boxes": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _i64, _vp, _vp, _i64, _vp, _vp]),
    "ib_eval_grad": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "ib_branch_workspace_size": (ctypes.c_size_t, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64]),
    "ib_branch": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64,
                                 _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp, _vp, _vp,
                                 _vp, _vp, _vp]),
    "ib_search_workspace_size": (ctypes.c_size_t, [ctypes.c_int]),
    "ib_search": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _vp, _vp, ctypes.c_int, _vp, _vp, _vp, _vp,
                                 ctypes.c_size_t, _vp]),
    "ib_compact_le": (ctypes.c_int, [_vp, _i64, ctypes.c_double, _vp, _vp, _vp, ctypes.c_size_t, _vp]),
    "ib_ipc_get_handle": (ctypes.c_int, [_vp, _vp]),
    "ib_ipc_open": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_void_p)]),
    "ib_ipc_close": (ctypes.c_int, [_vp]),
    "ib_select_workspace_size": (ctypes.c_size_t, [_i64]),
    "ib_select": (ctypes.c_int, [_vp, _i64, ctypes.c_double, _i64, _vp, _vp, ctypes.POINTER(_i64),
                                 ctypes.POINTER(_i64), _vp, ctypes.c_size_t, _vp]),
}


def lib():
    """Load libibnb.so (building it if the sources are newer)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or _build.stale():
            _build.build()
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2507_01770_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _check(rc: int, what: str):
    if rc != 0:
        msg = lib().ib_last_error().decode()
        raise RuntimeError(f"{what} failed (rc={rc}): {msg}")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ib_version() -> str:
    return lib().ib_version().decode()


def ib_last_error() -> str:
    return lib().ib_last_error().decode()


def ib_num_functions() -> int:
    return lib().ib_num_functions()


def options(**kw) -> IbOptions:
    o = IbOptions()
    for k, v in kw.items():
        if v is not None:
            setattr(o, k, int(v))
    return o


@dataclass
class SolveResult:
    f_lo: float
    f_hi: float
    iters: int
    evals: int
    n_surv: int
    peak_pool: int
    max_width: float
    status: int
    lo: object = None
    hi: object = None
    lb: object = None
    prof: dict = None
    n_kernels: int = 0
    f_search: float = float("inf")
    search_rounds: int = 0
    rebalanced: int = 0
    transfers: int = 0


def _res(r: IbResult, lo=None, hi=None, lb=None) -> SolveResult:
    prof = {c: {"ms": r.t_ms[i], "launches": r.launches[i], "units": r.units[i]}
            for i, c in enumerate(PROF_CLASSES)}
    prof["list"]["radix_records"] = r.radix_records
    return SolveResult(r.f_lo, r.f_hi, r.iters, r.evals, r.n_surv, r.peak_pool, r.max_width, r.status,
                       lo, hi, lb, prof, r.n_kernels, r.f_search, r.search_rounds, r.rebalanced, r.transfers)


EXCHANGE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p)
TRANSFER_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t)


class Workspace:
    """Caller-owned device workspace (a torch uint8 tensor), reusable."""

    def __init__(self, nbytes: int, device=None):
        torch = _torch()
        self.t = torch.empty(int(nbytes), dtype=torch.uint8, device=device or "cuda")

    @property
    def nbytes(self):
        return self.t.numel()

    def ptr(self):
        return ctypes.c_void_p(self.t.data_ptr())


def solve_workspace_bytes(fid: int, n: int, opts: IbOptions | None = None, pool_cap: int = 0) -> int:
    o = opts or IbOptions()
    nb = lib().ib_solve_workspace_size(fid, n, ctypes.byref(o), int(pool_cap))
    if nb == 0:
        _check(-1, "ib_solve_workspace_size")
    return int(nb)


def ib_solve(fid: int, l, u, eps_f: float = 1e-6, eps_x: float = 1e-6, opts: IbOptions | None = None,
             surv_cap: int = 1 << 16, workspace: Workspace | None = None, stream=None) -> SolveResult:
    """End-to-end solve with HOST inputs and outputs (numpy)."""
    _torch()
    l = np.ascontiguousarray(l, np.float64)
    u = np.ascontiguousarray(u, np.float64)
    n = l.size
    o = opts or IbOptions()
    ws = workspace or Workspace(solve_workspace_bytes(fid, n, o))
    slo = np.zeros((surv_cap, n))
    shi = np.zeros((surv_cap, n))
    slb = np.zeros(surv_cap)
    r = IbResult()
    rc = lib().ib_solve(fid, n, l.ctypes.data_as(_dp), u.ctypes.data_as(_dp), float(eps_f), float(eps_x),
                        ctypes.byref(o), ws.ptr(), ws.nbytes, ctypes.byref(r), slo.ctypes.data_as(_dp),
                        shi.ctypes.data_as(_dp), slb.ctypes.data_as(_dp), int(surv_cap), _stream(stream))
    _check(rc, "ib_solve")
    k = min(r.n_surv, surv_cap)
    return _res(r, slo[:k], shi[:k], slb[:k])


def ib_solve_dev(fid: int, l, u, eps_f: float = 1e-6, eps_x: float = 1e-6, opts: IbOptions | None = None,
                 surv_cap: int = 0, workspace: Workspace | None = None, stream=None) -> SolveResult:
    """Solve with DEVICE inputs (torch cuda float64 tensors) and device outputs."""
    torch = _torch()
    n = l.numel()
    o = opts or IbOptions()
    ws = workspace or Workspace(solve_workspace_bytes(fid, n, o))
    slo = shi = slb = None
    if surv_cap > 0:
        slo = torch.empty((surv_cap, n), dtype=torch.float64, device=l.device)
        shi = torch.empty_like(slo)
        slb = torch.empty(surv_cap, dtype=torch.float64, device=l.device)
    r = IbResult()
    rc = lib().ib_solve_dev(fid, n, _ptr(l), _ptr(u), float(eps_f), float(eps_x), ctypes.byref(o), ws.ptr(),
                            ws.nbytes, ctypes.byref(r), _ptr(slo), _ptr(shi), _ptr(slb), int(surv_cap),
                            _stream(stream))
    _check(rc, "ib_solve_dev")
    k = min(r.n_surv, surv_cap)
    return _res(r, None if slo is None else slo[:k], None if shi is None else shi[:k],
                None if slb is None else slb[:k])


def ib_solve_dev_ex(fid: int, l, u, exchange, eps_f: float = 1e-6, eps_x: float = 1e-6,
                    opts: IbOptions | None = None, surv_cap: int = 0, workspace: Workspace | None = None,
                    stream=None) -> SolveResult:
    """ib_solve_dev with a per-iteration incumbent exchange.  ``exchange(xchg)``
    receives a cuda float64 tensor of 2 elements and must replace it, in place,
    by its element-wise minimum over all ranks (all_reduce MIN)."""
    torch = _torch()
    n = l.numel()
    o = opts or IbOptions()
    ws = workspace or Workspace(solve_workspace_bytes(fid, n, o))
    xchg = torch.zeros(2, dtype=torch.float64, device=l.device)
    cb = EXCHANGE_FN(lambda _user: exchange(xchg))
    slo = shi = slb = None
    if surv_cap > 0:
        slo = torch.empty((surv_cap, n), dtype=torch.float64, device=l.device)
        shi = torch.empty_like(slo)
        slb = torch.empty(surv_cap, dtype=torch.float64, device=l.device)
    r = IbResult()
    rc = lib().ib_solve_dev_ex(fid, n, _ptr(l), _ptr(u), float(eps_f), float(eps_x), ctypes.byref(o), ws.ptr(),
                               ws.nbytes, ctypes.byref(r), _ptr(slo), _ptr(shi), _ptr(slb), int(surv_cap),
                               _stream(stream), ctypes.cast(cb, ctypes.c_void_p), None, _ptr(xchg))
    _check(rc, "ib_solve_dev_ex")
    k = min(r.n_surv, surv_cap)
    return _res(r, None if slo is None else slo[:k], None if shi is None else shi[:k],
                None if slb is None else slb[:k])


def ib_solve_dev_mg(fid: int, l, u, exchange, transfer, rank: int, eps_f: float = 1e-6, eps_x: float = 1e-6,
                    opts: IbOptions | None = None, surv_cap: int = 0, workspace: Workspace | None = None,
                    tbuf_bytes: int = 64 << 20, stream=None) -> SolveResult:
    """ib_solve_dev with the per-chunk incumbent exchange and box rebalancing.
    ``exchange(xchg)``: replace the cuda float64 tensor of 4 elements by its
    element-wise MIN over all ranks.  ``transfer(src, dst, tbuf, nbytes)``:
    called on every rank; copy the first nbytes of rank src's tbuf (cuda uint8
    tensor) to rank dst's tbuf."""
    torch = _torch()
    n = l.numel()
    o = opts or IbOptions()
    ws = workspace or Workspace(solve_workspace_bytes(fid, n, o))
    xchg = torch.zeros(4, dtype=torch.float64, device=l.device)
    tbuf = torch.empty(int(tbuf_bytes), dtype=torch.uint8, device=l.device)
    cb = EXCHANGE_FN(lambda _user: exchange(xchg))
    tcb = TRANSFER_FN(lambda _user, src, dst, _buf, nbytes: transfer(src, dst, tbuf, int(nbytes)))
    slo = shi = slb = None
    if surv_cap > 0:
        slo = torch.empty((surv_cap, n), dtype=torch.float64, device=l.device)
        shi = torch.empty_like(slo)
        slb = torch.empty(surv_cap, dtype=torch.float64, device=l.device)
    r = IbResult()
    rc = lib().ib_solve_dev_mg(fid, n, _ptr(l), _ptr(u), float(eps_f), float(eps_x), ctypes.byref(o), ws.ptr(),
                               ws.nbytes, ctypes.byref(r), _ptr(slo), _ptr(shi), _ptr(slb), int(surv_cap),
                               _stream(stream), ctypes.cast(cb, ctypes.c_void_p), ctypes.cast(tcb, ctypes.c_void_p),
                               None, _ptr(xchg), int(rank), _ptr(tbuf), int(tbuf_bytes))
    _check(rc, "ib_solve_dev_mg")
    k = min(r.n_surv, surv_cap)
    return _res(r, None if slo is None else slo[:k], None if shi is None else shi[:k],
                None if slb is None else slb[:k])


def ib_eval_boxes(fid: int, lo, hi, stream=None):
    """lo, hi: cuda float64 (nbox, n) -> (nbox, 2) enclosures of f."""
    torch = _torch()
    lo = lo.contiguous()
    hi = hi.contiguous()
    nbox, n = lo.shape
    out = torch.empty((nbox, 2), dtype=torch.float64, device=lo.device)
    _check(lib().ib_eval_boxes(fid, n, nbox, _ptr(lo), _ptr(hi), n, _ptr(out), _stream(stream)), "ib_eval_boxes")
    return out


def ib_eval_grad(fid: int, lo, hi, req_box, req_dim, stream=None):
    torch = _torch()
    lo = lo.contiguous()
    hi = hi.contiguous()
    nbox, n = lo.shape
    rb = req_box.to(torch.int64).contiguous()
    rd = req_dim.to(torch.int32).contiguous()
    out = torch.empty((rb.numel(), 2), dtype=torch.float64, device=lo.device)
    _check(lib().ib_eval_grad(fid, n, rb.numel(), _ptr(lo), _ptr(hi), n, _ptr(rb), _ptr(rd), _ptr(out),
                              _stream(stream)), "ib_eval_grad")
    return out


def ib_branch(fid: int, plo, phi, pcyc, d: int, m: int, l, u, gub: float = float("inf"), mono: bool = True,
              stream=None):
    """One iteration on explicit parents (cuda float64 (nb, n)).  Returns a
    dict of cuda tensors: parent, code, lb, w (survivors) and gub (float)."""
    torch = _torch()
    plo = plo.contiguous()
    phi = phi.contiguous()
    nb, n = plo.shape
    dev = plo.device
    kids = int(m) ** int(d)
    cap = nb * kids
    pc = pcyc.to(torch.int32).contiguous()
    g = torch.tensor([gub], dtype=torch.float64, device=dev)
    out_parent = torch.empty(cap, dtype=torch.int32, device=dev)
    out_code = torch.empty(cap, dtype=torch.int32, device=dev)
    out_lb = torch.empty(cap, dtype=torch.float64, device=dev)
    out_w = torch.empty(cap, dtype=torch.float64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    wsb = lib().ib_branch_workspace_size(fid, n, d, m, nb)
    if wsb == 0:
        _check(-1, "ib_branch_workspace_size")
    ws = torch.empty(int(wsb), dtype=torch.uint8, device=dev)
    _check(lib().ib_branch(fid, n, d, m, int(bool(mono)), nb, _ptr(plo), _ptr(phi), n, _ptr(pc), _ptr(l),
                           _ptr(u), _ptr(g), _ptr(ws), int(wsb), _ptr(out_parent), _ptr(out_code), _ptr(out_lb),
                           _ptr(out_w), _ptr(cnt), _stream(stream)), "ib_branch")
    k = int(cnt.item())
    return {
        "gub": float(g.item()),
        "parent": out_parent[:k],
        "code": out_code[:k].to(torch.int64) & 0xFFFFFFFF,
        "lb": out_lb[:k],
        "w": out_w[:k],
    }


def ib_search(fid: int, l, u, rounds: int = 32, stream=None):
    """Coordinate pattern search (reading R9) on device bounds l, u (cuda
    float64).  Returns (x: cuda tensor, f_upper: float, rounds: int)."""
    torch = _torch()
    n = l.numel()
    x = torch.empty(n, dtype=torch.float64, device=l.device)
    f = torch.empty(1, dtype=torch.float64, device=l.device)
    r = torch.zeros(1, dtype=torch.int32, device=l.device)
    wsb = lib().ib_search_workspace_size(n)
    if wsb == 0:
        _check(-1, "ib_search_workspace_size")
    ws = torch.empty(int(wsb), dtype=torch.uint8, device=l.device)
    _check(lib().ib_search(fid, n, _ptr(l.contiguous()), _ptr(u.contiguous()), int(rounds), _ptr(x), _ptr(f), _ptr(r),
                           _ptr(ws), int(wsb), _stream(stream)), "ib_search")
    return x, float(f.item()), int(r.item())


def ib_compact_le(keys, thr: float, stream=None):
    torch = _torch()
    keys = keys.contiguous()
    n = keys.numel()
    out = torch.empty(max(n, 1), dtype=torch.int64, device=keys.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=keys.device)
    wsb = 8 * (n // 1024 + 2) + 512
    ws = torch.empty(wsb, dtype=torch.uint8, device=keys.device)
    _check(lib().ib_compact_le(_ptr(keys), n, float(thr), _ptr(out), _ptr(cnt), _ptr(ws), wsb, _stream(stream)),
           "ib_compact_le")
    return out[: int(cnt.item())]


def ib_select(lb, gub: float, bmax: int, stream=None):
    torch = _torch()
    lb = lb.contiguous()
    n = lb.numel()
    sel = torch.empty(max(n, 1), dtype=torch.int64, device=lb.device)
    keep = torch.empty(max(n, 1), dtype=torch.int64, device=lb.device)
    ns, nk = _i64(0), _i64(0)
    wsb = lib().ib_select_workspace_size(n)
    ws = torch.empty(int(wsb), dtype=torch.uint8, device=lb.device)
    _check(lib().ib_select(_ptr(lb), n, float(gub), int(bmax), _ptr(sel), _ptr(keep), ctypes.byref(ns),
                           ctypes.byref(nk), _ptr(ws), int(wsb), _stream(stream)), "ib_select")
    return sel[: ns.value], keep[: nk.value]


# ---------------------------------------------------------------- multi-GPU incumbent word
def ib_ipc_get_handle(t) -> bytes:
    """64-byte inter-process handle of the device allocation holding tensor t."""
    _torch()
    h = ctypes.create_string_buffer(64)
    _check(lib().ib_ipc_get_handle(ctypes.c_void_p(t.data_ptr()), ctypes.cast(h, ctypes.c_void_p)), "ib_ipc_get_handle")
    return h.raw


def ib_ipc_open(handle: bytes) -> int:
    """Device address of another process's allocation (ib_ipc_get_handle)."""
    _torch()
    p = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(handle), 64)
    _check(lib().ib_ipc_open(ctypes.cast(buf, ctypes.c_void_p), ctypes.byref(p)), "ib_ipc_open")
    return int(p.value)


def ib_ipc_close(ptr: int) -> None:
    _check(lib().ib_ipc_close(ctypes.c_void_p(ptr)), "ib_ipc_close")
