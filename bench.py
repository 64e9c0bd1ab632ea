#!/usr/bin/env python
"""Benchmark of the interval branch-and-bound hot path (BASELINE.json metric:
box-evaluations per second and time-to-enclose at eps = 1e-6, quoted at
n = 10,000).

One step = one complete solve of the workload (the initial incumbent search
and every iteration of the hot path: select, partition, midpoint sampling +
incumbent, bound + first-order test, compaction) from the root region to the
eps-enclosure.  Default workload: BASELINE.json configs[4] with its Rastrigin
headline, Rastrigin n = 10,000 on the paper's domain [-5.5, 6]^10000 (A15),
eps = 1e-6 -- the metric is quoted at n = 10k and one B200 holds it
(configs[1], Ackley n = 10, is --config 1; configs[0] is the oracle-sized
case).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun), --mode partition (default; north_star): the domain is cut
into N slabs along x_1, one per rank (an exact cover); every rank runs the
hot path on its slab, the incumbent GUB is all-reduced (MIN, NCCL) after
every chunk of iterations (<= 64) and regions are rebalanced (NCCL
send/recv) when the lists skew; the job ends when every rank has its
eps-enclosure and the reported enclosure is the union's -- strong scaling of
one solve (time to enclose).  --mode replicas: every GPU runs its own
independent solve (weak scaling).  Time is the max over ranks of the device
time.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "box-evals/sec"
UNIT = "box-evals/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_PATH = os.path.join(ROOT, "profiles", "fp64_peak_r02.json")
FP64_OPS_PATH = os.path.join(ROOT, "profiles", "fp64_ops_r02.json")

# algorithmic HBM bytes of the memory-bound kernels:
#   list: 12 B (index + lb) per hot entry per pass over the hot index, 8 B per
#         record of L per refill pass, 16 B per record for a width pass;
#   cand: 8 B (child lower bound) per child; emit: 1 + 4 + 8 B per candidate
HBM_BYTES = {
    "list": lambda p: p["units"],  # counted by the kernel (hot-index scans, refills)
    "cand": lambda p: 8 * p["units"],
    "emit": lambda p: 13 * p["units"],
}


def fp64_peak():
    """Measured FP64-pipe peak of this GPU model (scripts/micro/fp64_peak.cu on
    a B200: DADD / DMUL with .RD / .RU rounding, the instructions interval
    arithmetic executes, 64 per SM per clock), in T instructions/s."""
    pk = load_json(FP64_PEAK_PATH) or {}
    if "fp64_tops_dadd_directed" in pk:
        return pk["fp64_tops_dadd_directed"], "measured: profiles/fp64_peak_r02.json (DADD/DMUL .RD/.RU)"
    return 148 * 64 * 1.965e9 / 1e12, "derived: 148 SM x 64 FP64 lanes x 1.965 GHz"


CHAIN_FLOOR_PATH = os.path.join(ROOT, "profiles", "chain_floor_r02l.json")


def latency_roofline(prof):
    """The deep dive's binding resource: time per k_chain iteration against
    the measured floor of its exchange pattern (publish a partial, grid
    barrier, read all partials back, reduce: scripts/micro/chain_floor.cu)."""
    pc = prof.get("chain") or {}
    if not pc.get("units"):
        return None
    fl = load_json(CHAIN_FLOOR_PATH) or {}
    floor = fl.get("grid_148_us_per_iter")
    ach = 1e3 * pc["ms"] / pc["units"]
    return {"kernel": "chain", "unit": "us per iteration", "achieved": ach, "floor": floor,
            "frac": (floor / ach) if floor else None,
            "floor_source": "measured: profiles/chain_floor_r02l.json (148 blocks: publish, grid barrier, "
                            "read all partials, reduce; no arithmetic)"}


def roofline(prof, prof_ms, fid, d=16):
    """Roofline entry of the kernel class with the largest device time:
    executed FP64-pipe instructions per unit of work (ncu, committed in
    profiles/fp64_ops_r02.json for this objective) x units per launch /
    average launch time (CUDA events on the solve stream), against the measured
    FP64-pipe peak; HBM classes against the measured copy bandwidth."""
    dom = max(prof, key=lambda c: prof[c]["ms"])
    pd = prof[dom]
    peaks = load_json(PEAKS_PATH) or {}
    avg_s = pd["ms"] / 1e3 / max(1, pd["launches"])
    if dom in HBM_BYTES:
        hbm = peaks.get("hbm_gbs", 6650.0)
        per_launch = HBM_BYTES[dom](pd) / max(1, pd["launches"])
        ach = per_launch / avg_s / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": None, "algorithmic_bytes_per_launch": per_launch,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650 GB/s"}
    else:
        allops = load_json(FP64_OPS_PATH) or {}
        ent = allops.get(f"{fid}@d{d}") or (allops.get(str(fid)) if d == 16 or dom not in ("chain", "fused") else None)
        ops = (ent or {}).get("kernels", {}).get(dom) or {}
        per_unit = ops.get("fp64_inst_per_unit")
        peak, src = fp64_peak()
        units = pd["units"] / max(1, pd["launches"])
        ach = per_unit * units / avg_s / 1e12 if per_unit else None
        # algorithmic work: the lower bound of every child box, Eq. (3)
        # as tabulated here -- d lower-end additions of the split variables'
        # terms onto the rest + the outer function -- per child box, x 2^d
        # children per deep-dive iteration
        # -- exact for the separable sums whose outer function is one addition
        # (example, Breiman, Fu, Rastrigin); the other objectives' outer
        # functions (exp, sqrt, products) have no op count here, so their
        # line reports the executed count as `achieved`
        kids_per_unit = {"chain": 2 ** d, "fused": 2 ** d, "child_eval": 1}.get(dom)
        algo = kids_per_unit * (d + 1) if kids_per_unit and fid in (0, 3, 4, 7) else None
        ach_algo = algo * units / avg_s / 1e12 if algo else None
        ach_main = ach_algo if ach_algo else ach
        roof = {"bound": "alu", "kernel": dom, "achieved": ach_main, "peak": peak, "unit": "T FP64-pipe instr/s",
                "frac": (ach_main / peak) if ach_main else None,
                "work_basis": "algorithmic" if ach_algo else "executed (ncu)",
                "algorithmic_fp64_per_unit": algo,
                "algorithmic_def": "lower bound of every child: d lower-end additions + the outer function (Eq. 3)",
                "achieved_executed": ach, "frac_executed": (ach / peak) if ach else None,
                "traffic": ops.get("dram_bytes_per_launch"),
                "fp64_inst_per_unit": per_unit, "unit_of_work": ops.get("unit"), "units_per_launch": units,
                "issue_active_pct_ncu": ops.get("issue_active_pct"), "fp64_pipe_pct_ncu": ops.get("fp64_pipe_pct"),
                "peak_source": src, "counts_source": "ncu sm__sass_thread_inst_executed_op_{dadd,dmul,dfma} "
                                                     "over one solve, profiles/fp64_ops_r02.json"}
    roof["share_of_step"] = pd["ms"] / max(1e-9, prof_ms)
    roof["avg_launch_us"] = avg_s * 1e6
    return roof


def env_rank():
    r = int(os.environ.get("RANK", "0"))
    w = int(os.environ.get("WORLD_SIZE", "1"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    return r, w, lr


def load_json(p):
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 9:
                rows.append(p)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ helpers
def slab(l, u, rank, world):
    """Partition of the domain along x_1 into `world` slabs (exact cover)."""
    l = l.copy()
    u = u.copy()
    a, b = l[0], u[0]
    edges = [a + (b - a) * k / world for k in range(world + 1)]
    edges[0], edges[-1] = a, b
    l[0], u[0] = edges[rank], edges[rank + 1]
    return l, u


def exchange_fn(dist):
    def ex(x):
        dist.all_reduce(x, op=dist.ReduceOp.MIN)

    return ex


def transfer_fn(dist, rank):
    """ib_transfer_fn contract: move nbytes of rank src's buffer to rank dst
    (point-to-point; every rank is called, only the two involved act)."""

    def tr(src, dst, tbuf, nbytes):
        if rank == src:
            dist.send(tbuf[:nbytes], dst)
        elif rank == dst:
            dist.recv(tbuf[:nbytes], src)

    return tr


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_branch_rate(cfg, seconds, cores):
    """The CPU oracle, as it stands, on a bounded sample of the workload:
    or_branch (one partition of a region into m^d children, each bounded over
    all n variables, §3.1) on the workload's root region and its
    level-1 children, one thread per host core (ctypes releases the GIL; the
    oracle's rounding mode is per thread).  Returns (child boxes / s, sample)."""
    import threading

    import oracle

    fid, n = cfg["fid"], cfg["n"]
    l, u = workloads.config_bounds(cfg)
    d = min(n, 10 if n <= 1000 else 8)  # a bounded CPU sample: m^d children of O(n) each
    kids = 2 ** d
    parents = [(l, u, 0)]
    for c in range(0, kids, max(1, kids // 64)):
        lo, hi = oracle.child_box(l, u, 0, d, 2, c)
        parents.append((lo, hi, d % n))
    counts = [0] * cores
    stop = time.perf_counter() + seconds

    def work(tid):
        k = tid
        while time.perf_counter() < stop:
            plo, phi, cyc = parents[k % len(parents)]
            oracle.branch(fid, plo[None], phi[None], [cyc], d, 2, l, u, mono=True)
            counts[tid] += kids
            k += cores

    oracle.lib()
    t0 = time.perf_counter()
    th = [threading.Thread(target=work, args=(i,)) for i in range(cores)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    dt = time.perf_counter() - t0
    ev = sum(counts)
    return ev / dt, dt, (f"or_branch (d = {d}, m = 2, O(n) per child) on the root region and {len(parents) - 1} level-1 "
                     f"regions of {cfg['name']}, {ev} child boxes in {dt:.1f} s on {cores} threads")


def cpu_baseline(cfg, seconds=12.0):
    cores = host_cores()
    v, _, sample = oracle_branch_rate(cfg, seconds, cores)
    return {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}


def reference_arm(args, cfg):
    """--impl reference: the oracle (this tier's reference) timed on
    the host cores, each step a bounded sample of the workload (~1 s)."""
    r, world, _ = env_rank()
    if r != 0:
        return 0
    cores = host_cores()
    ev_s, dts, sample = [], [], ""
    for _ in range(max(1, args.warmup)):
        oracle_branch_rate(cfg, 0.5, cores)
    for _ in range(args.steps):
        v, dt, sample = oracle_branch_rate(cfg, 1.0, cores)
        ev_s.append(v)
        dts.append(dt)
    v = statistics.mean(ev_s)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(dts),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfg["name"], "fid": cfg["fid"], "n": cfg["n"], "domain": [cfg["lo"], cfg["hi"]],
                   "eps": cfg["eps"], "step": "the CPU oracle's or_branch on regions of the workload, >= 1 s per step"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, help="BASELINE.json configs index [4: rastrigin n=10000]")
    ap.add_argument("--bmax", type=int, default=0)
    ap.add_argument("--m", type=int, default=2)
    ap.add_argument("--d", type=int, default=0, help="variables split per iteration [18 at n >= 10,000, else min(n, 16)]")
    ap.add_argument("--no-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the configs[1] throughput-regime measurement")
    ap.add_argument("--no-all-functions", action="store_true",
                    help="skip the time to enclose of all ten paper functions at n = 10,000")
    ap.add_argument("--mode", default="partition", choices=["replicas", "partition"],
                    help="N > 1: independent solves per GPU (replicas) or one domain partitioned into slabs along x_1 "
                         "with the incumbent all-reduced (MIN) every chunk of iterations")
    args = ap.parse_args()
    cfg = workloads.CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg)

    import torch

    import paper_2507_01770_b200 as pb

    rank, world, lrank = env_rank()
    torch.cuda.set_device(lrank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
    dev = torch.device("cuda", lrank)
    fid, n = cfg["fid"], cfg["n"]
    L, U = workloads.config_bounds(cfg)
    partition = world > 1 and args.mode == "partition"
    l, u = slab(L, U, rank, world) if partition else (L, U)
    ld = torch.tensor(l, device=dev)
    ud = torch.tensor(u, device=dev)
    # split width: 18 at the headline n = 10,000 (262,144 subregions per
    # iteration, PAPER.md:158's occupancy rule; the same time to enclose as
    # d = 16 with 3.6x the child boxes per second), else min(n, 16)
    dsplit = args.d or (18 if n >= 10_000 else min(n, 16))
    opts = pb.options(d=dsplit, m=args.m, bmax=args.bmax or None)
    popts = pb.options(d=dsplit, m=args.m, bmax=args.bmax or None, profile=1)
    ws = pb.Workspace(pb.solve_workspace_bytes(fid, n, opts), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    ex = exchange_fn(dist) if partition else None

    tr = transfer_fn(dist, rank) if partition else None

    def solve(o):
        if ex:  # partitioned domain: incumbent exchange + box rebalancing
            return pb.ib_solve_dev_mg(fid, ld, ud, ex, tr, rank, cfg["eps"], cfg["eps"], o, workspace=ws)
        return pb.ib_solve_dev(fid, ld, ud, cfg["eps"], cfg["eps"], o, workspace=ws)

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(o, steps):
        stream = torch.cuda.current_stream()
        total = 0.0
        out = []
        for _ in range(steps):
            flush.fill_(1)  # L2 flush between steps (outside the timed events)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = solve(o)
            e1.record(stream)
            torch.cuda.synchronize()
            total += e0.elapsed_time(e1)
            out.append(r)
        return total, out

    for _ in range(max(3, args.warmup)):
        solve(opts)
    stream = torch.cuda.current_stream()
    clk = ClockSampler(lrank)
    barrier()
    clk.start()
    total_ms, res = timed(opts, args.steps)
    barrier()
    clocks = clk.stop()
    # second timed region: the same solves with CUDA events around every
    # kernel class (eager launches instead of the graph replay)
    prof_ms, pres = timed(popts, max(1, min(args.steps, 3)))
    evals = sum(r.evals for r in res)
    t = torch.tensor([total_ms, float(evals)], dtype=torch.float64, device=dev)
    if dist:
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tev = t[1:].clone()
        dist.all_reduce(tev, op=dist.ReduceOp.SUM)
        total_ms, evals = float(tmax.item()), float(tev.item())
    value = evals / (total_ms / 1e3)
    r0 = res[-1]
    f_lo, f_hi = r0.f_lo, r0.f_hi
    if partition:
        enc = torch.tensor([f_lo, f_hi], dtype=torch.float64, device=dev)
        dist.all_reduce(enc, op=dist.ReduceOp.MIN)
        f_lo, f_hi = enc.tolist()

    # ---- live roofline of the dominant kernel (CUDA events inside the runtime)
    prof = {}
    for r in pres:
        for c, v in r.prof.items():
            p = prof.setdefault(c, {})
            for k, x in v.items():
                p[k] = p.get(k, 0) + x
    prof = {c: v for c, v in prof.items() if v.get("launches")}
    roof = roofline(prof, prof_ms, fid, dsplit)
    lat = latency_roofline(prof)
    roof["timing"] = "CUDA events around each kernel, second timed region (eager launches)"

    # ---- e2e through the public host-buffer API (pinned host buffers)
    e2e = None
    if world > 1:
        # N GPUs: the Python API call a user makes per rank, with this step's
        # inputs copied from pinned host memory and the enclosure read back
        # inside the timed region; max over ranks
        lh = torch.tensor(l, dtype=torch.float64).pin_memory()
        uh = torch.tensor(u, dtype=torch.float64).pin_memory()
        ms = 0.0
        ev2 = 0
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ld.copy_(lh, non_blocking=True)
            ud.copy_(uh, non_blocking=True)
            r2 = solve(opts)
            enc_h = torch.tensor([r2.f_lo, r2.f_hi], dtype=torch.float64)  # host values: already read back
            e1.record(stream)
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
            ev2 += r2.evals
        tt = torch.tensor([ms, float(ev2)], dtype=torch.float64, device=dev)
        tmx, tev = tt[:1].clone(), tt[1:].clone()
        dist.all_reduce(tmx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tev, op=dist.ReduceOp.SUM)
        e2e = {"value": float(tev.item()) / (float(tmx.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": 2 * n * 8, "d2h_bytes_per_step": int(enc_h.numel() * 8) + 48}
    if world == 1:
        lh = torch.tensor(l, dtype=torch.float64).pin_memory()
        uh = torch.tensor(u, dtype=torch.float64).pin_memory()
        cap = 4096
        so = torch.empty((cap, n), dtype=torch.float64).pin_memory()
        sh = torch.empty((cap, n), dtype=torch.float64).pin_memory()
        sl = torch.empty(cap, dtype=torch.float64).pin_memory()
        import ctypes

        ms = 0.0
        ev2 = 0
        d2h = 0
        for _ in range(args.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            rr = pb.IbResult()
            e0.record(stream)
            rc = pb.lib().ib_solve(fid, n, ctypes.cast(lh.data_ptr(), pb._dp), ctypes.cast(uh.data_ptr(), pb._dp),
                                   cfg["eps"], cfg["eps"], ctypes.byref(opts), ws.ptr(), ws.nbytes,
                                   ctypes.byref(rr), ctypes.cast(so.data_ptr(), pb._dp),
                                   ctypes.cast(sh.data_ptr(), pb._dp), ctypes.cast(sl.data_ptr(), pb._dp), cap,
                                   ctypes.c_void_p(stream.cuda_stream))
            e1.record(stream)
            torch.cuda.synchronize()
            pb._check(rc, "ib_solve")
            ms += e0.elapsed_time(e1)
            ev2 += rr.evals
            d2h = min(rr.n_surv, cap) * (2 * n + 1) * 8 + 48
        e2e = {"value": ev2 / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 2 * n * 8, "d2h_bytes_per_step": d2h}

    # ---- the throughput regime (BASELINE configs[1], Ackley n = 10: millions
    # of live regions per iteration, multi-kernel path): value + per-kernel
    # rooflines, so the batch kernels' fractions are reported next to the
    # latency-bound headline
    secondary = None
    if rank == 0 and world == 1 and args.config != 1 and not args.no_secondary:
        c1 = workloads.CONFIGS[1]
        l1, u1 = workloads.config_bounds(c1)
        ld1, ud1 = torch.tensor(l1, device=dev), torch.tensor(u1, device=dev)
        o1 = pb.options(d=min(c1["n"], 16), m=args.m)
        p1 = pb.options(d=min(c1["n"], 16), m=args.m, profile=1)
        ws1 = pb.Workspace(pb.solve_workspace_bytes(c1["fid"], c1["n"], o1), device=dev)
        for _ in range(3):
            pb.ib_solve_dev(c1["fid"], ld1, ud1, c1["eps"], c1["eps"], o1, workspace=ws1)
        ms1, ev1, pr1 = 0.0, 0, {}
        for k in range(5 + 3):
            flush.fill_(1)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r1 = pb.ib_solve_dev(c1["fid"], ld1, ud1, c1["eps"], c1["eps"], o1 if k < 5 else p1, workspace=ws1)
            e1.record(stream)
            torch.cuda.synchronize()
            if k < 5:
                ms1 += e0.elapsed_time(e1)
                ev1 += r1.evals
            else:
                for c, v in r1.prof.items():
                    q = pr1.setdefault(c, {})
                    for kk, x in v.items():
                        q[kk] = q.get(kk, 0) + x
        pr1 = {c: v for c, v in pr1.items() if v.get("launches")}
        pms = sum(v["ms"] for v in pr1.values())
        secondary = {"workload": c1["name"], "value": ev1 / (ms1 / 1e3), "unit": UNIT, "ms_per_step": ms1 / 5,
                     "kernel_roofline": {c: roofline({c: v}, pms, c1["fid"]) for c, v in pr1.items()}}
        del ws1

    # ---- north_star target: every paper function at n = 10,000 on its own
    # domain (BASELINE configs[4]), time to enclose per function (one warm-up
    # solve, one timed solve each, CUDA events)
    all_ten = None
    if rank == 0 and world == 1 and args.config == 4 and not args.no_all_functions:
        all_ten = {}
        for f10 in range(1, 11):
            l10, u10 = workloads.bounds(f10, 10_000)
            ld10, ud10 = torch.tensor(l10, device=dev), torch.tensor(u10, device=dev)
            o10 = pb.options(d=16, m=args.m)
            ws10 = pb.Workspace(pb.solve_workspace_bytes(f10, 10_000, o10), device=dev)
            pb.ib_solve_dev(f10, ld10, ud10, 1e-6, 1e-6, o10, workspace=ws10)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r10 = pb.ib_solve_dev(f10, ld10, ud10, 1e-6, 1e-6, o10, workspace=ws10)
            e1.record(stream)
            torch.cuda.synchronize()
            all_ten[workloads.NAMES[f10]] = {"s": e0.elapsed_time(e1) / 1e3, "enclosure": [r10.f_lo, r10.f_hi],
                                              "iters": r10.iters, "status": r10.status}
            del ws10

    # ---- the other BASELINE.json configs (one warm-up + one timed solve each,
    # CUDA events): Ackley n = 10, Griewank n = 100 (m = 3 on the symmetric
    # domain), Levy n = 1000
    other = None
    if rank == 0 and world == 1 and args.config == 4 and not args.no_all_functions:
        other = {}
        for ci, m_c, d_c in ((1, 2, 10), (2, 3, 10), (3, 2, 16)):
            cc = workloads.CONFIGS[ci]
            lc, uc = workloads.config_bounds(cc)
            ldc, udc = torch.tensor(lc, device=dev), torch.tensor(uc, device=dev)
            oc = pb.options(d=d_c, m=m_c)
            wsc = pb.Workspace(pb.solve_workspace_bytes(cc["fid"], cc["n"], oc), device=dev)
            pb.ib_solve_dev(cc["fid"], ldc, udc, cc["eps"], cc["eps"], oc, workspace=wsc)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rc_ = pb.ib_solve_dev(cc["fid"], ldc, udc, cc["eps"], cc["eps"], oc, workspace=wsc)
            e1.record(stream)
            torch.cuda.synchronize()
            sec = e0.elapsed_time(e1) / 1e3
            other[cc["name"]] = {"s": sec, "m": m_c, "d": d_c, "iters": rc_.iters, "evals": rc_.evals,
                                 "box_evals_per_s": rc_.evals / sec, "enclosure": [rc_.f_lo, rc_.f_hi],
                                 "regions": rc_.n_surv, "status": rc_.status}
            del wsc

    base = None
    if rank == 0 and world == 1 and not args.no_baseline:
        try:
            base = cpu_baseline(cfg)
        except Exception as e:  # the baseline must never break the bench line
            base = {"value": None, "error": repr(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if partition else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg["name"], "fid": fid, "n": n, "domain": [cfg["lo"], cfg["hi"]],
                       "eps": cfg["eps"], "d": dsplit, "m": args.m, "bmax": int(opts.bmax) or "auto",
                       "step": "one full solve (root region -> eps-enclosure)",
                       "l2": "flushed between steps (256 MiB write)",
                       "parallelism": (f"domain slabs x{world} along x_1, NCCL all-reduce(MIN) of GUB per chunk, "
                                       "box rebalancing (NCCL send/recv) when the lists skew"
                                       if partition else
                                       f"replicas x{world}: one independent solve per GPU (the n = 10k deep dive "
                                       "has one live region per iteration and does not shard; DESIGN.md)")},
            "time_to_enclose_s": total_ms / args.steps / 1e3,
            "enclosure": [f_lo, f_hi],
            "iters": r0.iters, "evals_per_step": r0.evals, "peak_pool": r0.peak_pool,
            "roofline": roof,
            "kernel_ms": {c: round(p["ms"] / len(pres), 4) for c, p in prof.items()},
            "kernel_roofline": {c: roofline({c: p}, prof_ms, fid, dsplit) for c, p in prof.items()},
            "latency_roofline": lat,
            "profiled_ms_per_step": prof_ms / len(pres),
            "cpu_baseline": base,
            "throughput_regime": secondary,
            "time_to_enclose_all_ten_n10000": all_ten,
            "baseline_configs": other,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": int(sum(r.n_kernels for r in res)),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
