#!/usr/bin/env python
"""Benchmark of the B200 IRK solve phase (BASELINE.json metric).

Workload (BASELINE configs[1], "C2"): 2D heat on a 1024x1024-cell P1 grid
(1,046,529 free dofs per stage), Radau IIA s=3 (3,139,587 unknowns),
h_t = 1e-3, u0 = sin(pi x) sin(pi y) + U[-0.01, 0.01] (seeded), GMRES(50),
rtol 1e-8, block LDU (P_LD) preconditioner with one AMG V(1,1) damped-Jacobi
cycle per diagonal block, fp64.  A "step" is one IRK timestep solve (stage
rhs -> GMRES -> u_{n+1}); timed steps advance the trajectory u_0 -> u_K.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  `value` = timestep solves/s over all ranks
with inputs resident in HBM (irkdev_step_device); `e2e` = the same metric
through the host-pointer C ABI (irkdev_step: H2D of u_n, D2H of u_{n+1} and
the report inside the timed region).  Multi-GPU runs are independent replicas
(the solve does not shard), reported as weak scaling.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "IRK timestep solves/s (2D heat, Radau IIA); solve-phase HBM GB/s vs peak"
UNIT = "solves/s"
# BASELINE.json configs.  C2 is the headline workload; the
# others are selectable with --workload for the record (profiles/).
WORKLOADS = {
    "C1": dict(problem="heat", cells=64, scheme=0, s=2, ht=1e-2, noise=0.0, seed=0, steps=1,
               desc="C1: heat 64^2 P1, Radau IIA s=2, h_t=1e-2, P_LD + AMG V(1,1) Jacobi, GMRES(50) rtol 1e-8"),
    "C2": dict(problem="heat", cells=1024, scheme=0, s=3, ht=1e-3, noise=0.01, seed=1, steps=10,
               desc="C2: heat 1024^2 P1, Radau IIA s=3, h_t=1e-3, P_LD + AMG V(1,1) Jacobi, GMRES(50) rtol 1e-8"),
    "C3": dict(problem="heat", cells=2048, scheme=1, s=5, ht=1e-3, noise=0.01, seed=1, steps=5,
               desc="C3: heat 2048^2 P1, Lobatto IIIC s=5, h_t=1e-3, P_LD + AMG V(1,1) Jacobi, GMRES(50) rtol 1e-8"),
    "C4": dict(problem="dg", cells=1024, scheme=0, s=4, ht=1e-2, noise=None, seed=0, steps=10,
               desc="C4: double glazing 1024^2 P1 SUPG (eps 0.005), Radau IIA s=4, h_t=1e-2, u0=0, "
                    "P_LD + AMG V(1,1) Jacobi, GMRES(50) rtol 1e-8"),
}
WL = WORKLOADS["C2"]
CELLS, S, HT = WL["cells"], WL["s"], WL["ht"]
WORKLOAD = WL["desc"]


def set_workload(name: str, cells: int | None = None):
    global WL, CELLS, S, HT, WORKLOAD
    WL = dict(WORKLOADS[name])
    if cells:
        WL["cells"] = cells
    CELLS, S, HT, WORKLOAD = WL["cells"], WL["s"], WL["ht"], WL["desc"]


def make_problem(P):
    """(ProblemSetup, Butcher table, u0, f_lift or None) of the workload."""
    if WL["problem"] == "heat":
        prob = P.make_heat_setup(CELLS)
        u0 = prob.initial(WL["noise"], WL["seed"])
        lift = None
    else:
        prob = P.make_double_glazing_setup(CELLS, 0.005)
        u0 = np.zeros(prob.M.n_rows)
        lift = np.ascontiguousarray(prob.f_lift)
    table = P.make_table(P.Scheme(WL["scheme"]), S)
    return prob, table, u0, lift


DATA = "synthetic (seeded u0 noise / zero u0 for C4, BASELINE configs; no dataset involved)"


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def config(extra=None):
    n = (CELLS - 1) ** 2 if WL["problem"] == "heat" else None
    c = {"workload": WORKLOAD, "grid": f"{CELLS}x{CELLS}", "dofs_per_stage": n,
         "stages": S, "unknowns": S * n if n else None, "ht": HT, "preconditioner": "LD",
         "gmres_restart": 50, "rel_tol": 1e-8,
         "l2_policy": "inputs larger than L2 (>=2.8 GB streamed per GMRES iteration vs 126 MB L2)"}
    if extra:
        c.update(extra)
    return c


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------------ byte model
def cycle_lengths(iters, restart=50):
    """Columns m_k of each GMRES(restart) cycle of a solve with `iters` iterations."""
    out = []
    while iters > 0:
        out.append(min(restart, iters))
        iters -= out[-1]
    return out or [0]


def survey_model_bytes(dev_info, levels, iters, n, s, nnz_mk, restart=50):
    """Algorithmic HBM bytes of one IRK solve per SURVEY.md §8(d)'s formula:
    CSR operators (4 B index + 8 B value per nonzero), every array read once
    and written once per kernel, no cross-kernel cache credit.

    levels[k] = [(n_l, nnz_A, nnz_P, nnz_R), ...].  ORTH(j) is the delayed-CGS2
    cost the device runs, 8 sN (2j + 6): block-dot (j + 2 vectors) + update
    (j + 4); DCGS2 folds the second Gram-Schmidt pass into the next block-dot,
    so no separate re-orthogonalisation pass is charged.
    """
    N = n
    sN = s * N
    OP = 4 * (N + 1) + 4 * nnz_mk + 16 * nnz_mk + 8 * sN + 8 * sN

    def VC(lv):
        b = 0
        for l in range(len(lv) - 1):
            nl, nA, nP, nR = lv[l]
            nc = lv[l + 1][0]
            b += 2 * (4 * (nl + 1) + 12 * nA) + 4 * (nl + 1) + 12 * nP + 4 * (nc + 1) + 12 * nR
            b += 104 * nl + 16 * nc
        nL = lv[-1][0]
        return b + 8 * nL * nL + 16 * nL

    sob = dev_info["solver_of_block"]
    PREC = sum(VC(levels[sob[i]]) for i in range(s))
    PREC += (s - 1) * (4 * (N + 1) + 12 * nnz_mk + 16 * N) + sum(8 * N * (i + 2) for i in range(1, s))
    ms = cycle_lengths(iters, restart)
    total = sum(OP + PREC + 8 * sN * (2 * j + 6) for m in ms for j in range(m))
    total += 8 * sN * (iters + 1) + PREC + OP + 16 * sN + 8 * N * (s + 2) + (4 * (N + 1) + 12 * nnz_mk)
    total += (len(ms) - 1) * (PREC + OP + 8 * sN * (restart + 1) + 24 * sN)
    return total


def format_model_bytes(mb, iters, restart=50):
    """Bytes of one solve from the device's own per-kernel tally
    (irkdev_model_bytes: each kernel's operands once, in their STORED formats
    -- row classes, u8/u16 codes, SELL/CSR indices)."""
    pre, cyc, cyc_m, it, it_j, post = mb[:6]
    ms = cycle_lengths(iters, restart)
    total = pre + post
    for m in ms:
        total += cyc + m * cyc_m + sum(it + j * it_j for j in range(m))
    return total


# ------------------------------------------------------------------ reference arm
def run_reference_steps(steps, warmup, budget_s=None):
    """The reference's own CPU implementation (oracle/_ref: irkprec compiled from
    its sources) on the same workload: setup excluded, steps timed.

    Nothing here imports the product package: M, K, f_lift come from the
    reference's own assembly and u0 from ref_problem_initial (the project's
    seeded u0 recipe restated on the reference mesh, pinned bit for bit to
    irk_problem_initial by tests/test_bench_ref.py).  With `budget_s`, the step
    count is cut so that the timed steps fit the budget (measured on the first
    warm-up step).  Returns (seconds, iterations, steps, warmup)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from refs import Ref, RefSolver  # noqa: E402
    if not Ref.available():
        raise RuntimeError("oracle/_ref/libirkref.so not built")
    noise = WL["noise"] if WL["noise"] is not None else 0.0
    ref_prob = Ref.problem(WL["problem"], CELLS, initial=(noise, WL["seed"]))
    u0 = ref_prob["u0"] if WL["noise"] is not None else np.zeros(len(ref_prob["f_lift"]))
    lift = ref_prob["f_lift"] if WL["problem"] != "heat" else None
    rs = RefSolver(ref_prob["M"], ref_prob["K"], WL["scheme"], S, 3, HT)
    u = u0.copy()
    for w in range(warmup):
        r = rs.step(u, lift)
        u = r["u_next"]
        if w == 0 and budget_s:
            steps = max(1, min(steps, int(budget_s / max(r["seconds"], 1e-9))))
    u = u0.copy()
    secs, its = [], []
    for _ in range(steps):
        r = rs.step(u, lift)
        secs.append(r["seconds"])
        its.append(r["iterations"])
        u = r["u_next"]
    return sum(secs), its, steps, warmup


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # Same warm-up and step count as our arm, cut only if the reference would
    # need more than ~4 minutes for the timed steps (C3: ~50 s per step).
    total, its, steps, warm = run_reference_steps(args.steps, max(1, args.warmup), budget_s=240.0)
    value = steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": 1e3 * total / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": config({"reference_iterations": its}),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_threads(), "cpu_model": cpu_model(),
                         "kind": "reference",
                         "sample": f"{steps} {WORKLOAD[:2]} timesteps (after {warm} warm-up) of the reference "
                                   "irk_step (irkprec compiled from /root/reference sources by oracle/Makefile, "
                                   f"OpenMP on {cpu_threads()} threads, GMRES(50) wrapper), setup excluded"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--cells", type=int, default=None, help="override the workload's grid")
    args = ap.parse_args()
    set_workload(args.workload, args.cells)
    # torchrun exports OMP_NUM_THREADS=1 per process; the reference's CPU path
    # (and the host setup) should use every host thread this process may run
    # on.  Set before the first OpenMP library (libirkdev / libirkref) loads.
    os.environ["OMP_NUM_THREADS"] = str(cpu_threads())
    if args.impl == "reference":
        return reference_arm(args)
    return our_arm(args)


def our_arm(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2010_11377_b200 as P
    from paper_2010_11377_b200 import _abi, replicas
    L = _abi.lib()

    t_setup = time.time()
    prob, table, u0, lift = make_problem(P)
    coeff = P.precond_coeff(table, P.CoeffKind.LowerFactor)
    Pc = P.BlockPreconditioner(prob.M, prob.F, coeff, HT, P.AmgParams(), table=table, device=local)
    dev = Pc._dev
    setup_s = time.time() - t_setup
    n = prob.M.n_rows
    d_lift = torch.from_numpy(lift).cuda() if lift is not None else None
    lift_ptr = C.c_void_p(d_lift.data_ptr()) if d_lift is not None else None
    cfg = P.GmresConfig(restart=50).c()

    d_u = torch.from_numpy(u0).cuda()
    d_un = torch.empty_like(d_u)
    stream_ptr = C.c_void_p()
    _abi.check(L.irkdev_stream(dev._h, C.byref(stream_ptr)))
    st = torch.cuda.ExternalStream(stream_ptr.value)

    def dstep(u_t, un_t):
        rep = _abi.irk_report()
        _abi.check(L.irkdev_step_device(dev._h, C.c_void_p(u_t.data_ptr()), lift_ptr, C.byref(cfg),
                                        C.c_void_p(un_t.data_ptr()), None, C.byref(rep)))
        return rep

    for _ in range(args.warmup):
        dstep(d_u, d_un)
    # timed: the trajectory u_0 -> u_K, inputs resident in HBM
    cur = torch.from_numpy(u0).cuda()
    nxt = torch.empty_like(cur)
    reps = []
    torch.cuda.synchronize()
    replicas.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(st)
        for _ in range(args.steps):
            reps.append(dstep(cur, nxt))
            cur, nxt = nxt, cur
        e1.record(st)
        torch.cuda.synchronize()
    ms = replicas.max_over_ranks(e0.elapsed_time(e1), device="cuda")
    replicas.barrier()
    its = [r.iterations for r in reps]
    value = replicas.whole_job_throughput(args.steps, world, ms)

    # e2e: host pointers through the public C ABI (H2D u_n, D2H u_{n+1} + report)
    hu = torch.from_numpy(u0.copy()).pin_memory()
    h_lift = None if lift is None else _abi.as_d(torch.from_numpy(lift).pin_memory().numpy())
    hun = torch.empty_like(hu).pin_memory()
    hist = np.empty(501)
    torch.cuda.synchronize()
    replicas.barrier()
    t0 = time.perf_counter()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(st)
    for _ in range(args.steps):
        rep = _abi.irk_report()
        _abi.check(L.irkdev_step(dev._h, _abi.as_d(hu.numpy()), h_lift, C.byref(cfg),
                                 _abi.as_d(hun.numpy()), None, C.byref(rep), _abi.as_d(hist)))
        hu, hun = hun, hu
    e3.record(st)
    torch.cuda.synchronize()
    e2e_ms = replicas.max_over_ranks(e2.elapsed_time(e3), device="cuda")
    wall_e2e = time.perf_counter() - t0

    # launches inside the timed region: per-phase kernel counts of the graph
    cnt = (C.c_int * 4)()
    _abi.check(L.irkdev_launch_counts(dev._h, cnt))
    launches = sum(cnt[0] + cnt[3] + cnt[1] * r.cycles + cnt[2] * r.iterations for r in reps)

    # roofline of the dominant kernel: fine-level smoother SpMV (DIA, 7 diagonals)
    info = dev.info()
    nh = info["n_hier"]
    levels = []
    for k in range(nh):
        lv = []
        for l in range(L.irkdev_num_levels(dev._h, k)):
            a, b_, c_, d_, f_ = (C.c_int() for _ in range(5))
            _abi.check(L.irkdev_level_info(dev._h, k, l, C.byref(a), C.byref(b_), C.byref(c_),
                                           C.byref(d_), C.byref(f_)))
            lv.append((a.value, b_.value, c_.value, d_.value))
        levels.append(lv)
    pk = peaks()
    hbm_peak = pk.get("hbm_gbs", 6650.0)
    # Dominant kernel (launch list, profiles/r1): the delayed-CGS2 fused
    # block-dot k_dgs_dot.  Algorithmic bytes of one launch at the average
    # inner index j = 15: v_0..v_{j-1}, v_j (unnormalised) and w = (j + 2)
    # vectors of sN doubles, each read once.
    jd = 15
    kms = C.c_double()
    _abi.check(L.irkdev_time_kernel(dev._h, 600 + jd, 50, C.byref(kms)))
    k_bytes = (jd + 2) * 8 * S * n
    k_gbs = k_bytes / (kms.value * 1e-3) / 1e9
    traffic = None
    try:  # dram__bytes_read.sum + dram__bytes_write.sum of the same launch (ncu --set full)
        traffic = json.loads((ROOT / "profiles" / "r2" / "traffic.json").read_text())["k_dgs_dot_j15"]
    except Exception:
        pass
    # fine-level smoother: bytes it must move in its own format -- row classes
    # (1 class byte + x, r, y per row; the stencil and omega/diagonal come from
    # the per-class table) or u8 codes (7 code bytes + x, r, diagonal code, y)
    sms = C.c_double()
    _abi.check(L.irkdev_time_kernel(dev._h, 1, 200, C.byref(sms)))
    vf0 = C.c_int()
    _abi.check(L.irkdev_level_value_format(dev._h, 0, 0, C.byref(vf0)))
    s_fmt = "row classes" if vf0.value == 3 else "u8 value codes"
    s_bytes = (1 + 8 + 8 + 8) * n if vf0.value == 3 else (7 + 8 + 8 + 1 + 8) * n
    # the composed V-cycle's level-0 legs (the V-cycle's two biggest kernels):
    # algorithmic bytes from the kernel's own tally (operands once, stored formats)
    legs = {}
    for which, name in ((7, "down leg r_1 = G_0 r_0"), (8, "up leg z_0 = [S_0 Q_0][r_0; z_1]")):
        lms, lb = C.c_double(), C.c_double()
        if L.irkdev_time_kernel(dev._h, which, 200, C.byref(lms)) != 0:
            break  # recursive (uncomposed) hierarchy
        _abi.check(L.irkdev_last_timed_bytes(dev._h, C.byref(lb)))
        legs[name] = {"bytes_per_launch": lb.value, "ms_per_launch": lms.value,
                      "achieved_gbs": lb.value / (lms.value * 1e-3) / 1e9,
                      "frac": lb.value / (lms.value * 1e-3) / 1e9 / hbm_peak}
    # whole-solve byte models on the actual hierarchies and iterations
    nnz_mk = prob.M.nnz
    mb = (C.c_double * 8)()
    _abi.check(L.irkdev_model_bytes(dev._h, mb))
    fmt_model = [format_model_bytes(list(mb), r.iterations) for r in reps]
    survey = [survey_model_bytes(info, levels, r.iterations, n, S, nnz_mk) for r in reps]
    secs = ms / 1e3
    fmt_gbs = sum(fmt_model) / secs / 1e9
    survey_gbs = sum(survey) / secs / 1e9
    # measured DRAM traffic of one whole step (ncu, every launch, caches not
    # flushed: tools/step_traffic.sh -> profiles/r2/traffic_<W>.json), scaled by
    # each step's iteration count
    meas = None
    try:
        tr = json.loads((ROOT / "profiles" / "r2" / f"traffic_{WORKLOAD[:2]}.json").read_text())
        mbytes = sum(tr["dram_bytes_per_iteration"] * r.iterations for r in reps)
        meas = {"dram_bytes_per_iteration": tr["dram_bytes_per_iteration"],
                "achieved_gbs": mbytes / secs / 1e9, "frac": mbytes / secs / 1e9 / hbm_peak,
                "source": f"profiles/r2/traffic_{WORKLOAD[:2]}.json (ncu dram__bytes_read.sum + "
                          f"dram__bytes_write.sum over all {tr['launches']} launches of one "
                          f"{tr['iterations']}-iteration step)"}
    except Exception:
        pass

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": config({"parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                          "gmres_iterations": its,
                          "restart_cycles": [r.cycles for r in reps],
                          "true_rel_residual": [r.true_rel_residual for r in reps],
                          "launches_per_iteration": cnt[2], "setup_seconds": setup_s,
                          "hierarchy_sizes": [[x[0] for x in lv] for lv in levels]}),
        "e2e": {"value": replicas.whole_job_throughput(args.steps, world, e2e_ms), "unit": UNIT,
                "h2d_bytes_per_step": 8 * n * (1 if lift is None else 2),
                "d2h_bytes_per_step": 8 * n + 4 * 8 + 8 * 501,
                "wall_seconds": wall_e2e},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "k_dgs_dot (DCGS2 fused block-dot, j=15: 17 x sN doubles)",
                     "achieved": k_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": k_gbs / hbm_peak,
                     "traffic": traffic, "bytes_per_launch": k_bytes, "ms_per_launch": kms.value,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in pk
                     else "fallback 6650 GB/s (B200_PROFILING.md)"},
        "smoother_roofline": {"kernel": f"fine-level Jacobi smoother k_spmv_dia (DIA, {s_fmt}); on the product path only "
                                        "for recursive hierarchies (IRK_COMPOSE=0, V(pre,post) != V(1,1))",
                              "bytes_per_launch": s_bytes, "ms_per_launch": sms.value,
                              "achieved_gbs": s_bytes / (sms.value * 1e-3) / 1e9,
                              "frac": s_bytes / (sms.value * 1e-3) / 1e9 / hbm_peak},
        "vcycle_level0_roofline": legs,
        "solve_roofline": {
            "frac": (meas or {}).get("frac", fmt_gbs / hbm_peak),
            "basis": "measured DRAM traffic" if meas else "format model",
            "measured": meas,
            "format_model": {"bytes_per_solve": sum(fmt_model) / len(fmt_model), "achieved_gbs": fmt_gbs,
                             "frac": fmt_gbs / hbm_peak,
                             "definition": "each kernel's operands read once and results written once in "
                                           "their stored formats (irkdev_model_bytes), per solve"},
            "survey_model": {"bytes_per_solve": sum(survey) / len(survey), "achieved_gbs": survey_gbs,
                             "frac": survey_gbs / hbm_peak,
                             "definition": "SURVEY.md §8(d) formula (CSR operators, DCGS2 ORTH 8sN(2j+6))"},
            "peak_gbs": hbm_peak},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            total, rits, nref, _ = run_reference_steps(1 if CELLS > 1024 else 2, 0)
            line["cpu_baseline"] = {
                "value": nref / total, "unit": UNIT, "cores": cpu_threads(), "cpu_model": cpu_model(),
                "kind": "reference",
                "sample": f"{nref} {WORKLOAD[:2]} timesteps of the reference irk_step (irkprec compiled from its "
                          "own sources, OpenMP on all host threads, GMRES(50) wrapper), setup "
                          f"excluded; reference iterations {rits}"}
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": cpu_threads(),
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
