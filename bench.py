"""Benchmark of the per-time-step collision-resolution path (BASELINE.json metric).

One "step" = one pass of the whole hot path over the
C5 workload: build_contacts, assemble_D, U_ext = RPY(F_ext), q, and BBPGD for a
fixed 50 iterations (BASELINE.json configs[4]: 262,144 spheres, volume fraction
0.3).  All inside one C-ABI call (sc_collision_step) with inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
      (N > 1: each rank evaluates its share of the symmetric RPY kernel's super-block pairs into
       fixed-point row accumulators, all-reduced exactly as int64 over NCCL; constraints are owned
       by the rank of their first body)

Prints ONE JSON line on rank 0.  value = whole-job RPY pair-interactions per
second (every executed RPY apply counts N(N-1) pairs), device-timed with CUDA
events on the library's stream, max over ranks.  The reference arm
(--impl reference) times the CPU oracle (test infrastructure, oracle/) on the
host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RPY pair-interactions/s and BBPGD iters/s at N spheres, 1/2/4/8 B200, % FP64 peak"
UNIT = "pair-interactions/s"
# FP64 peak derived from unit counts and clocks: 148 SMs x 64 FP64 FMA lanes x 2 flop x 1.965 GHz
# (DESIGN.md "Roofline"); the DFMA microbenchmark measured 34.24 TFLOP/s (profiles/r01/fp64_probe.log).
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
FLOPS_PER_PAIR = 37  # canonical algorithmic FP64 flops per ordered pair
WORKLOAD = "C5"
FIXED_ITERS = 50


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                s = float(f[1])
                smax = float(f[2])
                power.append(float(f[3]))
            except ValueError:
                continue
            if s > 500:  # under load
                sm.append(s)
            for k, nm in enumerate(names):
                if f[5 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(self.lines),
                "power_w_max": max(power) if power else None}


def cpu_baseline(seconds_target=15.0):
    """The oracle (as it stands) on the host cores: RPY rows of the C5 workload."""
    import numpy as np

    import oracle
    from paper_1909_06623_b200.synthetic import make_problem
    p = make_problem(WORKLOAD)
    FT = p.force
    cores = os.cpu_count() or 1
    rows = 256
    t0 = time.perf_counter()
    oracle.rpy_apply_rows(p.pos, p.radius, p.mu, FT, 0, rows)
    dt = time.perf_counter() - t0
    rows2 = int(min(p.n, max(rows, rows * seconds_target / max(dt, 1e-6))))
    t0 = time.perf_counter()
    oracle.rpy_apply_rows(p.pos, p.radius, p.mu, FT, 0, rows2)
    dt2 = time.perf_counter() - t0
    pairs = rows2 * (p.n - 1)
    return {"value": pairs / dt2, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": _cpu_model(),
            "sample": f"oracle RPY apply (long-double sums), {rows2} target rows x {p.n} sources of {WORKLOAD}, "
                      f"{dt2:.1f} s, OMP over rows, threads={os.environ.get('OMP_NUM_THREADS', cores)}"}


def _cpu_model():
    """The host CPU model (lscpu / /proc/cpuinfo), recorded beside the CPU baseline."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle on a bounded sample of the workload (rank 0 only)."""
    if rank != 0:
        return
    import numpy as np

    import oracle
    from paper_1909_06623_b200.synthetic import make_problem
    p = make_problem(WORKLOAD)
    rows = 1024
    cores = os.cpu_count() or 1
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.rpy_apply_rows(p.pos, p.radius, p.mu, p.force, 0, rows)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = rows * (p.n - 1) / (ms / 1e3)
    sample = f"oracle RPY apply of {rows} target rows x {p.n} sources of {WORKLOAD} per step"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": _config(args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(args, world):
    return {"workload": f"{WORKLOAD}: 262,144 monodisperse spheres a=1, volume fraction 0.3, RPY all-pairs, "
                        f"F_ext ~ N(0,1)^3, dt=0.005, contacts gap<0.1a, BBPGD BB1 fixed {FIXED_ITERS} iterations",
            "n_bodies": 262144, "bbpgd_iters": FIXED_ITERS, "parallelism": f"rpy-sym-pair-tiles-x{world}",
            "l2": "flushed between steps (256 MiB write on the library stream)",
            "step": "build_contacts+assemble_D+U_ext+q+bbpgd_solve (one sc_collision_step call)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    rank, world, local = _env_int("RANK", 0), _env_int("WORLD_SIZE", 1), _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1909_06623_b200 import Context, nccl_unique_id
    from paper_1909_06623_b200.synthetic import make_problem

    torch.cuda.set_device(local)
    if world > 1:
        # NCCL's communicator-init lines (nranks, ring/NVLS setup) go to stderr for the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = Context(local, nccl_id=obj[0], rank=rank, world=world)
    else:
        ctx = Context(local)
    dev = torch.device(f"cuda:{local}")
    p = make_problem(WORKLOAD)
    pos = torch.as_tensor(p.pos, device=dev)
    rad = torch.as_tensor(p.radius, device=dev)
    F = torch.as_tensor(p.force, device=dev)
    Fc = torch.empty((p.n, 6), dtype=torch.float64, device=dev)
    Uc = torch.empty((p.n, 6), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = ctx.torch_stream()

    def step(pos_, rad_, F_, Fc_, Uc_):
        return ctx.collision_step("spheres", pos_, F_, radius=rad_, gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu,
                                  dt=p.dt, tol=p.tol, max_iter=FIXED_ITERS, fixed_iters=True, Fc_out=Fc_, Uc_out=Uc_)

    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        r = step(pos, rad, F, Fc, Uc)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    ctx.set_timing(True)
    ctx.reset_timing()
    l0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    sampler.start()
    ev0.record(stream)
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        r = step(pos, rad, F, Fc, Uc)
    ev1.record(stream)
    barrier()
    clocks = sampler.stop()
    ms_total = ev0.elapsed_time(ev1)
    launches = ctx.launch_count() - l0
    tim = ctx.get_timing()
    ctx.set_timing(False)
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    n = p.n
    pairs_per_apply = n * (n - 1)
    applies_per_step = 1 + 1 + FIXED_ITERS  # U_ext, alpha_0 MVOP, one per iteration (gamma_0 = 0: Step 2 is free)
    value = applies_per_step * pairs_per_apply / (ms_step / 1e3)
    # roofline of the dominant kernel (RPY), live CUDA-event timing on the library stream
    rpy_ms, rpy_n = tim["rpy"]
    rpy_avg_ms = rpy_ms / max(rpy_n, 1)
    flops_launch = FLOPS_PER_PAIR * rank_ordered_pairs(n, world, rank)
    achieved = flops_launch / (rpy_avg_ms / 1e3) / 1e12
    kern = "rpy_sym_kernel" if n >= 4096 else "rpy_partial_kernel"
    prof = ncu_profile_summary(kern)
    roofline = {"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": prof.get("traffic_bytes"),
                "kernel": kern, "avg_launch_ms": rpy_avg_ms, "launches_timed": rpy_n,
                "algorithmic_flops_per_pair": FLOPS_PER_PAIR,
                "hw_fp64_instr_per_ordered_pair": 18 if kern == "rpy_sym_kernel" else 26,
                "ncu_fp64_pipe_active_pct": prof.get("fp64_pipe_pct"), "ncu_profile": prof.get("file"),
                "traffic_note": "dram read+write of one launch (ncu --set full, profiles/r02): positions and forces "
                                "(~17 MB) re-read across super-block pairs; the fixed-point row accumulators "
                                "(19 MB of int64 limbs, RED.ADD.64) stay in L2 -- 0 B of DRAM writes (round 1's "
                                "per-(partner, row) slots wrote 3.2 GB per launch)",
                "peak_note": "FP64 derived from unit counts: 148 SM x 64 FP64 lanes x 2 flop x 1.965 GHz "
                             "(DFMA microbenchmark on this pool: 34.24 TFLOP/s); the symmetric kernel evaluates "
                             "each unordered pair once, so 37 algorithmic flops per ordered pair cost 18 FP64 "
                             "instructions"}
    share = {k: v[0] / max(ms_total, 1e-9) for k, v in tim.items()}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": _config(args, world),
           "bbpgd_iters_per_s": FIXED_ITERS / (ms_step / 1e3), "pct_fp64_peak": 100 * roofline["frac"],
           "n_c": r["nc"], "mvops": r["mvops"], "residual": r["residual"], "roofline": roofline,
           "kernel_time_share": share, "clocks": clocks, "gpu_launches": launches,
           "nccl": ctx.comm_info()}
    # e2e: the same call with HOST (pinned) buffers, copies inside the timed region
    if not args.no_e2e:
        hpos = torch.as_tensor(p.pos).pin_memory()
        hrad = torch.as_tensor(p.radius).pin_memory()
        hF = torch.as_tensor(p.force).pin_memory()
        hFc = torch.empty((n, 6), dtype=torch.float64).pin_memory()
        hUc = torch.empty((n, 6), dtype=torch.float64).pin_memory()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step(hpos, hrad, hF, hFc, hUc)
        barrier()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        te = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te.item())
        out["e2e"] = {"value": applies_per_step * pairs_per_apply / (e2e_ms / 1e3), "unit": UNIT,
                      "h2d_bytes_per_step": int(hpos.numel() * 8 + hrad.numel() * 8 + hF.numel() * 8),
                      "d2h_bytes_per_step": int(hFc.numel() * 8 + hUc.numel() * 8), "ms_per_step": e2e_ms}
    if world == 1 and not args.no_e2e:
        out["other_configs"] = other_configs()
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


HBM_GBS = 6534.5  # MEASURED_PEAKS.json hbm_gbs (copy bandwidth) on this pool; read live when present


def _hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return HBM_GBS, "measured (round-1 copy of MEASURED_PEAKS.json)"


def other_configs():
    """Time to solution (device-timed, CUDA events on the library stream around the solve, inputs
    resident) of the converged BASELINE configs: C1 (512 spheres, persistent loop), C2 (8,192
    polydisperse spheres), C3 (65,536 spheres, phi = 0.5), C4 (200,000 rods) and C5 converged
    (262,144 spheres).  Plus the HBM roofline of the D-gather (a3) and D^T (a5) kernels from a
    second solve with CUDA events around every launch (algorithmic bytes of SURVEY.md section 8(d):
    spheres 96 B/constraint + 28 B/body and 120 B/constraint, rods 144 B/constraint + 84 B/body and
    216 B/constraint).  Rods: the gather also forms the per-incidence half rates that the D^T pass
    sums, so the column work of D^T runs in the gather -- the per-kernel split
    of the section 8(d) bytes is nominal there and `iteration_frac` is the figure.  Context for the
    BBPGD-iterations/s half of the metric; not part of `value`."""
    import torch

    from paper_1909_06623_b200 import Context
    from paper_1909_06623_b200.synthetic import make_problem
    peak, peak_kind = _hbm_peak()
    res = {}
    for name, reps in (("C1", 5), ("C2", 5), ("C4", 5), ("C3", 1), ("C5", 1)):
        p = make_problem(name, fixed_iters=0)
        t = lambda a: None if a is None else torch.as_tensor(a, device="cuda:0")
        ctx = Context(0)
        if p.kind == "spheres":
            nc = ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
        else:
            nc = ctx.build_contacts_rods(t(p.pos), t(p.direction), t(p.length), p.rod_radius, p.gap_abs)
        ctx.assemble_D()
        ctx.lcp_q(p.dt, ctx.mobility_apply(t(p.force), mu=p.mu))
        solve = lambda: ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter, want_Fc=False, want_Uc=False)
        if reps > 1:  # (the seconds-long converged C3 / C5 solves are timed once, without a warm-up solve)
            solve()
        s = ctx.torch_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(reps):
            r = solve()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        d = {"n": p.n, "n_c": nc, "bbpgd_iters": r["iters"], "residual": r["residual"],
             "converged": r["converged"], "time_to_solution_ms": ms,
             "bbpgd_iters_per_s": r["iters"] / (ms / 1e3), "us_per_iter": 1e3 * ms / max(r["iters"], 1)}
        if name in ("C4", "C5"):  # HBM roofline of the a3 / a5 kernels (event-timed launch path)
            ctx.set_timing(True)
            ctx.reset_timing()
            r2 = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=min(p.max_iter, 60), fixed_iters=True,
                                 want_Fc=False, want_Uc=False)
            tim = ctx.get_timing()
            ctx.set_timing(False)
            rods = p.kind == "rods"
            gb = (144 if rods else 96) * nc + (84 if rods else 28) * p.n
            db = (216 if rods else 120) * nc
            gus = 1e3 * tim["gather"][0] / max(tim["gather"][1], 1)
            dus = 1e3 * tim["dt"][0] / max(tim["dt"][1], 1)
            d["roofline_hbm"] = {
                "peak_gbs": peak, "peak_kind": peak_kind, "l2": "not flushed (the loop's working set)",
                "gather": {"algorithmic_bytes": gb, "avg_launch_us": gus, "achieved_gbs": gb / gus / 1e3,
                           "frac": gb / gus / 1e3 / peak, "launches": tim["gather"][1]},
                "dt": {"algorithmic_bytes": db, "avg_launch_us": dus, "achieved_gbs": db / dus / 1e3,
                       "frac": db / dus / 1e3 / peak, "launches": tim["dt"][1]},
                "iteration_frac": (gb + db) / (d["us_per_iter"] * 1e3) / peak,
                "note": "iteration_frac: algorithmic bytes of gather + D^T per iteration / time to solution "
                        "per iteration (device-side graph loop, no per-launch events)" + (
                            "; rods: D^T sums the gather's per-incidence half rates, so the per-kernel "
                            "fractions split the section 8(d) bytes nominally" if rods else "")}
        res[name] = d
        ctx.close()
    # C5 with the fast O(N) RPY summation (NEXT row f4(i), order 8, approximate operator: rel. L2
    # error of the apply ~1e-6): the same 50 fixed iterations, for the BBPGD-iterations/s context
    p = make_problem("C5")
    t = lambda a: torch.as_tensor(a, device="cuda:0")
    ctx = Context(0)
    ctx.set_mobility_model("rpy_fmm")
    ctx.set_fmm_params(8, 0)
    kw = dict(radius=t(p.radius), gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol,
              max_iter=FIXED_ITERS, fixed_iters=True)
    ctx.collision_step("spheres", t(p.pos), t(p.force), **kw)
    s = ctx.torch_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    r = ctx.collision_step("spheres", t(p.pos), t(p.force), **kw)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    res["C5_fast_summation_order8"] = {"n": p.n, "n_c": r["nc"], "bbpgd_iters": r["iters"], "step_ms": ms,
                                       "bbpgd_iters_per_s": r["iters"] / (ms / 1e3), "fmm": ctx.fmm_info(),
                                       "note": "approximate RPY operator (DESIGN.md section 11; order 8 with the compressed M2L); "
                                               "not part of value"}
    ctx.close()
    return res


def ncu_profile_summary(kernel):
    """dram bytes per launch and FP64-pipe utilisation of `kernel` from the committed ncu
    summaries (profiles/*/*_ncu.txt, written by tools/summarize_ncu.py from --set full captures)."""
    import glob
    best = {}
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "*_ncu.txt"))):
        cur = None
        vals = {}
        for line in open(f):
            if line.startswith("== "):
                cur = line
                continue
            if cur is None or kernel not in cur:
                continue
            parts = line.split()
            if len(parts) >= 2:
                vals[parts[0]] = (parts[1], parts[2] if len(parts) > 2 else "")
        if vals:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tb = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                if k in vals:
                    tb += float(vals[k][0]) * scale.get(vals[k][1], 1)
            best = {"file": os.path.relpath(f, ROOT), "traffic_bytes": tb or None}
            if "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active" in vals:
                best["fp64_pipe_pct"] = float(vals["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"][0])
    return best


def rank_ordered_pairs(n, world, rank):
    """Ordered RPY pairs this rank's kernel launches evaluate per apply: the symmetric kernel's
    super-block pairs of this rank (a diagonal super-block pair holds 512 x 511 ordered pairs, an
    off-diagonal one 2 x 512^2), or the target-row kernel's rows x (N - 1) below N = 4096."""
    from paper_1909_06623_b200 import plan_partition, sym_pair_table
    if n < 4096:
        pp = plan_partition(n, world, rank)
        return (pp["row_hi"] - pp["row_lo"]) * (n - 1)
    nsb = -(-n // 512)
    t = sym_pair_table(nsb, world, rank)
    diag = int((t[:, 0] == t[:, 1]).sum())
    return diag * 512 * 511 + (len(t) - diag) * 2 * 512 * 512


if __name__ == "__main__":
    main()
