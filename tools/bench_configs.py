"""Run every BASELINE.json config (C1-C5) through the CUDA path and report, per config:
n_c, BBPGD iterations / MVOPs, residual, time to solution, iterations/s, RPY
pair-interactions/s (spheres) or the HBM roofline of the gather / D^T kernels (rods),
kernel time shares, and parity against the CPU oracle where the oracle is affordable
(converged gamma for C1, C2, C4; sampled certificate rows for C3, C5).

  python tools/bench_configs.py [--configs C1,C2,...] [--no-oracle] > profiles/rNN/configs.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

def _hbm_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6555.8  # an earlier pod's MEASURED_PEAKS.json


HBM_GBS = _hbm_gbs()  # MEASURED_PEAKS.json hbm_gbs (driver-written per pod)
FP64_PEAK = 148 * 64 * 2 * 1.965e9
BYTES = {"spheres": {"gather_c": 96, "gather_b": 28, "dt_c": 120},
         "rods": {"gather_c": 144, "gather_b": 84, "dt_c": 216}}


def run(name, fixed, use_oracle):
    p = make_problem(name, fixed_iters=fixed)
    dev = torch.device("cuda:0")
    t = lambda a: None if a is None else torch.as_tensor(a, device=dev)
    pos, rad, dire, length, F = t(p.pos), t(p.radius), t(p.direction), t(p.length), t(p.force)
    Fc = torch.empty((p.n, 6), dtype=torch.float64, device=dev)
    Uc = torch.empty((p.n, 6), dtype=torch.float64, device=dev)
    ctx = Context(0)
    jmax = p.fixed_iters if p.fixed_iters else p.max_iter
    kw = dict(radius=rad, direction=dire, length=length, b=p.rod_radius, gap_abs=p.gap_abs, gap_rel=p.gap_rel,
              mu=p.mu, dt=p.dt, tol=p.tol, max_iter=jmax, fixed_iters=bool(p.fixed_iters), Fc_out=Fc, Uc_out=Uc)
    ctx.collision_step(p.kind, pos, F, **kw)  # warm-up (allocations, module load)
    torch.cuda.synchronize()
    stream = ctx.torch_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # time to solution without per-launch events (they add a few us to every small kernel)
    e0.record(stream)
    r = ctx.collision_step(p.kind, pos, F, **kw)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    # kernel-family shares from a second, event-instrumented run
    ctx.set_timing(True)
    ctx.reset_timing()
    e0.record(stream)
    ctx.collision_step(p.kind, pos, F, **kw)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_timed = e0.elapsed_time(e1)
    tim = ctx.get_timing()
    out = {"config": name, "kind": p.kind, "n": p.n, "n_c": r["nc"], "mode": "fixed" if p.fixed_iters else "converged",
           "iters": r["iters"], "mvops": r["mvops"], "residual": r["residual"], "converged": r["converged"],
           "time_with_per_launch_events_ms": ms_timed,
           "bb_breakdowns": r["bb_breakdowns"], "active": r["active"], "time_to_solution_ms": ms,
           "bbpgd_iters_per_s": r["iters"] / (ms / 1e3) if r["iters"] else None,
           "kernel_ms": {k: round(v[0], 3) for k, v in tim.items()},
           "kernel_launches": {k: v[1] for k, v in tim.items()}}
    nc = r["nc"]
    if p.kind == "spheres":
        applies = tim["rpy"][1]
        pairs = applies * p.n * (p.n - 1)
        out["rpy_pairs_per_s_in_kernel"] = pairs / (tim["rpy"][0] / 1e3)
        out["rpy_pairs_per_s_whole"] = pairs / (ms / 1e3)
        out["rpy_frac_fp64_peak"] = 37 * out["rpy_pairs_per_s_in_kernel"] / FP64_PEAK
    b = BYTES[p.kind]
    g_ms, g_n = tim["gather"]
    d_ms, d_n = tim["dt"]
    if g_n:
        gb = b["gather_c"] * nc + b["gather_b"] * p.n
        out["gather_GBps"] = gb / (g_ms / g_n / 1e3) / 1e9
        out["gather_frac_hbm"] = out["gather_GBps"] / HBM_GBS
    if d_n:
        db = b["dt_c"] * nc
        out["dt_GBps"] = db / (d_ms / d_n / 1e3) / 1e9
        out["dt_frac_hbm"] = out["dt_GBps"] / HBM_GBS
    if use_oracle:
        out.update(oracle_check(p, ctx, Fc, r))
    ctx.close()
    return out


def oracle_check(p, ctx, Fc, r):
    import oracle
    res = {}
    t0 = time.perf_counter()
    if p.name in ("C1", "C2", "C4") and not p.fixed_iters:
        o = oracle.solve_problem(p)
        c = ctx.get_contacts()
        Fo = o["Fc"]
        res["oracle_iters"] = o["iters"]
        res["oracle_residual"] = o["residual"]
        res["rel_L2_Fc"] = float(np.linalg.norm(Fc.cpu().numpy() - Fo) / np.linalg.norm(Fo))
        res["contacts_equal"] = bool(c["i"].shape[0] == o["system"].ct.nc)
    elif p.kind == "spheres":
        # sampled complementarity certificate: g_l = n.(U_i - U_j) + gap/dt from the oracle's
        # RPY rows applied to the GPU's F_c + F_ext; min(gamma_l, g_l) must be ~0
        ct = oracle.contacts_spheres(p.pos, p.radius, p.gap_abs, p.gap_rel)
        FT = Fc.cpu().numpy() + p.force
        rng = np.random.default_rng(0)
        ls = rng.choice(ct.nc, 16, replace=False)
        gs = []
        for l in ls:
            i, j = ct.i[l], ct.j[l]
            ui = oracle.rpy_apply_rows(p.pos, p.radius, p.mu, FT, i, i + 1)[0]
            uj = oracle.rpy_apply_rows(p.pos, p.radius, p.mu, FT, j, j + 1)[0]
            gs.append(float(np.dot(ct.normal[l], ui[:3] - uj[:3]) + ct.gap[l] / p.dt))
        res["certificate_min_g_sampled"] = float(min(gs))
        res["contacts_equal"] = bool(ctx.nc == ct.nc)
    res["oracle_seconds"] = time.perf_counter() - t0
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--c5-converged", action="store_true", help="also run C5 to convergence (long)")
    ap.add_argument("--apgd", default="", help="configs to also solve with APGD (BBPGD vs APGD MVOPs)")
    a = ap.parse_args()
    for name in a.configs.split(","):
        print(json.dumps(run(name, None, not a.no_oracle)), flush=True)
        if name == "C5" and a.c5_converged:
            print(json.dumps(run(name, 0, False)), flush=True)
    for name in [c for c in a.apgd.split(",") if c]:
        print(json.dumps(apgd_compare(name)), flush=True)


def apgd_compare(name):
    """The paper's BBPGD-vs-APGD comparison on one config: MVOPs and time."""
    p = make_problem(name, fixed_iters=0)
    dev = torch.device("cuda:0")
    t = lambda a: None if a is None else torch.as_tensor(a, device=dev)
    ctx = Context(0)
    if p.kind == "spheres":
        ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
    else:
        ctx.build_contacts_rods(t(p.pos), t(p.direction), t(p.length), p.rod_radius, p.gap_abs)
    ctx.assemble_D()
    ctx.lcp_q(p.dt, ctx.mobility_apply(t(p.force), mu=p.mu))
    out = {"config": name, "compare": "bbpgd_vs_apgd"}
    for label, fn in (("bbpgd", lambda: ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)),
                      ("apgd", lambda: ctx.apgd_solve(mu=p.mu, tol=p.tol, max_iter=20 * p.max_iter))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        out[label] = {"iters": r["iters"], "mvops": r["mvops"], "residual": r["residual"],
                      "converged": r["converged"], "seconds": time.perf_counter() - t0}
        out[label + "_gamma_norm"] = float(r["gamma"].norm())
    ctx.close()
    return out


if __name__ == "__main__":
    main()
