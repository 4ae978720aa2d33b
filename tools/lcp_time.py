"""Per-iteration time of the LCP kernels (D-gather a3, D^T a5) on C4 (rods, drag mobility) and C5
(spheres): converged / fixed-iteration solves with (1) no per-launch events (time to solution,
CUDA events on the library stream around the solve) and (2) per-launch events (kernel family
totals).  Reports the HBM roofline fraction of each kernel from the algorithmic bytes of
SURVEY.md section 8(d).
  python tools/lcp_time.py [C4 C5 ...]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6534.5


def algo_bytes(kind, nc, n):
    """(gather, D^T) algorithmic bytes per iteration."""
    if kind == "rods":
        return 144 * nc + 84 * n, 216 * nc
    return 96 * nc + 28 * n, 120 * nc


def run(name, iters=None):
    p = make_problem(name, fixed_iters=iters or 0)
    t = lambda a: None if a is None else torch.as_tensor(a, device="cuda:0")
    ctx = Context(0)
    args = (p.kind, t(p.pos), t(p.force))
    kw = dict(radius=t(p.radius), direction=t(p.direction), length=t(p.length), b=p.rod_radius, gap_abs=p.gap_abs,
              gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol, max_iter=iters or p.max_iter,
              fixed_iters=bool(iters))
    r = ctx.collision_step(*args, **kw)
    s = ctx.torch_stream()
    # (1) time to solution, no per-launch events: the solve only (contacts etc. once before)
    ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel) if p.kind == "spheres" else \
        ctx.build_contacts_rods(t(p.pos), t(p.direction), t(p.length), p.rod_radius, p.gap_abs)
    ctx.assemble_D()
    U = ctx.mobility_apply(t(p.force), mu=p.mu)
    ctx.lcp_q(p.dt, U)
    ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=kw["max_iter"], fixed_iters=bool(iters))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=kw["max_iter"], fixed_iters=bool(iters))
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    # (2) per-launch events
    ctx.set_timing(True)
    ctx.reset_timing()
    ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=kw["max_iter"], fixed_iters=bool(iters))
    tim = ctx.get_timing()
    ctx.set_timing(False)
    it = r["iters"]
    gb, db = algo_bytes(p.kind, r["nc"] if "nc" in r else ctx.nc, p.n)
    g_us = 1e3 * tim["gather"][0] / max(tim["gather"][1], 1)
    d_us = 1e3 * tim["dt"][0] / max(tim["dt"][1], 1)
    out = {"config": name, "n": p.n, "n_c": ctx.nc, "iters": it, "converged": r["converged"],
           "residual": r["residual"], "solve_ms": ms, "us_per_iter": 1e3 * ms / max(it, 1),
           "gather_us_event": g_us, "dt_us_event": d_us,
           "gather_hbm_frac": gb / (g_us * 1e-6) / 1e9 / HBM, "dt_hbm_frac": db / (d_us * 1e-6) / 1e9 / HBM,
           "iter_hbm_frac": (gb + db) / (1e-3 * ms / max(it, 1)) / 1e9 / HBM,
           "timing_families": {k: v for k, v in tim.items() if v[1]}, "env": {k: v for k, v in os.environ.items()
                                                                               if k.startswith("SC_")}}
    ctx.close()
    return out


if __name__ == "__main__":
    for name in (sys.argv[1:] or ["C4", "C5"]):
        iters = 50 if name == "C5" else None
        print(json.dumps(run(name, iters)), flush=True)
