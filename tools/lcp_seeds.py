"""Time to solution of the converged BBPGD over several seeds of one config (default C4): the
iteration count of a BB method depends on rounding once phi nears the FP64 noise floor, so one
seed's count is a sample, not a property of the kernels.  Per seed: iterations, solve time (CUDA
events on the library stream around bbpgd_solve, mean of 3 solves, no per-launch events), us per
iteration, and the phi trace's last decade (how flat the tail is).
  python tools/lcp_seeds.py [C4] [--seeds 1 2 3 4 5]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402


def run(name, seed):
    p = make_problem(name, seed=seed)
    t = lambda a: None if a is None else torch.as_tensor(a, device="cuda:0")
    ctx = Context(0)
    if p.kind == "spheres":
        ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
    else:
        ctx.build_contacts_rods(t(p.pos), t(p.direction), t(p.length), p.rod_radius, p.gap_abs)
    ctx.assemble_D()
    ctx.lcp_q(p.dt, ctx.mobility_apply(t(p.force), mu=p.mu))
    ctx.set_residual_trace(100000)
    r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    tr = ctx.residual_trace()
    ctx.set_residual_trace(0)
    s = ctx.torch_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    it = int(r["iters"])
    # first iteration with phi < 10 tol: how many iterations the last decade took
    below = np.flatnonzero(tr < 10 * p.tol)
    out = {"config": name, "seed": seed, "n_c": ctx.nc, "iters": it, "residual": r["residual"], "solve_ms": ms,
           "us_per_iter": 1e3 * ms / max(it, 1), "iters_last_decade": int(it - below[0]) if len(below) else None,
           "env": {k: v for k, v in os.environ.items() if k.startswith("SC_")}}
    ctx.close()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("name", nargs="?", default="C4")
    ap.add_argument("--seeds", type=int, nargs="*", default=[1, 2, 3, 4, 5])
    a = ap.parse_args()
    for sd in a.seeds:
        print(json.dumps(run(a.name, sd)), flush=True)
