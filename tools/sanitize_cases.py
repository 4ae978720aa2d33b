"""Small solves that exercise the race-prone constructs, for compute-sanitizer (one tool per run):
  C1  (512 spheres): the persistent cooperative BBPGD loop (grid barriers, redundant finalize)
  C2  (4,096 polydisperse spheres): the symmetric RPY kernel with hs = 8 source parts (per-warp
      shared reverse accumulators, TMA + mbarrier, fixed-point RED limbs) and the fused D^T +
      last-CTA finalize (threadfence + counter), CUDA-graph replay
  C4  (20,000 rods, box walls): the persistent rods loop and the launch path's fused D^T
  C5  (5,000 spheres): the symmetric kernel (hs > 1), mobility apply, emulated 2-rank world
  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cases.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

t = lambda a: None if a is None else torch.as_tensor(a, device="cuda:0")


def solve(ctx, p, max_iter=None, fixed=False):
    ctx.set_walls(p.walls)
    if p.kind == "spheres":
        ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
    else:
        ctx.build_contacts_rods(t(p.pos), t(p.direction), t(p.length), p.rod_radius, p.gap_abs)
    ctx.assemble_D()
    ctx.lcp_q(p.dt, ctx.mobility_apply(t(p.force), mu=p.mu))
    return ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=max_iter or p.max_iter, fixed_iters=fixed)


cases = sys.argv[1:] or ["C1", "C2", "C4", "C5"]
for name in cases:
    ctx = Context(0)
    if name == "C1":
        p = make_problem("C1", fixed_iters=0)
        r = solve(ctx, p)
    elif name == "C2":
        p = make_problem("C2", n=4096, fixed_iters=0)
        r = solve(ctx, p, max_iter=60)
    elif name == "C4":
        p = make_problem("C4", n=20000, walls="box", fixed_iters=0)
        r = solve(ctx, p, max_iter=40)
        os.environ["SC_NO_PERSIST"] = "1"
        c2 = Context(0)
        os.environ.pop("SC_NO_PERSIST")
        r2 = solve(c2, p, max_iter=40)
        assert torch.equal(r["gamma"], r2["gamma"])
        c2.close()
    else:
        p = make_problem("C5", n=5000)
        r = solve(ctx, p, max_iter=10, fixed=True)
        ctx.set_emulated_world(2)
        r2 = solve(ctx, p, max_iter=10, fixed=True)
        assert torch.equal(r["gamma"], r2["gamma"])
    torch.cuda.synchronize()
    print(name, "n_c", ctx.nc, "iters", r["iters"], "phi", r["residual"], flush=True)
    ctx.close()
print("sanitize_cases: ok")
