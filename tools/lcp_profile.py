"""Driver for ncu captures of the LCP kernels (D-gather, D^T): one C4 solve (rods, converged)
and one C5 solve (spheres, a few fixed iterations).  Not product code.
  ncu --set full -k regex:"gather_kernel|dt_kernel" python tools/lcp_profile.py [C4|C5|both] [iters]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
for name in (["C4", "C5"] if which == "both" else [which]):
    p = make_problem(name, fixed_iters=iters)
    t = lambda a: None if a is None else torch.as_tensor(a, device="cuda:0")
    ctx = Context(0)
    r = ctx.collision_step(p.kind, t(p.pos), t(p.force), radius=t(p.radius), direction=t(p.direction),
                           length=t(p.length), b=p.rod_radius, gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu,
                           dt=p.dt, tol=p.tol, max_iter=iters, fixed_iters=True)
    torch.cuda.synchronize()
    print(name, r["nc"], r["iters"])
    ctx.close()
