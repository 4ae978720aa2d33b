"""One C1 solve (the persistent loop), for profilers.  Not product code."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

p = make_problem("C1", fixed_iters=0)
ctx = Context(0)
t = lambda a: torch.as_tensor(a, device="cuda:0")
for _ in range(2):
    r = ctx.collision_step(p.kind, t(p.pos), t(p.force), radius=t(p.radius), gap_abs=p.gap_abs, gap_rel=p.gap_rel,
                           mu=p.mu, dt=p.dt, tol=p.tol, max_iter=2000)
torch.cuda.synchronize()
print(r["iters"])
