"""C1: time of the setup (contacts, assemble, U_ext, q, alpha_0) vs the BBPGD loop, via
collision_step with 1 fixed iteration vs converged.  Not product code."""
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
args = (p.kind, t(p.pos), t(p.force))
for label, kw in (("1 fixed iteration", dict(max_iter=1, fixed_iters=True)), ("converged", dict(max_iter=2000))):
    k = dict(radius=t(p.radius), gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol, **kw)
    ctx.collision_step(*args, **k)
    s = ctx.torch_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(20):
        r = ctx.collision_step(*args, **k)
    e1.record(s)
    torch.cuda.synchronize()
    print(label, f"{e0.elapsed_time(e1) / 20:.3f} ms", r["iters"], "iterations", ctx.launch_count())
import time
ctx.set_timing(True); ctx.reset_timing()
r = ctx.collision_step(*args, radius=t(p.radius), gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol,
                       max_iter=2000)
print({k: (round(v[0], 3), v[1]) for k, v in ctx.get_timing().items()})
