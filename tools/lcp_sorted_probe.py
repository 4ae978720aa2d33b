"""Does spatial body order speed up the D-gather / D^T passes?  Runs the C4 (and C5) solve with
the bodies in the generator's random order or pre-sorted by cell (same physics, relabelled).
Use under ncu (-k regex:"gather|dt_kernel").  Not product code."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

name, order, iters = sys.argv[1], sys.argv[2], int(sys.argv[3])
p = make_problem(name, fixed_iters=iters)
if order == "sorted":
    h = 5.1 if p.kind == "rods" else 2.1
    c = np.floor((p.pos - p.pos.min(0)) / h).astype(np.int64)
    m = c.max(0) + 1
    key = (c[:, 2] * m[1] + c[:, 1]) * m[0] + c[:, 0]
    perm = np.argsort(key, kind="stable")
    p.pos = np.ascontiguousarray(p.pos[perm])
    p.force = np.ascontiguousarray(p.force[perm])
    if p.radius is not None:
        p.radius = np.ascontiguousarray(p.radius[perm])
    if p.direction is not None:
        p.direction = np.ascontiguousarray(p.direction[perm])
        p.length = np.ascontiguousarray(p.length[perm])
t = lambda a: None if a is None else torch.as_tensor(a, device="cuda:0")
ctx = Context(0)
r = ctx.collision_step(p.kind, t(p.pos), t(p.force), radius=t(p.radius), direction=t(p.direction),
                       length=t(p.length), b=p.rod_radius, gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt,
                       tol=p.tol, max_iter=iters, fixed_iters=True)
torch.cuda.synchronize()
print(name, order, r["nc"], r["iters"])
