"""Event-timed averages of the LCP kernel families (gather a3, D^T a5) over a fixed-iteration solve
of a config (per-launch CUDA events on the library stream; the RPY apply runs in between, as in the
bench step).  For same-box A/B of kernel variants (tools/ab/ab_libs.sh-style SC_LIB= builds).
  python tools/lcp_kernels.py C5 [iters] [reps]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
p = make_problem(name, fixed_iters=iters)
t = lambda a: None if a is None else torch.as_tensor(a, device="cuda:0")
ctx = Context(0)
if p.kind == "spheres":
    ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
else:
    ctx.build_contacts_rods(t(p.pos), t(p.direction), t(p.length), p.rod_radius, p.gap_abs)
ctx.assemble_D()
ctx.lcp_q(p.dt, ctx.mobility_apply(t(p.force), mu=p.mu))
ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=iters, fixed_iters=True)
ctx.set_timing(True)
ctx.reset_timing()
for _ in range(reps):
    ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=iters, fixed_iters=True)
tim = ctx.get_timing()
out = {"config": name, "n_c": ctx.nc, "iters": iters, "reps": reps,
       "gather_us": 1e3 * tim["gather"][0] / max(tim["gather"][1], 1), "gather_launches": tim["gather"][1],
       "dt_us": 1e3 * tim["dt"][0] / max(tim["dt"][1], 1), "dt_launches": tim["dt"][1],
       "env": {k: v for k, v in os.environ.items() if k.startswith("SC_")}}
print(json.dumps(out), flush=True)
ctx.close()
