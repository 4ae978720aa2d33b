"""N = 2^20 spheres (the C5 recipe: volume fraction 0.3) on one B200 with the direct symmetric
RPY kernel: contacts, one mobility apply and a few fixed BBPGD iterations -- the scale the
paper reaches with KIFMM, here by brute force.  Not product code."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
p = make_problem("C5", n=n, fixed_iters=iters)
t = lambda a: torch.as_tensor(a, device="cuda:0")
ctx = Context(0)
ctx.set_timing(True)
torch.cuda.synchronize()
t0 = time.perf_counter()
r = ctx.collision_step("spheres", t(p.pos), t(p.force), radius=t(p.radius), gap_abs=p.gap_abs, gap_rel=p.gap_rel,
                       mu=p.mu, dt=p.dt, tol=p.tol, max_iter=iters, fixed_iters=True)
torch.cuda.synchronize()
secs = time.perf_counter() - t0
tim = ctx.get_timing()
rpy_ms, rpy_n = tim["rpy"]
pairs = n * (n - 1)
print(json.dumps({"n": n, "n_c": r["nc"], "iters": r["iters"], "mvops": r["mvops"], "residual": r["residual"],
                  "seconds": secs, "rpy_ms_per_apply": rpy_ms / rpy_n,
                  "rpy_pairs_per_s": pairs / (rpy_ms / rpy_n) * 1e3,
                  "rpy_frac_fp64_peak": 37 * pairs / (rpy_ms / rpy_n * 1e-3) / (148 * 64 * 2 * 1.965e9),
                  "kernel_ms": {k: round(v[0], 2) for k, v in tim.items()}}))
