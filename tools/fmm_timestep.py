"""Time stepping with the fast summation (C5 recipe): every step rebuilds the tree; the compressed
M2L's bases are reused while the laddered root side is unchanged.  Reports per-step time, solver
iterations, and device memory drift.  python tools/fmm_timestep.py [log2n] [steps] [order]"""
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

k = int(sys.argv[1]) if len(sys.argv) > 1 else 17
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
order = int(sys.argv[3]) if len(sys.argv) > 3 else 8
p = make_problem("C5", n=1 << k, fixed_iters=0)
t = lambda a: torch.as_tensor(a, device="cuda:0")
ctx = Context(0)
ctx.set_mobility_model("rpy_fmm")
ctx.set_fmm_params(order, 0)
pos, rad, F = t(p.pos), t(p.radius), t(p.force)
quat = t(np.tile([1.0, 0, 0, 0], (p.n, 1)))
rows = []
free0 = None
for s in range(steps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = ctx.time_step("spheres", pos, F, radius=rad, gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt,
                      tol=p.tol, max_iter=p.max_iter, quat=quat, want_U=False, warm_start=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    assert r["status"] == 0 and r["converged"] == 1, (s, r["status"])
    pos = r["pos"]
    if s == 2:
        free0 = torch.cuda.mem_get_info()[0]
    rows.append((dt, r["iters"], ctx.fmm_info()["leaf_level"]))
free1 = torch.cuda.mem_get_info()[0]
print(json.dumps({"n": p.n, "order": order, "steps": steps, "first_step_s": rows[0][0],
                  "mean_step_s_after_3": float(np.mean([x[0] for x in rows[3:]])) if steps > 3 else None,
                  "iters": [x[1] for x in rows], "leaf_levels": sorted(set(x[2] for x in rows)),
                  "finite": bool(torch.isfinite(pos).all()), "device_free_bytes_drift": int(free0 - free1)}))
