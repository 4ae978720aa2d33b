"""Robustness run: many time steps through the public API (f1 + f2), checking that every solve
converges, the configuration stays finite, no body passes through a wall, and device memory
stays flat (no per-step allocations).  Not product code."""
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


def run(name, steps, walls, host=False):
    p = make_problem(name, fixed_iters=0, walls=walls)
    dev = torch.device("cuda:0")
    t = (lambda a: None if a is None else torch.as_tensor(a).pin_memory()) if host else \
        (lambda a: None if a is None else torch.as_tensor(a, device=dev))
    ctx = Context(0)
    ctx.set_walls(p.walls)
    pos, dire, rad, length, F = t(p.pos), t(p.direction), t(p.radius), t(p.length), t(p.force)
    quat = t(np.tile([1.0, 0, 0, 0], (p.n, 1)))
    free0 = None
    iters, worst_floor = [], np.inf
    t0 = time.perf_counter()
    for k in range(steps):
        r = ctx.time_step(p.kind, pos, F, radius=rad, direction=dire, length=length, b=p.rod_radius,
                          gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol, max_iter=p.max_iter,
                          quat=quat, want_U=False, warm_start=True)
        assert r["status"] == 0 and r["converged"] == 1, (k, r)
        pos = r["pos"] if not host else r["pos"].cpu().pin_memory()
        if p.kind == "rods":
            dire = r["dir"] if not host else r["dir"].cpu().pin_memory()
        iters.append(r["iters"])
        if k == 2:
            torch.cuda.synchronize()
            free0 = torch.cuda.mem_get_info()[0]
        z = pos[:, 2].cpu().numpy() if p.kind == "spheres" else None
        if z is not None and walls == "floor":
            worst_floor = min(worst_floor, float((z - p.radius).min()))
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    pn = pos.cpu().numpy()
    ctx.close()
    return {"config": name, "walls": walls, "host_buffers": host, "steps": steps,
            "seconds": time.perf_counter() - t0, "mean_iters": float(np.mean(iters)), "max_iters": int(max(iters)),
            "finite": bool(np.isfinite(pn).all()), "min_floor_gap_seen": worst_floor,
            "device_free_bytes_drift": int(free0 - free1)}


if __name__ == "__main__":
    for args in [("C2", 200, "floor"), ("C2", 50, "floor", True), ("C4", 100, "box"), ("C1", 300, "box")]:
        print(json.dumps(run(*args)), flush=True)
