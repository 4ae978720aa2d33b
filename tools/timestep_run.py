"""Time-stepping runs (NEXT rows f1 + f2 + f4(ii)) on the GPU: per step the four steps of
P:L480-L489 (U_nc, contacts + D, BBPGD, Euler update).  Records per-step BBPGD iterations,
constraint counts and wall time, with and without the warm start across steps.
Not product code; output: one JSON line per run."""
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


def run(name, steps, warm, walls=None, model="rpy"):
    p = make_problem(name, fixed_iters=0, walls=walls)
    dev = torch.device("cuda:0")
    t = lambda a: None if a is None else torch.as_tensor(a, device=dev)
    ctx = Context(0)
    ctx.set_walls(p.walls)
    if p.kind == "spheres":
        ctx.set_mobility_model(model)
    pos, dire = t(p.pos), t(p.direction)
    rad, length, F = t(p.radius), t(p.length), t(p.force)
    quat = t(np.tile([1.0, 0, 0, 0], (p.n, 1)))
    iters, ncs, walls_c = [], [], []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        r = ctx.time_step(p.kind, pos, F, radius=rad, direction=dire, length=length, b=p.rod_radius,
                          gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol, max_iter=p.max_iter,
                          quat=quat, want_U=False, warm_start=warm)
        assert r["status"] == 0, r
        pos = r["pos"]
        if p.kind == "rods":
            dire = r["dir"]
        iters.append(r["iters"])
        ncs.append(r["nc"])
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    c = ctx.get_contacts()
    nwall = int((c["j"] >= p.n).sum()) if p.walls is not None else 0
    ctx.close()
    return {"config": name, "n": p.n, "walls": walls, "mobility": model, "warm_start": warm, "steps": steps,
            "seconds": secs, "steps_per_s": steps / secs, "iters_per_step": iters, "n_c_per_step": ncs,
            "wall_constraints_last_step": nwall, "mean_iters": float(np.mean(iters))}


if __name__ == "__main__":
    for args in [("C2", 20, False, "floor"), ("C2", 20, True, "floor"), ("C4", 20, False, "box"),
                 ("C4", 20, True, "box"), ("C3", 3, False, None, "rpy6")]:
        print(json.dumps(run(*args)), flush=True)
