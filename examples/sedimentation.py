"""Sedimentation onto a floor with the Python binding: the C2 recipe (polydisperse spheres,
gravity -a^3 z plus noise) above the plane z = 0, advanced by whole time steps (P:L480-L489:
U_nc, contacts incl. the wall, BBPGD, explicit Euler), warm-started from the previous step's
gamma.  Prints per-step statistics.

  python examples/sedimentation.py [n_bodies] [steps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    p = make_problem("C2", n=n, fixed_iters=0, walls="floor")
    dev = torch.device("cuda:0")
    t = lambda a: torch.as_tensor(a, device=dev)
    ctx = Context(0)
    ctx.set_walls(p.walls)
    pos, rad, F = t(p.pos), t(p.radius), t(p.force)
    quat = t(np.tile([1.0, 0.0, 0.0, 0.0], (n, 1)))
    t0 = time.perf_counter()
    for k in range(steps):
        r = ctx.time_step("spheres", pos, F, radius=rad, gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt,
                          tol=p.tol, max_iter=p.max_iter, quat=quat, warm_start=True)
        pos = r["pos"]
        if k % 10 == 0 or k == steps - 1:
            z = pos[:, 2] - rad
            print(f"step {k:4d}: n_c = {r['nc']:6d}, BBPGD iterations = {r['iters']:4d}, phi = {r['residual']:.2e}, "
                  f"mean height = {float(pos[:, 2].mean()):8.3f}, min gap to the floor = {float(z.min()):+.2e}")
    torch.cuda.synchronize()
    print(f"{steps} steps of {n} spheres in {time.perf_counter() - t0:.2f} s")
    ctx.close()


if __name__ == "__main__":
    main()
