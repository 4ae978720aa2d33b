"""A moving boundary (NEXT row f2): monodisperse spheres in a box whose lid moves down
with a prescribed velocity, compressing the suspension.  The lid enters the LCP only through
q_l = Phi/dt + D^T U_ext - n.V (sc_set_wall_velocities); sc_time_step moves the plane each step.
Prints the lid height and how tightly the spheres are packed against it.

  python examples/piston.py [n_bodies] [steps]
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
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    p = make_problem("C1", n=n, fixed_iters=0, walls="box")
    walls = p.walls.copy()
    lid = int(np.argmin(walls[:, 2]))  # the face with normal -z: the lid
    V = np.zeros((len(walls), 3))
    V[lid, 2] = -20.0  # the lid moves down
    dev = torch.device("cuda:0")
    t = lambda a: torch.as_tensor(a, device=dev)
    ctx = Context(0)
    ctx.set_walls(walls)
    ctx.set_wall_velocities(V)
    pos, F = t(p.pos), t(np.zeros((n, 6)))
    t0 = time.perf_counter()
    for k in range(steps):
        r = ctx.time_step("spheres", pos, F, radius=t(p.radius), gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu,
                          dt=p.dt, tol=p.tol, max_iter=p.max_iter)
        pos = r["pos"]
        h = -ctx.get_walls()[lid, 3]  # plane -z = -h  <=>  z = h
        if k % 10 == 0 or k == steps - 1:
            top = float((pos[:, 2] + 1.0).max())
            print(f"step {k:4d}: lid at z = {h:8.3f}, highest sphere top = {top:8.3f}, n_c = {r['nc']:6d}, "
                  f"BBPGD iterations = {r['iters']:4d}, phi = {r['residual']:.2e}")
    torch.cuda.synchronize()
    print(f"{steps} steps of {n} spheres in {time.perf_counter() - t0:.2f} s")
    ctx.close()


if __name__ == "__main__":
    main()
