import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_1909_06623_b200 import Context
from paper_1909_06623_b200.synthetic import make_problem
p = make_problem("C2", fixed_iters=0, walls="floor")
t = lambda a: torch.as_tensor(a, device="cuda:0")
ctx = Context(0); ctx.set_walls(p.walls)
pos = t(p.pos)
z0 = p.pos[:, 2] - p.radius
print("initial min z-a", z0.min(), "count<0.1a", (z0 < 0.1 * p.radius).sum())
for k in range(4):
    r = ctx.time_step("spheres", pos, t(p.force), radius=t(p.radius), gap_abs=p.gap_abs, gap_rel=p.gap_rel,
                      mu=p.mu, dt=p.dt, tol=p.tol, max_iter=p.max_iter)
    c = ctx.get_contacts()
    wall = (c["j"] >= p.n).cpu().numpy()
    pos = r["pos"]
    z = pos[:, 2].cpu().numpy() - p.radius
    i = int(np.argmin(z))
    print(k, "min z-a", z.min(), "at", i, "wall constraints", wall.sum(), "status", r["status"], r["iters"],
          "body i had wall contact:", bool(((c["i"].cpu().numpy() == i) & wall).any()))
