import sys, time, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_1909_06623_b200 import Context
from paper_1909_06623_b200.synthetic import make_problem

def morton_perm(pos, h):
    k = np.floor((pos - pos.min(0)) / h).astype(np.int64)
    def spread(x):
        x = x & 0x1FFFFF
        x = (x | (x << 32)) & 0x1F00000000FFFF
        x = (x | (x << 16)) & 0x1F0000FF0000FF
        x = (x | (x << 8)) & 0x100F00F00F00F00F
        x = (x | (x << 4)) & 0x10C30C30C30C30C3
        x = (x | (x << 2)) & 0x1249249249249249
        return x
    code = spread(k[:, 0]) | (spread(k[:, 1]) << 1) | (spread(k[:, 2]) << 2)
    return np.argsort(code, kind="stable")

for name in ("C4", "C5"):
    p = make_problem(name)
    for label, perm in (("user", np.arange(p.n)), ("morton", morton_perm(p.pos, 2.0))):
        t = lambda a: None if a is None else torch.as_tensor(np.ascontiguousarray(a[perm]), device="cuda")
        ctx = Context(0)
        kw = dict(radius=t(p.radius), direction=t(p.direction), length=t(p.length), b=p.rod_radius,
                  gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol,
                  max_iter=(50 if name == "C5" else p.max_iter), fixed_iters=(name == "C5"))
        ctx.collision_step(p.kind, t(p.pos), t(p.force), **kw)
        ctx.set_timing(True); ctx.reset_timing()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = ctx.collision_step(p.kind, t(p.pos), t(p.force), **kw)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        tim = ctx.get_timing()
        print(name, label, r["iters"], round(dt * 1e3, 2), "ms", {k: (round(v[0], 3), v[1]) for k, v in tim.items() if v[1]})
        ctx.close()
