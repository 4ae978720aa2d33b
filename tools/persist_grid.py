"""Persistent small-problem loop vs its grid size (SC_PERSIST_GRID caps the CTAs; default one per SM):
collision_step time (contacts + solve), CUDA events, 20 reps, for C1, C2 at N = 1,000, C5 at 2,000."""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1909_06623_b200 import Context
from paper_1909_06623_b200.synthetic import make_problem
for name, n in (("C1", None), ("C2", 1000), ("C5", 2000)):
    p = make_problem(name, n=n, fixed_iters=0)
    ctx = Context(0)
    t = lambda a: torch.as_tensor(a, device="cuda:0")
    args = (p.kind, t(p.pos), t(p.force))
    kw = dict(radius=t(p.radius), gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol, max_iter=p.max_iter)
    ctx.collision_step(*args, **kw)
    s = ctx.torch_stream(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); reps = 20; e0.record(s)
    for _ in range(reps): r = ctx.collision_step(*args, **kw)
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"cfg": name, "n": p.n, "grid": os.environ.get("SC_PERSIST_GRID", "148"), "ms": ms, "iters": r["iters"], "us_per_iter": 1e3 * ms / max(r["iters"], 1)}))
    ctx.close()
