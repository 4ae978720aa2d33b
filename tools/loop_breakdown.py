"""Per-family event-timed kernel averages (gather, RPY, combine, D^T) of a 200-iteration fixed
solve, plus the graph-loop time per iteration: C2 and the C5 recipe at N = 16,384 / 32,768."""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1909_06623_b200 import Context
from paper_1909_06623_b200.synthetic import make_problem
for name, n in (("C2", None), ("C5", 16384), ("C5", 32768)):
    p = make_problem(name, n=n, fixed_iters=0)
    t = lambda a: torch.as_tensor(a, device="cuda:0")
    ctx = Context(0)
    ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
    ctx.assemble_D(); ctx.lcp_q(p.dt, ctx.mobility_apply(t(p.force), mu=p.mu))
    ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=200, fixed_iters=True)
    s = ctx.torch_stream(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record(s)
    r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=200, fixed_iters=True)
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ctx.set_timing(True); ctx.reset_timing()
    ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=200, fixed_iters=True)
    tim = ctx.get_timing()
    print(json.dumps({"cfg": name, "n": p.n, "us_per_iter_graph": 1e3 * ms / 200,
                      "families_us_per_launch": {k: round(1e3 * v[0] / max(v[1], 1), 2) for k, v in tim.items() if v[1]},
                      "launches": {k: v[1] for k, v in tim.items() if v[1]}}))
    ctx.close()
