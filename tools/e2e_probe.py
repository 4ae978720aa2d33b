"""Diagnose the e2e (host-buffer) path of bench.py: wall time of sc_collision_step with pinned
host buffers vs device buffers, repeated.  Not product code."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
p = make_problem(name)
ctx = Context(0)
dev = torch.device("cuda:0")
kw = dict(gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol, max_iter=50, fixed_iters=True)
hpos = torch.as_tensor(p.pos).pin_memory()
hrad = torch.as_tensor(p.radius).pin_memory()
hF = torch.as_tensor(p.force).pin_memory()
hFc = torch.empty((p.n, 6), dtype=torch.float64).pin_memory()
hUc = torch.empty((p.n, 6), dtype=torch.float64).pin_memory()
dpos, drad, dF = hpos.to(dev), hrad.to(dev), hF.to(dev)
dFc = torch.empty((p.n, 6), dtype=torch.float64, device=dev)
dUc = torch.empty((p.n, 6), dtype=torch.float64, device=dev)
for rep in range(3):
    for label, args in (("device", (dpos, dF, drad, dFc, dUc)), ("host", (hpos, hF, hrad, hFc, hUc))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.collision_step("spheres", args[0], args[1], radius=args[2], Fc_out=args[3], Uc_out=args[4], **kw)
        torch.cuda.synchronize()
        print(rep, label, f"{(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)

# phase-by-phase with host buffers
def tm(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"   {label}: {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
    return r


for rep in range(2):
    print("phases rep", rep)
    tm("build_contacts(host)", lambda: ctx.build_contacts_spheres(hpos, hrad, p.gap_abs, p.gap_rel))
    tm("assemble", lambda: ctx.assemble_D())
    hU = torch.empty((p.n, 6), dtype=torch.float64).pin_memory()
    tm("mobility(host F, host U)", lambda: ctx.mobility_apply(hF, out=hU))
    tm("mobility(dev)", lambda: ctx.mobility_apply(dF))
    tm("lcp_q(host U)", lambda: ctx.lcp_q(p.dt, hU))
    tm("bbpgd(dev outs)", lambda: ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=50, fixed_iters=True))
    tm("bbpgd(host outs)", lambda: ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=50, fixed_iters=True,
                                                   out={"Fc": hFc, "Uc": hUc}))
