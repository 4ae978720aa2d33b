import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1909_06623_b200 import Context
from paper_1909_06623_b200.synthetic import make_problem
order = int(sys.argv[1]); n = 1 << int(sys.argv[2])
p = make_problem("C5", n=n); t = lambda a: torch.as_tensor(a, device="cuda:0")
ctx = Context(0); ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
ctx.set_mobility_model("rpy_fmm"); ctx.set_fmm_params(order, 0); ctx.set_fmm_compression(1)
F = t(p.force)
for _ in range(3): U = ctx.mobility_apply(F)
torch.cuda.synchronize()
