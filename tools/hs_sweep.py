"""Source-split sweep of the symmetric RPY kernel at small N: one public mobility apply (incl. its
pack / combine kernels), CUDA events, 20 reps.  SC_SYM_HS=1|2|4|8 forces the split (0: cost model).
  SC_SYM_HS=4 python tools/hs_sweep.py C5 16384"""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_1909_06623_b200 import Context
from paper_1909_06623_b200.synthetic import make_problem
cfg, n = sys.argv[1], int(sys.argv[2])
p = make_problem(cfg, n=n)
t = lambda a: torch.as_tensor(a, device="cuda:0")
ctx = Context(0)
ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
F = t(p.force)
U = ctx.mobility_apply(F, mu=p.mu)
s = ctx.torch_stream(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
reps = 20
torch.cuda.synchronize(); e0.record(s)
for _ in range(reps): U = ctx.mobility_apply(F, mu=p.mu, out=U)
e1.record(s); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
fl = (39 if cfg == "C2" else 37) * p.n * (p.n - 1)
print(json.dumps({"cfg": cfg, "n": p.n, "hs": os.environ.get("SC_SYM_HS", "auto"), "us": 1e3 * ms, "pct": 100 * fl / (ms * 1e-3) / 37.22e12}))
