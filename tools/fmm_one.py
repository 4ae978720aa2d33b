"""One fast-summation apply (C5 recipe) for ncu captures: python tools/fmm_one.py ORDER LOG2N [compress]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

order, n = int(sys.argv[1]), 1 << int(sys.argv[2])
p = make_problem("C5", n=n)
t = lambda a: torch.as_tensor(a, device="cuda:0")
ctx = Context(0)
ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
ctx.set_mobility_model("rpy_fmm")
ctx.set_fmm_params(order, 0)
if len(sys.argv) > 3:
    ctx.set_fmm_compression(int(sys.argv[3]))
F = t(p.force)
for _ in range(2):
    ctx.mobility_apply(F)
torch.cuda.synchronize()
