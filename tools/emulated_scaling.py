"""Per-rank RPY work of the multi-GPU decomposition, measured on one GPU: with an emulated world
of W ranks (sc_set_emulated_world) one C5 mobility apply launches the symmetric kernel once per
rank (each on that rank's super-block pairs, nothing waiting on anything); run under
  ncu --metrics gpu__time_duration.sum -k regex:rpy_sym_kernel --csv python tools/emulated_scaling.py
the per-launch times give each rank's compute share, hence the load balance max_r T_r / (T_1 / W).
Not product code; it does not measure communication."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

p = make_problem("C5")
t = lambda a: torch.as_tensor(a, device="cuda:0")
ctx = Context(0)
ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
F = t(p.force)
for W in (1, 2, 4, 8):
    ctx.set_emulated_world(W)
    ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
    ctx.mobility_apply(F)
    torch.cuda.synchronize()
    print("world", W, flush=True)
ctx.close()
