"""Device time of one full-6N RPY apply (NEXT row f4(ii)) at C3 and C5 sizes vs the BASELINE
(translational) apply.  Not product code."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

for name in ("C3", "C5"):
    p = make_problem(name)
    ctx = Context(0)
    dev = torch.device("cuda:0")
    pos, rad, F = (torch.as_tensor(a, device=dev) for a in (p.pos, p.radius, p.force))
    ctx.build_contacts_spheres(pos, rad, p.gap_abs, p.gap_rel)
    out = {}
    for model in ("rpy", "rpy6"):
        ctx.set_mobility_model(model)
        ctx.mobility_apply(F)
        s = ctx.torch_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(3):
            ctx.mobility_apply(F)
        e1.record(s)
        torch.cuda.synchronize()
        out[model] = e0.elapsed_time(e1) / 3
    pairs = p.n * (p.n - 1)
    print(f"{name} N={p.n}: rpy {out['rpy']:.2f} ms ({pairs / out['rpy'] * 1e3:.3e} pairs/s), "
          f"rpy6 {out['rpy6']:.2f} ms ({pairs / out['rpy6'] * 1e3:.3e} pairs/s)")
    ctx.close()
