"""C1 time to solution (timer off, CUDA events around sc_collision_step): persistent loop vs
the kernel-per-step path with CUDA-graph replay (SC_NO_PERSIST=1).  Not product code."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

for name, n in (("C1", None), ("C5", 512), ("C2", 1000)):
    p = make_problem(name, n=n, fixed_iters=0)
    for env in ("0", "1"):
        os.environ["SC_NO_PERSIST"] = env
        ctx = Context(0)
        t = lambda a: torch.as_tensor(a, device="cuda:0")
        args = (p.kind, t(p.pos), t(p.force))
        kw = dict(radius=t(p.radius), gap_abs=p.gap_abs, gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol,
                  max_iter=p.max_iter)
        ctx.collision_step(*args, **kw)
        s = ctx.torch_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        reps = 20
        e0.record(s)
        for _ in range(reps):
            r = ctx.collision_step(*args, **kw)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"{name} n={p.n} {'persistent' if env == '0' else 'per-kernel+graphs'}: {ms:.3f} ms/solve, "
              f"{r['iters']} iterations, {r['iters'] / ms * 1e3:.0f} iterations/s")
        ctx.close()
