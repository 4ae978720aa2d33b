"""C5 (262,144 spheres) solved to convergence on the GPU, certified by the CPU oracle on a
random sample of constraints (SURVEY.md section 8(c) "large LCPs": one oracle MVOP row per
sampled body gives g_l independently; require gamma >= 0 and |min(gamma_l, g_l)| small).
A converged oracle run at this size is hours, so this is the parity evidence for it."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

nsample = int(sys.argv[1]) if len(sys.argv) > 1 else 64
p = make_problem("C5", fixed_iters=0)
dev = torch.device("cuda:0")
t = lambda a: torch.as_tensor(a, device=dev)
ctx = Context(0)
torch.cuda.synchronize()
t0 = time.perf_counter()
nc = ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
ctx.assemble_D()
U = ctx.mobility_apply(t(p.force), mu=p.mu)
ctx.lcp_q(p.dt, U)
r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
torch.cuda.synchronize()
secs = time.perf_counter() - t0
gam = r["gamma"].cpu().numpy()
g = r["g"].cpu().numpy()
Fc = r["Fc"].cpu().numpy()
# oracle certificate on sampled constraints
ct = oracle.contacts_spheres(p.pos, p.radius, p.gap_abs, p.gap_rel)
assert ct.nc == nc
rng = np.random.default_rng(0)
act = np.flatnonzero(gam > 0)
ls = np.concatenate([rng.choice(act, nsample // 2, replace=False), rng.choice(nc, nsample // 2, replace=False)])
FT = Fc + p.force
t1 = time.perf_counter()
go, mm = [], []
for l in ls:
    i, j = ct.i[l], ct.j[l]
    ui = oracle.rpy_apply_rows(p.pos, p.radius, p.mu, FT, i, i + 1)[0]
    uj = oracle.rpy_apply_rows(p.pos, p.radius, p.mu, FT, j, j + 1)[0]
    gl = float(np.dot(ct.normal[l], ui[:3] - uj[:3]) + ct.gap[l] / p.dt)
    go.append(gl)
    mm.append(min(gam[l], gl))
go = np.array(go)
mm = np.array(mm)
out = {"config": "C5 converged", "n": p.n, "n_c": int(nc), "iters": r["iters"], "mvops": r["mvops"],
       "residual": r["residual"], "converged": r["converged"], "active": r["active"],
       "time_to_solution_s": secs, "gamma_min": float(gam.min()),
       "sample": int(ls.size), "sample_active": int(nsample // 2),
       "max_abs_g_gpu_minus_oracle": float(np.abs(g[ls] - go).max()),
       "max_abs_minmap_sampled": float(np.abs(mm).max()),
       "rms_minmap_sampled_x_sqrt_nc": float(np.sqrt(np.mean(mm ** 2) * nc)),
       "oracle_seconds": time.perf_counter() - t1}
print(json.dumps(out))
ctx.close()
