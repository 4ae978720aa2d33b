"""Full-vector oracle certificates of converged full-size GPU solves (SURVEY.md section 8(c)
"Large LCPs"; Eq. abserrcqp): the GPU solves C3 / C5 to tol 1e-8, then ONE oracle
MVOP on gamma_GPU over every constraint gives g_oracle = D^T M (F_ext + D gamma) + gap/dt (plain
C, long-double RPY sums).  Reports gamma >= 0, phi(gamma_GPU, g_oracle) over all constraints,
max |g_GPU - g_oracle|, and the GPU residual trace phi_j (written beside the JSON).

  python tools/certify_full.py C3 C5 [--out profiles/r02]
"""
import argparse
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


def certify(name, out_dir):
    p = make_problem(name, fixed_iters=0)
    dev = torch.device("cuda:0")
    t = lambda a: torch.as_tensor(a, device=dev)
    ctx = Context(0)
    ctx.set_residual_trace(p.max_iter + 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nc = ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
    ctx.assemble_D()
    U = ctx.mobility_apply(t(p.force), mu=p.mu)
    ctx.lcp_q(p.dt, U)
    r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    trace = ctx.residual_trace()
    gam = r["gamma"].cpu().numpy()
    g = r["g"].cpu().numpy()
    ctx.close()
    t1 = time.perf_counter()
    sysm = oracle.system_for(p)
    assert sysm.ct.nc == nc
    F = oracle.apply_D(p.n, sysm.ct, gam) + p.force
    Uo = sysm.mobility(F)
    go = sysm.lcp_q(p.dt, Uo)  # gap/dt + D^T M (F_ext + D gamma)
    osec = time.perf_counter() - t1
    mm = np.minimum(gam, go)
    act = gam > 0
    out = {"config": f"{name} converged", "n": p.n, "n_c": int(nc), "iters": r["iters"], "mvops": r["mvops"],
           "status": r["status"], "phi_gpu": r["residual"], "bb_breakdowns": r["bb_breakdowns"],
           "active": int(act.sum()), "time_to_solution_s": secs, "gamma_min": float(gam.min()),
           "phi_gpu_gamma_oracle_g": float(np.linalg.norm(mm)),
           "max_abs_g_gpu_minus_oracle": float(np.abs(g - go).max()),
           "rms_g_gpu_minus_oracle_active": float(np.sqrt(np.mean((g - go)[act] ** 2))) if act.any() else 0.0,
           "max_abs_g_oracle_on_active": float(np.abs(go[act]).max()) if act.any() else 0.0,
           "phi_trace_min": float(trace.min()) if trace.size else None,
           "phi_trace_last10": [float(x) for x in trace[-10:]],
           "oracle_seconds": osec, "oracle_threads": os.cpu_count()}
    np.savetxt(os.path.join(out_dir, f"phi_trace_{name}.txt"), trace,
               header=f"{name}: phi_j = ||min(gamma_j, g_j)||_2 of the GPU BBPGD iterates (j = 0..{trace.size - 1})")
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C3", "C5"])
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02"))
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    for c in a.configs:
        res = certify(c, a.out)
        print(json.dumps(res), flush=True)
        with open(os.path.join(a.out, f"certificate_{c}.json"), "w") as f:
            json.dump(res, f, indent=1)
