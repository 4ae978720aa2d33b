"""Compressed vs direct M2L of the fast summation (sc_set_fmm_compression), C5 recipe: time per apply
(CUDA events, after a warm-up apply that also builds the bases), relative L2 error against the
ORACLE's direct rows on 48 sampled bodies, and the two operators' relative difference.
  python tools/fmm_compress_check.py [log2n ...]    (FMM_RECIPE=C2: polydisperse)"""
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


def timed(ctx, F, mu, reps=3):
    s = ctx.torch_stream()
    t0 = time.perf_counter()
    U = ctx.mobility_apply(F, mu=mu)
    torch.cuda.synchronize()
    first = time.perf_counter() - t0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        U = ctx.mobility_apply(F, mu=mu, out=U)
    e1.record(s)
    torch.cuda.synchronize()
    return U, e0.elapsed_time(e1) / reps, first


for k in [int(x) for x in sys.argv[1:]] or [16, 18, 20]:
    n = 1 << k
    p = make_problem(os.environ.get("FMM_RECIPE", "C5"), n=n)
    t = lambda a: torch.as_tensor(a, device="cuda:0")
    ctx = Context(0)
    ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
    F = t(p.force)
    rows = np.sort(np.random.default_rng(k).choice(n, 48, replace=False))
    Uo = np.stack([oracle.rpy_apply_rows(p.pos, p.radius, p.mu, p.force, int(r), int(r) + 1)[0] for r in rows])
    ctx.set_mobility_model("rpy_fmm")
    row = {"n": n, "recipe": os.environ.get("FMM_RECIPE", "C5")}
    for order in (4, 6, 8):
        ctx.set_fmm_params(order, 0)
        res = {}
        for comp in (0, 1):
            ctx.set_fmm_compression(comp)
            U, ms, first = timed(ctx, F, p.mu)
            u = U.cpu().numpy()
            res[comp] = u
            row[f"n{order}_{'svd' if comp else 'direct'}"] = {
                "ms": ms, "first_call_s": first, "leaf_level": ctx.fmm_info()["leaf_level"],
                "vs_oracle_sample_relL2": float(np.linalg.norm(u[rows, :3] - Uo[:, :3]) / np.linalg.norm(Uo[:, :3]))}
        row[f"n{order}_svd_vs_direct_relL2"] = float(np.linalg.norm(res[1][:, :3] - res[0][:, :3]) /
                                                     np.linalg.norm(res[0][:, :3]))
        ctx.set_fmm_compression(0)
    ctx.close()
    print(json.dumps(row), flush=True)
