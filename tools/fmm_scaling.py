"""NEXT row f4(i): the fast RPY summation (fmm.cu) against the direct symmetric kernel, C5 recipe
(monodisperse a = 1, volume fraction 0.3, forces N(0,1)^3) at N = 2^14 .. 2^22: time per apply
(CUDA events on the library stream, mean of several applies after a warm-up), the relative L2 error
of the FMM apply against (a) the direct GPU apply (N <= 2^20) and (b) the ORACLE's direct rows on a
random sample of 48 bodies (long-double sums; independent of every GPU kernel).
--recipe C2: the polydisperse recipe (radii U[0.5, 1], volume fraction 0.4) instead.
  python tools/fmm_scaling.py [--orders 4 6 8] [--max-log2n 22] [--recipe C5|C2]"""
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


def timed_apply(ctx, F, reps, mu):
    s = ctx.torch_stream()
    U = ctx.mobility_apply(F, mu=mu)  # warm-up (builds the tree)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        U = ctx.mobility_apply(F, mu=mu, out=U)
    e1.record(s)
    torch.cuda.synchronize()
    return U, e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--orders", type=int, nargs="*", default=[4, 6, 8])
    ap.add_argument("--min-log2n", type=int, default=14)
    ap.add_argument("--max-log2n", type=int, default=22)
    ap.add_argument("--direct-max-log2n", type=int, default=21)
    ap.add_argument("--recipe", default="C5", choices=["C5", "C2"])
    a = ap.parse_args()
    for k in range(a.min_log2n, a.max_log2n + 1):
        n = 1 << k
        p = make_problem(a.recipe, n=n)
        dev = torch.device("cuda:0")
        t = lambda x: torch.as_tensor(x, device=dev)
        ctx = Context(0)
        ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
        F = t(p.force)
        row = {"n": n, "recipe": a.recipe}
        Ud = None
        if k <= a.direct_max_log2n:
            Ud, ms = timed_apply(ctx, F, 3 if k <= 20 else 1, p.mu)
            row["direct_ms"] = ms
            row["direct_pairs_per_s"] = n * (n - 1) / (ms / 1e3)
        rng = np.random.default_rng(k)
        rows = np.sort(rng.choice(n, 48, replace=False))
        Uo = np.stack([oracle.rpy_apply_rows(p.pos, p.radius, p.mu, p.force, int(r), int(r) + 1)[0] for r in rows])
        if Ud is not None:
            ud = Ud.cpu().numpy()
            row["direct_vs_oracle_sample_relL2"] = float(np.linalg.norm(ud[rows, :3] - Uo[:, :3]) /
                                                         np.linalg.norm(Uo[:, :3]))
        ctx.set_mobility_model("rpy_fmm")
        for order in a.orders:
            ctx.set_fmm_params(order, 0)
            Uf, ms = timed_apply(ctx, F, 3, p.mu)
            uf = Uf.cpu().numpy()
            info = ctx.fmm_info()
            d = {"ms": ms, "leaf_level": info["leaf_level"],
                 "vs_oracle_sample_relL2": float(np.linalg.norm(uf[rows, :3] - Uo[:, :3]) / np.linalg.norm(Uo[:, :3]))}
            if Ud is not None:
                ud = Ud.cpu().numpy()
                d["vs_direct_relL2"] = float(np.linalg.norm(uf[:, :3] - ud[:, :3]) / np.linalg.norm(ud[:, :3]))
                d["speedup_vs_direct"] = row["direct_ms"] / ms
            row[f"fmm_n{order}"] = d
        ctx.close()
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
