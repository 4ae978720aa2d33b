"""RPY apply (the MVOP's dominant kernel) vs N: device time per apply, pair-interactions/s and
the fraction of the derived FP64 peak (37 flops per ordered pair), C5 recipe (volume fraction
0.3, monodisperse) at several N, and the C2 recipe (polydisperse).  Not product code."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1909_06623_b200 import Context  # noqa: E402
from paper_1909_06623_b200.synthetic import make_problem  # noqa: E402

PEAK = 148 * 64 * 2 * 1.965e9
cases = [("C5", int(x)) for x in os.environ.get("RPY_NS", "").split(",") if x] or (
    [("C5", n) for n in (2048, 4096, 8192, 16384, 32768, 65536, 131072, 262144, 524288, 1048576)] +
    [("C2", 8192), ("C2", 65536)])
for name, n in cases:
    p = make_problem(name, n=n)
    ctx = Context(0)
    dev = torch.device("cuda:0")
    pos, rad, F = (torch.as_tensor(a, device=dev) for a in (p.pos, p.radius, p.force))
    ctx.build_contacts_spheres(pos, rad, p.gap_abs, p.gap_rel)
    ctx.mobility_apply(F)
    reps = max(2, min(200, int(2e11 / (n * n))))
    s = ctx.torch_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        ctx.mobility_apply(F)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps  # the public call: pack, RPY kernel(s), combine, unpack
    ctx.set_timing(True)
    ctx.reset_timing()
    for _ in range(reps):
        ctx.mobility_apply(F)
    tim = ctx.get_timing()
    ctx.set_timing(False)
    k_ms = tim["rpy"][0] / reps  # the pair kernel alone (CUDA events around its launches)
    c_ms = tim["combine"][0] / reps
    pairs = n * (n - 1)
    print(json.dumps({"recipe": name, "n": n, "api_ms_per_apply": ms, "kernel_ms": k_ms, "combine_ms": c_ms,
                      "kernel_pairs_per_s": pairs / k_ms * 1e3,
                      "kernel_frac_fp64_peak": 37 * pairs / (k_ms * 1e-3) / PEAK,
                      "api_frac_fp64_peak": 37 * pairs / (ms * 1e-3) / PEAK, "reps": reps}), flush=True)
    ctx.close()
