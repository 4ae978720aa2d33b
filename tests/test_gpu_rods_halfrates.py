"""Rods LCP loop with per-incidence half rates (lcp.cu) against the oracle.

The rods D-gather writes h_e = (signed column of incidence e) . (U, W) of e's body, and D^T sums
the two half rates of each constraint through the incidence positions einc[l] = (e_i, e_j).  Edge
cases of that layout: a body whose incidence list runs past the gather lane's straight-line part
(24 contacts on one rod), a lone rod-wall constraint (one incidence, e_j = -1), a problem with no
contacts, and U_c after a fixed-iteration solve (recomputed from the final gamma once the loop has
set its done flag)."""
import dataclasses

import numpy as np
import pytest
import torch

import oracle
from paper_1909_06623_b200 import Context
from paper_1909_06623_b200.synthetic import make_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    c = Context(0)
    yield c
    c.close()


def _cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def _np(t):
    return t.detach().cpu().numpy()


def _relL2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def _star(seed=5):
    """One rod of length 20 along x, crossed above and below by 24 rods along y at gaps 0.02-0.08
    (< 0.1): 24 contacts on the centre rod, none among the crossing rods (>= 1.6 apart)."""
    rng = np.random.default_rng(seed)
    pos, dirs, lens = [[0.0, 0.0, 0.0]], [[1.0, 0.0, 0.0]], [20.0]
    force = [[0.0, 0.0, 0.0]]
    for k in range(12):
        for side in (1.0, -1.0):
            x = -9.0 + 1.6 * k + (0.8 if side < 0 else 0.0)
            gap = rng.uniform(0.02, 0.08)
            pos.append([x, rng.uniform(-0.3, 0.3), side * (1.0 + gap)])
            dirs.append([0.0, 1.0, 0.0])
            lens.append(rng.uniform(2.0, 4.0))
            force.append([0.0, 0.0, -500.0 * side] + 10.0 * rng.normal(size=3))  # closes the gaps in dt
    n = len(pos)
    ft = np.zeros((n, 6))
    ft[:, :3] = np.array(force)
    base = make_problem("C4", n=64, fixed_iters=0)
    return dataclasses.replace(base, n=n, pos=np.array(pos), direction=np.array(dirs), length=np.array(lens),
                               force=ft)


def _solve(ctx, p, **kw):
    ctx.build_contacts_rods(_cuda(p.pos), _cuda(p.direction), _cuda(p.length), p.rod_radius, p.gap_abs)
    ctx.assemble_D()
    ctx.lcp_q(p.dt, ctx.mobility_apply(_cuda(p.force), mu=p.mu))
    fixed = kw.pop("fixed_iters", 0)
    return ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=kw.pop("max_iter", p.max_iter), fixed_iters=bool(fixed))


def test_star_rod_many_incidences_converged(ctx):
    p = _star()
    o = oracle.solve_problem(p)
    assert o["system"].ct.nc == 24 and int(np.bincount(o["system"].ct.i, minlength=p.n)[0]) == 24
    r = _solve(ctx, p)
    assert ctx.nc == 24
    assert r["status"] == 0 and r["residual"] < 1e-8 and o["residual"] < 1e-8
    assert int((_np(r["gamma"]) > 0).sum()) >= 12  # the pushed rods are in contact
    assert _relL2(_np(r["gamma"]), o["gamma"]) <= 1e-6
    assert _relL2(_np(r["Fc"]), o["Fc"]) <= 1e-6
    assert _relL2(_np(r["Uc"]), o["Uc"]) <= 1e-6


@pytest.mark.parametrize("iters", [1, 3, 17])
def test_star_rod_fixed_iterations_lockstep(ctx, iters):
    """Fixed j_max: gamma, g and U_c (recomputed after the loop's done flag) against the oracle's
    iterate j_max, to rounding."""
    p = _star(seed=7)
    o = oracle.solve_problem(p, max_iter=iters, fixed_iters=iters)
    r = _solve(ctx, p, max_iter=iters, fixed_iters=iters)
    assert r["iters"] == o["iters"] == iters
    assert _relL2(_np(r["gamma"]), o["gamma"]) <= 1e-10
    assert _relL2(_np(r["Uc"]), o["Uc"]) <= 1e-10


def test_rods_wall_single_incidence(ctx):
    """Rods on a floor: every rod-wall constraint has one incidence (e_j = -1 in einc)."""
    p = make_problem("C4", n=3000, fixed_iters=0)
    lo = float(p.pos[:, 2].min())
    p = dataclasses.replace(p, walls=np.array([[0.0, 0.0, 1.0, lo - 0.5]]))
    f = p.force.copy()
    f[:, 2] -= 2.0  # pushed onto the floor
    p = dataclasses.replace(p, force=f)
    o = oracle.solve_problem(p)
    ctx.set_walls(p.walls)
    try:
        r = _solve(ctx, p)
    finally:
        ctx.set_walls(None)
    nwall = int((o["system"].ct.j >= p.n).sum())
    assert nwall > 0
    assert r["status"] == 0 and r["residual"] < 1e-8
    assert _relL2(_np(r["gamma"]), o["gamma"]) <= 1e-6
    assert _relL2(_np(r["Uc"]), o["Uc"]) <= 1e-6


def test_rods_no_contacts(ctx):
    p = _star()
    far = p.pos.copy()
    far[:, 0] += 100.0 * np.arange(p.n)  # every rod far from every other
    p = dataclasses.replace(p, pos=far)
    r = _solve(ctx, p)
    assert ctx.nc == 0 and r["status"] == 0 and r["iters"] == 0
