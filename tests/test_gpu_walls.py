"""GPU parity for particle-boundary collisions (NEXT row f2) against the oracle.

Same bars as tests/test_gpu_parity.py: constraint list (pairs + walls) bit-exact, D / D^T / q
to rounding, converged gamma and D gamma rel. L2 <= 1e-6 with phi < 1e-8 on both sides.
A wall is body n + k in the constraint list, enters D on the particle only and is not in the
mobility.  Uses its own context (walls are context state).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_1909_06623_b200 import Context, ScError
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


def _gpu_contacts(ctx, p):
    ctx.set_walls(p.walls)
    if p.kind == "spheres":
        ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
        return ctx.get_contacts()
    ctx.build_contacts_rods(_cuda(p.pos), _cuda(p.direction), _cuda(p.length), p.rod_radius, p.gap_abs)
    return ctx.get_contacts(lever=True)


@pytest.mark.parametrize("name,n,walls", [("C1", None, "box"), ("C2", 3000, "floor"), ("C3", 4000, "box"),
                                          ("C4", 20000, "box"), ("C2", None, "box")])
def test_contacts_with_walls_bit_exact(ctx, name, n, walls):
    p = make_problem(name, n=n, walls=walls)
    g = _gpu_contacts(ctx, p)
    o = oracle.system_for(p).ct
    assert (o.j >= p.n).sum() > 0
    assert g["i"].shape[0] == o.nc
    np.testing.assert_array_equal(_np(g["i"]), o.i)
    np.testing.assert_array_equal(_np(g["j"]), o.j)
    np.testing.assert_array_equal(_np(g["gap"]).view(np.int64), o.gap.view(np.int64))
    np.testing.assert_array_equal(_np(g["normal"]).view(np.int64), o.normal.view(np.int64))
    if o.lever is not None:
        np.testing.assert_array_equal(_np(g["lever"]).view(np.int64), o.lever.view(np.int64))


@pytest.mark.parametrize("name,n,walls", [("C2", 3000, "floor"), ("C4", 20000, "box")])
def test_apply_D_DT_q_with_walls(ctx, name, n, walls):
    p = make_problem(name, n=n, walls=walls)
    _gpu_contacts(ctx, p)
    ctx.assemble_D()
    sysm = oracle.system_for(p)
    rng = np.random.default_rng(2)
    gam = rng.uniform(0, 3, sysm.ct.nc)
    Fo = oracle.apply_D(p.n, sysm.ct, gam)
    np.testing.assert_allclose(_np(ctx.apply_D(_cuda(gam))), Fo, rtol=0, atol=1e-13 * np.abs(Fo).max())
    U = rng.normal(size=(p.n, 6))
    wo = oracle.apply_DT(p.n, sysm.ct, U)
    np.testing.assert_allclose(_np(ctx.apply_DT(_cuda(U))), wo, rtol=0, atol=1e-13 * np.abs(wo).max())
    qo = sysm.lcp_q(p.dt, U)
    np.testing.assert_allclose(_np(ctx.lcp_q(p.dt, _cuda(U))), qo, rtol=0, atol=1e-13 * np.abs(qo).max())


@pytest.mark.parametrize("name,n,walls", [("C1", None, "box"), ("C2", 2048, "floor"), ("C4", 20000, "box"),
                                          ("C5", 3000, "floor")])
def test_bbpgd_converged_with_walls(ctx, name, n, walls):
    p = make_problem(name, n=n, fixed_iters=0, walls=walls)
    _gpu_contacts(ctx, p)
    ctx.assemble_D()
    ctx.lcp_q(p.dt, ctx.mobility_apply(_cuda(p.force), mu=p.mu))
    r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    o = oracle.solve_problem(p)
    assert o["status"] == 0 and o["residual"] < 1e-8
    assert r["status"] == 0 and r["converged"] == 1 and r["residual"] < 1e-8
    gam = _np(r["gamma"])
    assert gam.min() >= 0.0
    assert _relL2(gam, o["gamma"]) <= 1e-6
    assert _relL2(_np(r["Fc"]), o["Fc"]) <= 1e-6
    assert _relL2(_np(r["Uc"]), o["Uc"]) <= 1e-6
    g_cert = o["system"].mvop(gam) + o["q"]
    assert oracle.minmap_residual(gam, g_cert) < 1e-8
    # walls carry load: some wall constraint is active
    assert np.any(gam[o["system"].ct.j >= p.n] > 0)


@pytest.mark.parametrize("gap,F", [(0.05, 200.0), (0.0, 37.0)])
def test_single_sphere_on_floor_closed_form(ctx, gap, F):
    """gamma = max(0, F - 6 pi mu a gap / dt) (tests/test_oracle_walls.py); touching: gamma = F."""
    ctx.set_walls([[0.0, 0.0, 1.0, 0.0]])
    pos = np.array([[3.0, -2.0, 1.0 + gap]])
    Fext = np.zeros((1, 6)); Fext[0, 2] = -F
    assert ctx.build_contacts_spheres(_cuda(pos), _cuda(np.ones(1)), 0.0, 0.1) == 1
    ctx.assemble_D()
    ctx.lcp_q(0.01, ctx.mobility_apply(_cuda(Fext)))
    r = ctx.bbpgd_solve(tol=1e-12, max_iter=50)
    gap_b = (pos[0, 2] - 0.0) - 1.0
    want = max(0.0, F - 6 * math.pi * gap_b / 0.01)
    assert _np(r["gamma"])[0] == pytest.approx(want, rel=1e-12, abs=1e-12)
    if gap == 0.0:
        assert abs(_np(r["Uc"])[0, 2] - F / (6 * math.pi)) < 1e-12


def test_time_steps_with_floor_vs_oracle(ctx):
    """Sedimentation onto a floor: two whole time steps (U_nc, contacts incl. walls, LCP, Euler)."""
    p = make_problem("C2", n=1500, fixed_iters=0, walls="floor")
    po = make_problem("C2", n=1500, fixed_iters=0, walls="floor")
    ctx.set_walls(p.walls)
    pos_g = _cuda(p.pos)
    for _ in range(2):
        r = ctx.time_step("spheres", pos_g, _cuda(p.force), radius=_cuda(p.radius), gap_abs=p.gap_abs,
                          gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol, max_iter=p.max_iter)
        assert r["status"] == 0 and r["residual"] < 1e-8
        pos_g = r["pos"]
        o = oracle.time_step(po)
        po.pos = o["pos"]
    scale = np.abs(o["U"]).max() * p.dt
    np.testing.assert_allclose(_np(pos_g), po.pos, rtol=0, atol=1e-7 * scale + 1e-13)


def test_set_walls_errors(ctx):
    with pytest.raises(ScError) as e:
        ctx.set_walls([[0.0, 0.0, 2.0, 0.0]])  # not a unit normal
    assert e.value.code == -1
    with pytest.raises(ScError):
        ctx.set_walls(np.tile([0.0, 0.0, 1.0, 0.0], (9, 1)))  # > SC_MAX_WALLS
    ctx.set_walls(None)
    pos = np.array([[0.0, 0, 0.5], [5.0, 0, 0.5]])
    assert ctx.build_contacts_spheres(_cuda(pos), None, 0.0, 0.1) == 0  # no walls: no constraints


def test_time_steps_rods_in_box_vs_oracle(ctx):
    """Rods in a closed box: two whole time steps (contacts with pairs and walls, lever arms, drag,
    rod-axis update) against the oracle."""
    p = make_problem("C4", n=6000, fixed_iters=0, walls="box")
    po = make_problem("C4", n=6000, fixed_iters=0, walls="box")
    ctx.set_walls(p.walls)
    pos_g, dir_g = _cuda(p.pos), _cuda(p.direction)
    for _ in range(2):
        r = ctx.time_step("rods", pos_g, _cuda(p.force), direction=dir_g, length=_cuda(p.length), b=p.rod_radius,
                          gap_abs=p.gap_abs, mu=p.mu, dt=p.dt, tol=p.tol, max_iter=p.max_iter)
        assert r["status"] == 0 and r["residual"] < 1e-8
        pos_g, dir_g = r["pos"], r["dir"]
        o = oracle.time_step(po)
        po.pos, po.direction = o["pos"], o["direction"]
    scale = np.abs(o["U"]).max() * p.dt
    np.testing.assert_allclose(_np(pos_g), po.pos, rtol=0, atol=1e-7 * scale + 1e-13)
    np.testing.assert_allclose(_np(dir_g), po.direction, rtol=0, atol=1e-9)


def test_apgd_with_walls_vs_oracle(ctx):
    """The APGD comparison solver (NEXT row f3) on a problem with floor contacts."""
    p = make_problem("C1", fixed_iters=0, walls="floor")
    _gpu_contacts(ctx, p)
    ctx.assemble_D()
    ctx.lcp_q(p.dt, ctx.mobility_apply(_cuda(p.force), mu=p.mu))
    r = ctx.apgd_solve(mu=p.mu, tol=p.tol, max_iter=20000)
    sysm = oracle.system_for(p)
    q = sysm.lcp_q(p.dt, sysm.mobility(p.force))
    o = sysm.apgd(q, tol=p.tol, max_iter=20000)
    assert r["status"] == 0 and o["status"] == 0 and r["residual"] < 1e-8
    assert _relL2(_np(r["gamma"]), o["gamma"]) <= 1e-6


def test_full_rpy_with_floor(ctx):
    """Walls (f2) and the full 6N RPY (f4(ii)) together: converged solve vs the oracle."""
    p = make_problem("C3", n=1500, fixed_iters=0, walls="floor")
    p.mobility = "rpy6"
    ctx.set_mobility_model("rpy6")
    try:
        _gpu_contacts(ctx, p)
        ctx.assemble_D()
        ctx.lcp_q(p.dt, ctx.mobility_apply(_cuda(p.force), mu=p.mu))
        r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    finally:
        ctx.set_mobility_model("rpy")
    o = oracle.solve_problem(p)
    assert r["status"] == 0 and o["status"] == 0 and r["residual"] < 1e-8
    assert _relL2(_np(r["gamma"]), o["gamma"]) <= 1e-6
    assert _relL2(_np(r["Uc"]), o["Uc"]) <= 1e-6


def test_bb_breakdown_rule_squeezed_sphere(ctx):
    """Reading A5 on the GPU (and the oracle), a case where s^T y = 0 really occurs: sphere A
    (a = 1) squeezed between a floor z = 0 and a ceiling z = 1.5 (both gaps -0.25, bitwise equal),
    and sphere B (a = 0.5) near A (pair gap 0.02 > 0), no external force.  The two wall columns of
    A are +e_z and -e_z, so z = (1, 1, 0) spans null(D^T M D); q = (g_w/dt, g_w/dt, 0.02/dt).
    alpha_0 = |q|^2 / q^T M q is finite (the pair column), gamma_1 = -alpha_0 (q_1, q_1, 0) is in
    null(M): y = 0, s^T y = 0 -> breakdown; the LCP is infeasible (A cannot leave both walls), so
    every iteration breaks down, gamma grows linearly, status SC_NOT_CONVERGED and
    bb_breakdowns = iterations on both sides (Steps 14-15 run at j = j_max too)."""
    pos = np.array([[0.0, 0.0, 0.75], [1.52, 0.0, 0.75]])
    rad = np.array([1.0, 0.5])
    walls = np.array([[0.0, 0.0, 1.0, 0.0], [0.0, 0.0, -1.0, -1.5]])
    F = np.zeros((2, 6))
    dt = 0.01
    ctx.set_walls(walls)
    for J in (1, 5, 40):
        ctx.build_contacts_spheres(_cuda(pos), _cuda(rad), 0.0, 0.1)
        c = ctx.get_contacts()
        np.testing.assert_array_equal(_np(c["i"]), [0, 0, 0])
        np.testing.assert_array_equal(_np(c["j"]), [1, 2, 3])
        ctx.assemble_D()
        U = ctx.mobility_apply(_cuda(F))
        ctx.lcp_q(dt, U)
        r = ctx.bbpgd_solve(tol=1e-8, max_iter=J)
        ct = oracle.merge_contacts(oracle.contacts_spheres(pos, rad, 0.0, 0.1),
                                   oracle.contacts_walls("spheres", pos, walls, radius=rad, gap_abs=0.0,
                                                         gap_rel=0.1))
        sysm = oracle.System(oracle.ORC_SPHERES, 2, ct, pos=pos, radius=rad)
        q = sysm.lcp_q(dt, sysm.mobility(F))
        o = sysm.bbpgd(q, tol=1e-8, max_iter=J)
        gam = _np(r["gamma"])
        assert r["status"] == 1 and o["status"] == 1
        assert r["bb_breakdowns"] == J and o["bb_breakdowns"] == J and r["iters"] == J == o["iters"]
        assert gam[1] == gam[2] and gam[0] == 0.0 and gam[1] > 0  # grows along the null direction
        np.testing.assert_allclose(gam, o["gamma"], rtol=1e-12, atol=0)
        # gamma_J = J alpha_0 |q_w| (alpha kept at alpha_0; g_j = q)
        assert gam[1] == pytest.approx(J * r["alpha"] * abs(q[1]), rel=1e-12)
    ctx.set_walls(None)


@pytest.mark.parametrize("name,n,walls", [("C2", 3000, "floor"), ("C4", 20000, "box"), ("C1", None, "box")])
def test_moving_walls_q_and_solve_vs_oracle(ctx, name, n, walls):
    """Moving boundaries: q = gap/dt + D^T U_ext - n_k.V_k on wall rows (the
    oracle's orc_lcp_q_moving_walls), and the converged solve against the oracle's."""
    p = make_problem(name, n=n, walls=walls, fixed_iters=0)
    rng = np.random.default_rng(7)
    V = rng.normal(size=(len(p.walls), 3)) * 5.0
    _gpu_contacts(ctx, p)
    ctx.set_wall_velocities(V)
    ctx.assemble_D()
    F = _cuda(p.force)
    U = ctx.mobility_apply(F, mu=p.mu)
    q = _np(ctx.lcp_q(p.dt, U))
    r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    sysm = oracle.system_for(p)
    Uo = sysm.mobility(p.force)
    qo = sysm.lcp_q_moving_walls(p.dt, Uo, V)
    np.testing.assert_allclose(q, qo, rtol=0, atol=1e-12 * np.abs(qo).max())
    o = sysm.bbpgd(qo, tol=p.tol, max_iter=p.max_iter)
    assert r["status"] == 0 and o["status"] == 0
    assert _relL2(_np(r["gamma"]), o["gamma"]) <= 1e-6
    ctx.set_walls(None)


def test_moving_floor_closed_form_and_time_step(ctx):
    """One sphere above a floor moving up with V (F = 0): gamma = max(0, 6 pi (V - gap/dt)); the
    time step moves the plane to h + dt V_z and the sphere with the floor when in contact."""
    dt = 0.01
    pos = np.array([[0.0, 0.0, 1.05]])
    for V, expect in ((10.0, 6 * np.pi * (10.0 - 5.0)), (3.0, 0.0)):
        ctx.set_walls([[0.0, 0.0, 1.0, 0.0]])
        ctx.set_wall_velocities([[0.5, 0.0, V]])
        ctx.build_contacts_spheres(_cuda(pos), None, 0.0, 0.1)
        ctx.assemble_D()
        ctx.lcp_q(dt, ctx.mobility_apply(_cuda(np.zeros((1, 6)))))
        r = ctx.bbpgd_solve(tol=1e-10, max_iter=50)
        assert float(r["gamma"][0]) == pytest.approx(expect, rel=1e-12, abs=1e-12)
        quat = torch.tensor([[1.0, 0.0, 0.0, 0.0]], dtype=torch.float64, device="cuda")
        out = ctx.time_step("spheres", _cuda(pos), _cuda(np.zeros((1, 6))), dt=dt, tol=1e-10, quat=quat)
        w = ctx.get_walls()
        assert w[0, 3] == pytest.approx(dt * V, rel=1e-15)
        z1 = float(out["pos"][0, 2])
        if expect > 0:  # pushed by the floor: the linearised gap closes exactly at the step end
            assert z1 == pytest.approx(1.0 + dt * V, rel=1e-12)
        else:
            assert z1 == 1.05
    ctx.set_walls(None)


def test_wall_velocity_errors(ctx):
    ctx.set_walls([[0.0, 0.0, 1.0, 0.0], [0.0, 0.0, -1.0, -10.0]])
    with pytest.raises(ScError):
        ctx.set_wall_velocities([[0.0, 0.0, 1.0]])  # one velocity per wall
    with pytest.raises(ScError):
        ctx.set_wall_velocities([[0.0, 0.0, np.nan], [0.0, 0.0, 0.0]])
    ctx.set_wall_velocities([[0.0, 0.0, 1.0], [0.0, 0.0, 0.0]])
    ctx.set_walls([[0.0, 0.0, 1.0, 0.0]])  # new walls: velocities reset to 0
    np.testing.assert_array_equal(ctx.get_walls(), [[0.0, 0.0, 1.0, 0.0]])
    ctx.set_walls(None)
