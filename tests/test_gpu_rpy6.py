"""GPU parity for the full 6N RPY grand mobility (NEXT row f4(ii), reading A27) against the
oracle (tests/test_oracle_rpy6.py pins the oracle).  Bars: mobility rel. L2 <= 1e-12 (U and
Omega separately); converged gamma / D gamma / U_c rel. L2 <= 1e-6 with phi < 1e-8."""
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
    c.set_mobility_model("rpy6")
    yield c
    c.close()


def _cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def _np(t):
    return t.detach().cpu().numpy()


def _relL2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def _with_torques(p, seed=7):
    FT = p.force.copy()
    rng = np.random.default_rng(seed)
    FT[:, 3:] += rng.normal(size=(p.n, 3))
    return FT


@pytest.mark.parametrize("name,n", [("C1", None), ("C2", 1500), ("C3", 3000), ("C1", 1), ("C1", 3), ("C5", 700)])
def test_rpy6_apply_parity(ctx, name, n):
    p = make_problem(name, n=n)
    FT = _with_torques(p)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    UW = _np(ctx.mobility_apply(_cuda(FT), mu=p.mu))
    Uo = oracle.rpy6_apply(p.pos, p.radius, p.mu, FT)
    assert _relL2(UW[:, :3], Uo[:, :3]) <= 1e-12
    assert _relL2(UW[:, 3:], Uo[:, 3:]) <= 1e-12


def test_rpy6_full_size_c3_sampled_rows(ctx):
    p = make_problem("C3")
    FT = p.force  # the C3 rotor torques (0, 0, +-1)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    UW = _np(ctx.mobility_apply(_cuda(FT), mu=p.mu))
    rows = np.r_[0:24, 32760:32784, p.n - 24:p.n]
    for r0 in (0, 32760, p.n - 24):
        Uo = oracle.rpy6_apply(p.pos, p.radius, p.mu, FT, r0, r0 + 24)
        assert _relL2(UW[r0:r0 + 24, :3], Uo[:, :3]) <= 1e-12
        assert _relL2(UW[r0:r0 + 24, 3:], Uo[:, 3:]) <= 1e-12
    assert rows.size == 72


@pytest.mark.parametrize("name,n", [("C3", 2000), ("C1", None)])
def test_rpy6_collision_solve_parity(ctx, name, n):
    """With the coupling blocks, C3's rotor torques change q (through tr) and hence gamma."""
    p = make_problem(name, n=n, fixed_iters=0)
    p.mobility = "rpy6"
    FT = p.force if name == "C3" else _with_torques(p)
    p.force = FT
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    ctx.assemble_D()
    ctx.lcp_q(p.dt, ctx.mobility_apply(_cuda(FT), mu=p.mu))
    r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    o = oracle.solve_problem(p)
    assert o["status"] == 0 and r["status"] == 0 and r["residual"] < 1e-8
    gam = _np(r["gamma"])
    assert _relL2(gam, o["gamma"]) <= 1e-6
    assert _relL2(_np(r["Fc"]), o["Fc"]) <= 1e-6
    assert _relL2(_np(r["Uc"])[:, :3], o["Uc"][:, :3]) <= 1e-6
    assert _relL2(_np(r["Uc"])[:, 3:], o["Uc"][:, 3:]) <= 1e-6
    assert np.abs(o["Uc"][:, 3:]).max() > 0.0  # contact forces now spin the spheres
    if name == "C3":  # the torques are no longer inert (contrast reading A18)
        p0 = make_problem(name, n=n, fixed_iters=0)
        o0 = oracle.solve_problem(p0)
        assert _relL2(o0["gamma"], o["gamma"]) > 1e-6


def test_rpy6_time_step_quaternions(ctx):
    """A whole time step with the full mobility: centres and quaternions vs the oracle."""
    p = make_problem("C3", n=1500, fixed_iters=0)
    p.mobility = "rpy6"
    quat = np.tile([1.0, 0.0, 0.0, 0.0], (p.n, 1))
    qg = _cuda(quat)
    r = ctx.time_step("spheres", _cuda(p.pos), _cuda(p.force), radius=_cuda(p.radius), gap_abs=p.gap_abs,
                      gap_rel=p.gap_rel, mu=p.mu, dt=p.dt, tol=p.tol, max_iter=p.max_iter, quat=qg)
    o = oracle.time_step(p, quat=quat.copy())
    assert r["status"] == 0
    scale = np.abs(o["U"]).max() * p.dt
    np.testing.assert_allclose(_np(r["pos"]), o["pos"], rtol=0, atol=1e-7 * scale + 1e-13)
    np.testing.assert_allclose(_np(qg), o["quat"], rtol=0, atol=1e-9)
    assert np.abs(o["quat"][:, 1:]).max() > 1e-6  # the rotors turn
