"""Pins for the oracle's collision matrix D and D^T.

D^T = (grad_C Phi) G (Eq. Dtranspose) is checked by finite
differences of the oracle's own contact geometry under rigid motions: the
gap rate must equal D^T U.  This pins the sign convention, the normal and the
rod lever arms (12-nnz columns) independently of how D is stored.
"""
import numpy as np
import pytest

import oracle
from paper_1909_06623_b200.synthetic import make_problem


def test_single_pair_DtD_and_forces():
    pos = np.array([[0.0, 0, 0], [2.05, 0, 0]])
    ct = oracle.contacts_spheres(pos, np.ones(2), 0.0, 0.1)
    FT = oracle.apply_D(2, ct, np.array([5.0]))
    # +n on i, -n on j, n from j to i; no torque on spheres
    np.testing.assert_array_equal(FT[0], [-5, 0, 0, 0, 0, 0])
    np.testing.assert_array_equal(FT[1], [5, 0, 0, 0, 0, 0])
    # D^T D = [2]
    assert oracle.apply_DT(2, ct, oracle.apply_D(2, ct, np.array([1.0])))[0] == 2.0
    # head-on approach with speeds +-1: the gap shrinks at rate 2
    U = np.zeros((2, 6)); U[0, 0] = 1.0; U[1, 0] = -1.0
    assert oracle.apply_DT(2, ct, U)[0] == -2.0


@pytest.mark.parametrize("name,n", [("C1", 512), ("C2", 1500), ("C4", 1500)])
def test_adjoint_and_newton_third_law(name, n):
    p = make_problem(name, n=n)
    sysm = oracle.system_for(p)
    ct = sysm.ct
    rng = np.random.default_rng(3)
    gamma = rng.uniform(0, 2, ct.nc)
    U = rng.normal(size=(n, 6))
    F = oracle.apply_D(n, ct, gamma)
    lhs = float(np.sum(F * U))
    rhs = float(np.dot(gamma, oracle.apply_DT(n, ct, U)))
    assert abs(lhs - rhs) <= 1e-13 * (np.sum(np.abs(F * U)) + 1)
    # Newton's third law: contact forces sum to zero
    assert np.abs(F[:, :3].sum(0)).max() <= 1e-12 * np.abs(F[:, :3]).sum()
    if p.kind == "spheres":
        assert np.all(F[:, 3:] == 0.0)
    else:
        # total torque about the origin also vanishes: sum(c x F + T) = 0
        tot = np.cross(p.pos, F[:, :3]).sum(0) + F[:, 3:].sum(0)
        assert np.abs(tot).max() <= 1e-10 * np.abs(F).sum()


def _sphere_gaps(pos, radius, ct):
    d = pos[ct.i] - pos[ct.j]
    return np.linalg.norm(d, axis=1) - radius[ct.i] - radius[ct.j]


def test_fd_gap_rate_spheres():
    p = make_problem("C2", n=1200)
    ct = oracle.contacts_spheres(p.pos, p.radius, p.gap_abs, p.gap_rel)
    rng = np.random.default_rng(5)
    U = np.zeros((p.n, 6)); U[:, :3] = rng.normal(size=(p.n, 3))
    h = 1e-6
    fd = (_sphere_gaps(p.pos + h * U[:, :3], p.radius, ct) - _sphere_gaps(p.pos - h * U[:, :3], p.radius, ct)) / (2 * h)
    np.testing.assert_allclose(oracle.apply_DT(p.n, ct, U), fd, rtol=0, atol=1e-7)


def _rot(t, w, h):
    """Rotate the unit vectors t by angle |w| h about w (Rodrigues)."""
    th = np.linalg.norm(w, axis=1, keepdims=True) * h
    k = w / np.maximum(np.linalg.norm(w, axis=1, keepdims=True), 1e-300)
    return t * np.cos(th) + np.cross(k, t) * np.sin(th) + k * np.sum(k * t, axis=1, keepdims=True) * (1 - np.cos(th))


def _rod_gaps(center, direction, length, b, ct):
    out = np.empty(ct.nc)
    for l in range(ct.nc):
        i, j = ct.i[l], ct.j[l]
        P1, P2 = oracle.segment_closest(center[i], direction[i], length[i], center[j], direction[j], length[j])
        out[l] = np.linalg.norm(P1 - P2) - 2 * b
    return out


def test_fd_gap_rate_rods_levers():
    """Eq. Dtranspose for spherocylinders: pins the 12-nnz columns (n, r x n)."""
    p = make_problem("C4", n=1500)
    ct = oracle.contacts_rods(p.pos, p.direction, p.length, 0.5, 0.1)
    rng = np.random.default_rng(9)
    U = rng.normal(size=(p.n, 6))
    h = 1e-6
    gp = _rod_gaps(p.pos + h * U[:, :3], _rot(p.direction, U[:, 3:], h), p.length, 0.5, ct)
    gm = _rod_gaps(p.pos - h * U[:, :3], _rot(p.direction, U[:, 3:], -h), p.length, 0.5, ct)
    fd = (gp - gm) / (2 * h)
    an = oracle.apply_DT(p.n, ct, U)
    # exclude pairs near a clamp switch or with nearly crossing axes
    dist = ct.gap + 1.0
    keep = dist > 1e-3
    err = np.abs(fd - an)[keep]
    frac_ok = np.mean(err < 1e-6 * (1 + np.abs(an[keep])))
    assert keep.sum() > 500 and frac_ok > 0.98, frac_ok
    # contact torques are perpendicular to the rod axis (reading A15)
    F = oracle.apply_D(p.n, ct, rng.uniform(0, 1, ct.nc))
    assert np.abs(np.sum(F[:, 3:] * p.direction, axis=1)).max() < 1e-10 * (1 + np.abs(F).max())
