"""Pins for the oracle's time step (NEXT row f1).

* an isolated body translates by dt F/(6 pi mu a) exactly and its quaternion turns by
  |Omega| dt about Omega (first order), staying unit;
* rods: the axis rotates by Omega x t and stays unit;
* head-on contact: the linearised gap after the step is >= 0 and the pair separates no
  faster than complementarity allows (gap' = 0 for a touching pair pushed together);
* a C1 step leaves every linearised gap Phi + dt D^T U >= -tol*dt (complementarity).
"""
import math

import numpy as np
import pytest

import oracle
from paper_1909_06623_b200.synthetic import make_problem


def test_isolated_sphere_translation_and_rotation():
    pos = np.array([[1.0, 2.0, 3.0]])
    F = np.array([[6 * math.pi, 0, 0, 0, 0, 8 * math.pi * 0.1]])  # U = (1,0,0), Omega = (0,0,0.1)
    U = oracle.rpy_apply(pos, np.ones(1), 1.0, F)
    q0 = np.array([[1.0, 0, 0, 0]])
    dt = 0.01
    p1, q1, _ = oracle.euler_update(dt, U, pos, q0)
    np.testing.assert_allclose(p1, pos + dt * np.array([[1.0, 0, 0]]), rtol=0, atol=1e-15)
    assert abs(np.linalg.norm(q1) - 1) < 1e-15
    # rotation by angle |Omega| dt about z: q = (cos(th/2), 0, 0, sin(th/2)) to first order
    th = 0.1 * dt
    np.testing.assert_allclose(q1[0], [math.cos(th / 2), 0, 0, math.sin(th / 2)], atol=1e-7)


def test_rod_axis_rotates_and_stays_unit():
    t = np.array([[1.0, 0, 0]])
    W = np.array([[0, 0, 0, 0, 0, 2.0]])  # Omega = 2 z
    p, _, t1 = oracle.euler_update(0.001, W, np.zeros((1, 3)), None, t)
    assert abs(np.linalg.norm(t1) - 1) < 1e-15
    ang = math.atan2(t1[0, 1], t1[0, 0])
    assert ang == pytest.approx(math.atan(0.002), rel=1e-13)  # Euler + normalise: tan(angle) = |Omega| dt
    np.testing.assert_array_equal(p, 0.0)


def test_headon_touching_pair_stays_touching():
    p = make_problem("C1", n=2)
    p.pos = np.array([[0.0, 0, 0], [2.0, 0, 0]])
    p.force = np.zeros((2, 6)); p.force[0, 0] = 5.0; p.force[1, 0] = -5.0
    r = oracle.time_step(p)
    d = np.linalg.norm(r["pos"][0] - r["pos"][1])
    assert d == pytest.approx(2.0, abs=1e-12)  # pushed together, held at contact (gamma = F)
    assert r["gamma"][0] == pytest.approx(5.0, rel=1e-12)


def test_c1_step_linearised_gaps_nonnegative():
    p = make_problem("C1")
    r = oracle.time_step(p)
    sysm = r["system"]
    lin = sysm.ct.gap + p.dt * oracle.apply_DT(p.n, sysm.ct, r["U"])
    assert lin.min() >= -p.tol * p.dt * 10
    # the total velocity is U_nc + U_c and positions moved by dt U
    np.testing.assert_allclose(r["pos"], p.pos + p.dt * r["U"][:, :3], rtol=0, atol=1e-12)
