"""Pins for the oracle's full 6N RPY grand mobility (NEXT row f4(ii), reading A27).

The translation-rotation (rt, tr) and rotation-rotation (rr) pair blocks are not printed in the
paper (it cites RPY); they are pinned here independently of their formulas:
  * far field: rt = 1/2 curl of the translational RPY field of a point force (finite
    differences of orc_rpy_block, already pinned by test_oracle_mobility.py), rr = 1/2 curl of
    the rotlet field U(x) = tr block (the curl of a rotlet is a potential dipole);
  * the overlap branch joins the far field with a continuous value AND slope at r = 2a, and
    tends to the self blocks at r -> 0 (rt -> 0, rr -> I/(8 pi mu a^3));
  * grand-mobility symmetry M_ij = M_ji^T and positive definiteness of the 6N x 6N matrix;
  * with zero torques the translational output equals orc_rpy_apply's.
"""
import math

import numpy as np
import pytest

import oracle
from paper_1909_06623_b200.synthetic import make_problem

MU = 1.0


def _blk(xi, ai, xj, aj, self_block=False):
    return oracle.rpy6_block(np.asarray(xi, float), ai, np.asarray(xj, float), aj, MU, self_block)


def _curl(field, x, h=1e-5):
    """central-difference curl of a vector field R^3 -> R^3 at x."""
    J = np.zeros((3, 3))
    for k in range(3):
        e = np.zeros(3); e[k] = h
        J[:, k] = (field(x + e) - field(x - e)) / (2 * h)
    return np.array([J[2, 1] - J[1, 2], J[0, 2] - J[2, 0], J[1, 0] - J[0, 1]])


@pytest.mark.parametrize("r,ai,aj", [(3.0, 1.0, 1.0), (5.5, 1.0, 1.0), (2.6, 0.7, 0.9), (9.0, 0.5, 1.0)])
def test_far_field_blocks_are_half_curls(r, ai, aj):
    rng = np.random.default_rng(int(r * 10))
    d = rng.normal(size=3); d /= np.linalg.norm(d)
    xj = np.array([0.3, -0.2, 0.5])
    xi = xj + r * d
    F = rng.normal(size=3)
    T = rng.normal(size=3)
    M = _blk(xi, ai, xj, aj)
    # rt: Omega_i = 1/2 curl_x [ M_tt(x; x_j) F ] at x = x_i
    u_f = lambda x: oracle.rpy_block(x, ai, xj, aj, MU) @ F
    np.testing.assert_allclose(M[3:, :3] @ F, 0.5 * _curl(u_f, xi), rtol=1e-7, atol=1e-12)
    # rr: Omega_i = 1/2 curl_x [ M_tr(x; x_j) T ] at x = x_i (the rotlet field)
    u_t = lambda x: _blk(x, ai, xj, aj)[:3, 3:] @ T
    np.testing.assert_allclose(M[3:, 3:] @ T, 0.5 * _curl(u_t, xi), rtol=1e-7, atol=1e-12)
    # the rotlet is the textbook T x r / (8 pi mu r^3), r = x_i - x_j
    rv = xi - xj
    np.testing.assert_allclose(M[:3, 3:] @ T, np.cross(T, rv) / (8 * math.pi * MU * r ** 3), rtol=1e-13)


@pytest.mark.parametrize("ai,aj", [(1.0, 1.0), (0.6, 0.9)])
def test_branches_join_c1_at_contact_and_self_limits(ai, aj):
    a = 0.5 * (ai + aj)
    d = np.array([0.48, -0.6, 0.64])  # unit
    xj = np.zeros(3)
    blk = lambda r: _blk(xj + r * d, ai, xj, aj)
    r0 = 2 * a
    h = 1e-6 * r0
    lo, hi = blk(r0 * (1 - 1e-12)), blk(r0 * (1 + 1e-12))
    np.testing.assert_allclose(lo, hi, rtol=0, atol=1e-12)
    # slopes from each side agree (one-sided differences)
    dlo = (blk(r0 - 1e-9 * r0) - blk(r0 - h)) / (h - 1e-9 * r0)
    dhi = (blk(r0 + h) - blk(r0 + 1e-9 * r0)) / (h - 1e-9 * r0)
    np.testing.assert_allclose(dlo, dhi, rtol=0, atol=2e-5 * np.abs(dhi).max())
    # r -> 0: rt -> 0, rr -> the self rotation block, tt -> the self translation block
    small = blk(1e-9)
    np.testing.assert_allclose(small[3:, :3], 0.0, atol=1e-9)
    np.testing.assert_allclose(small[3:, 3:], np.eye(3) / (8 * math.pi * MU * a ** 3), rtol=1e-8, atol=1e-10)
    np.testing.assert_allclose(small[:3, :3], np.eye(3) / (6 * math.pi * MU * a), rtol=1e-8, atol=1e-10)


def test_self_blocks():
    S = _blk(np.zeros(3), 0.8, np.zeros(3), 0.8, self_block=True)
    np.testing.assert_allclose(S[:3, :3], np.eye(3) / (6 * math.pi * 0.8))
    np.testing.assert_allclose(S[3:, 3:], np.eye(3) / (8 * math.pi * 0.8 ** 3))
    assert np.all(S[:3, 3:] == 0) and np.all(S[3:, :3] == 0)


def _grand(pos, radius):
    n = pos.shape[0]
    M = np.zeros((6 * n, 6 * n))
    for i in range(n):
        for j in range(n):
            M[6 * i:6 * i + 6, 6 * j:6 * j + 6] = _blk(pos[i], radius[i], pos[j], radius[j], i == j)
    return M


@pytest.mark.parametrize("name,n", [("C1", 60), ("C3", 50), ("C2", 40)])
def test_grand_mobility_symmetric_positive_definite(name, n):
    p = make_problem(name, n=n)
    M = _grand(p.pos, p.radius)
    np.testing.assert_allclose(M, M.T, rtol=0, atol=1e-15)
    lam = np.linalg.eigvalsh(0.5 * (M + M.T))
    assert lam.min() > 0.0, lam.min()
    # apply == the dense matrix; zero torques reproduce the translational apply
    rng = np.random.default_rng(4)
    FT = rng.normal(size=(n, 6))
    np.testing.assert_allclose(oracle.rpy6_apply(p.pos, p.radius, MU, FT).ravel(), M @ FT.ravel(),
                               rtol=0, atol=1e-13 * np.abs(M @ FT.ravel()).max())
    F0 = FT.copy(); F0[:, 3:] = 0.0
    np.testing.assert_allclose(oracle.rpy6_apply(p.pos, p.radius, MU, F0)[:, :3],
                               oracle.rpy_apply(p.pos, p.radius, MU, F0)[:, :3], rtol=0, atol=1e-14)


def test_rotor_torques_now_move_neighbours():
    """C3's rotor torques are inert under the translational RPY (reading A18) but drive
    translational velocities through the tr coupling: U_i = sum_j T_j x r_ij / (8 pi mu r^3)."""
    p = make_problem("C3", n=300)
    T = np.zeros((p.n, 6)); T[:, 5] = p.force[:, 5]
    U6 = oracle.rpy6_apply(p.pos, p.radius, MU, T)
    U3 = oracle.rpy_apply(p.pos, p.radius, MU, T)
    assert np.abs(U3[:, :3]).max() == 0.0
    assert np.abs(U6[:, :3]).max() > 1e-3
    # the translational velocity of torque-driven spheres lies in the xy plane (T || z)
    assert np.abs(U6[:, 2]).max() <= 1e-15 * np.abs(U6[:, :2]).max() + 1e-300
