"""Pins for the oracle's mobility apply (RPY spheres, drag rods).

The formula is BASELINE.json configs[0] (the paper only cites RPY,
P:L87-L91; reading A10).  Pins independent of the formula's transcription:
single-sphere Stokes drag, continuity of the two branches at
r = 2a to closed-form constants, the far-field Stokeslet limit, symmetry and
positive definiteness of the assembled matrix by eigenvalues, translational
invariance, rotational equivariance, crowding speeds sedimentation
(P:L1198), and the rod drag eigen-decomposition.
"""
import math

import mpmath as mp
import numpy as np
import pytest

import oracle
from paper_1909_06623_b200.synthetic import make_problem

PI = math.pi


def test_single_sphere_drag():
    # U = F/(6 pi mu a), Omega = T/(8 pi mu a^3)
    for a, mu in [(1.0, 1.0), (0.5, 2.0)]:
        FT = np.array([[6 * PI * mu * a, 0, 0, 0, 0, 8 * PI * mu * a ** 3]])
        UW = oracle.rpy_apply(np.zeros((1, 3)), np.array([a]), mu, FT)
        np.testing.assert_allclose(UW[0], [1, 0, 0, 0, 0, 1], rtol=1e-15, atol=1e-16)
    UW = oracle.rpy_apply(np.zeros((1, 3)), np.ones(1), 1.0, np.array([[0, 0, 0, 0, 0, 1.0]]))
    assert UW[0, 5] == pytest.approx(0.039788735772973834, rel=1e-15)  # 1/(8 pi)


def test_branch_continuity_at_contact():
    # both branches at r = 2a: 7/(96 pi mu a) I + 1/(32 pi mu a) rhat rhat^T
    mp.mp.dps = 30
    ci = float(mp.mpf(7) / (96 * mp.pi))
    cr = float(mp.mpf(1) / (32 * mp.pi))
    assert ci == pytest.approx(0.02321009586756807, rel=1e-15)
    assert cr == pytest.approx(0.0099471839432434585, rel=1e-15)
    rh = np.array([1.0, 2.0, -2.0]) / 3.0
    want = ci * np.eye(3) + cr * np.outer(rh, rh)
    for eps in (1e-9, -1e-9):
        M = oracle.rpy_block(np.zeros(3), 1.0, (2.0 + eps) * rh, 1.0, 1.0)
        np.testing.assert_allclose(M, want, rtol=0, atol=1e-10)


def test_far_field_stokeslet():
    rh = np.array([0.0, 0.6, 0.8])
    for r in (1e3, 1e5):
        M = oracle.rpy_block(np.zeros(3), 1.0, r * rh, 1.0, 1.0)
        S = (np.eye(3) + np.outer(rh, rh)) / (8 * PI * r)
        np.testing.assert_allclose(M, S, rtol=0, atol=2.0 / r ** 3)


def test_overlap_branch_at_zero_separation_limit():
    # r -> 0: the near branch tends to the self mobility I/(6 pi mu a) (reading A10)
    M = oracle.rpy_block(np.zeros(3), 1.0, np.array([1e-12, 0, 0]), 1.0, 1.0)
    np.testing.assert_allclose(M, np.eye(3) / (6 * PI), atol=1e-12)


def _dense(pos, radius, mu):
    n = pos.shape[0]
    M = np.zeros((3 * n, 3 * n))
    for i in range(n):
        for j in range(n):
            M[3 * i:3 * i + 3, 3 * j:3 * j + 3] = oracle.rpy_block(pos[i], radius[i], pos[j], radius[j], mu, i == j)
    return M


@pytest.mark.parametrize("name,n", [("C1", 160), ("C2", 160), ("C3", 160)])
def test_assembled_matrix_symmetric_spd_and_matches_apply(name, n):
    p = make_problem(name, n=n)
    M = _dense(p.pos, p.radius, p.mu)
    assert np.abs(M - M.T).max() <= 1e-15 * np.abs(M).max()
    lam = np.linalg.eigvalsh(M)
    assert lam.min() > 0, lam.min()
    # matrix-free apply == dense matvec (the apply's loop, long double sums)
    F = np.zeros((n, 6)); F[:, :3] = np.random.default_rng(1).normal(size=(n, 3))
    UW = oracle.rpy_apply(p.pos, p.radius, p.mu, F)
    np.testing.assert_allclose(UW[:, :3].ravel(), M @ F[:, :3].ravel(), rtol=1e-13, atol=1e-15)


def test_invariance_and_equivariance():
    p = make_problem("C2", n=300)
    rng = np.random.default_rng(7)
    F = np.zeros((p.n, 6)); F[:, :3] = rng.normal(size=(p.n, 3)); F[:, 3:] = rng.normal(size=(p.n, 3))
    U0 = oracle.rpy_apply(p.pos, p.radius, 1.0, F)
    U1 = oracle.rpy_apply(p.pos + np.array([3.25, -7.5, 1e3]), p.radius, 1.0, F)
    np.testing.assert_allclose(U1, U0, rtol=0, atol=1e-12 * np.abs(U0).max())
    # rotate positions, forces and torques by R -> velocities rotate by R
    A = rng.normal(size=(3, 3)); R, _ = np.linalg.qr(A)
    if np.linalg.det(R) < 0:
        R[:, 0] *= -1
    FR = np.concatenate([F[:, :3] @ R.T, F[:, 3:] @ R.T], axis=1)
    UR = oracle.rpy_apply(p.pos @ R.T, p.radius, 1.0, FR)
    np.testing.assert_allclose(UR[:, :3], U0[:, :3] @ R.T, rtol=0, atol=1e-10 * np.abs(U0).max())
    np.testing.assert_allclose(UR[:, 3:], U0[:, 3:] @ R.T, rtol=0, atol=1e-12 * np.abs(U0).max())
    # storage-order permutation
    perm = rng.permutation(p.n)
    UP = oracle.rpy_apply(p.pos[perm], p.radius[perm], 1.0, F[perm])
    np.testing.assert_allclose(UP, U0[perm], rtol=0, atol=1e-13 * np.abs(U0).max())


def test_crowding_speeds_sedimentation():
    # two equal spheres pushed the same way sediment faster than one
    F = np.array([[0, 0, -1.0, 0, 0, 0], [0, 0, -1.0, 0, 0, 0]])
    one = oracle.rpy_apply(np.zeros((1, 3)), np.ones(1), 1.0, F[:1])[0, 2]
    for d in (2.5, 5.0, 1.5):
        two = oracle.rpy_apply(np.array([[0, 0, 0.0], [d, 0, 0]]), np.ones(2), 1.0, F)
        assert two[0, 2] < one < 0 and two[0, 2] == two[1, 2]
    # coupling decays ~1/r (leading Stokeslet order)
    c = [oracle.rpy_block(np.zeros(3), 1, np.array([d, 0, 0]), 1, 1)[1, 1] for d in (50.0, 100.0)]
    assert c[0] / c[1] == pytest.approx(2.0, rel=1e-3)


def test_equal_radii_reduce_to_monodisperse():
    p = make_problem("C1", n=200)
    F = np.random.default_rng(2).normal(size=(200, 6))
    U1 = oracle.rpy_apply(p.pos, np.ones(200), 1.0, F)
    U2 = oracle.rpy_apply(p.pos * 0.5, np.full(200, 0.5), 1.0, F)
    # scaling: positions and radii by s -> translational mobility by 1/s, rotational by 1/s^3
    np.testing.assert_allclose(U2[:, :3], 2 * U1[:, :3], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(U2[:, 3:], 8 * U1[:, 3:], rtol=1e-14)


def test_rod_drag_eigenvectors():
    b, mu = 0.5, 1.0
    for L in (2.0, 3.3, 4.0):
        lg = math.log(L / (2 * b))
        zpar = 2 * PI * mu * L / lg
        zperp = 2 * zpar
        zrot = PI * mu * L ** 3 / (3 * lg)
        t = np.array([[0.0, 0.6, 0.8]])
        tp = np.array([1.0, 0.0, 0.0])
        F = np.concatenate([t[0], [0.0, 0.0, 0.0]])[None]
        U = oracle.rod_drag_apply(t, np.array([L]), b, mu, F)
        np.testing.assert_allclose(U[0, :3], t[0] / zpar, rtol=1e-14)
        F = np.concatenate([tp, [0.3, -0.2, 0.1]])[None]
        U = oracle.rod_drag_apply(t, np.array([L]), b, mu, F)
        np.testing.assert_allclose(U[0, :3], tp / zperp, rtol=1e-14, atol=1e-17)
        np.testing.assert_allclose(U[0, 3:], np.array([0.3, -0.2, 0.1]) / zrot, rtol=1e-14)
