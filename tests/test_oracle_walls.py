"""Pins for the oracle's particle-boundary constraints (NEXT row f2).

A boundary contributes columns D_l with entries on the particle only and does not appear in
the mobility.  Pinned here by hand examples, a brute-force minimisation of the
rod-plane distance, a finite-difference check of Eq. Dtranspose for wall
columns (pins the rod lever arm), and the closed form of a single sphere pushed onto a floor:
A = n.M n = 1/(6 pi mu a), q = gap/dt - F/(6 pi mu a), gamma = max(0, F - 6 pi mu a gap/dt).
"""
import math

import numpy as np
import pytest

import oracle
from paper_1909_06623_b200.synthetic import make_problem, make_walls

FLOOR = np.array([[0.0, 0.0, 1.0, 0.0]])


def test_sphere_floor_hand_examples():
    pos = np.array([[5.0, 5.0, 1.05], [9.0, 9.0, 1.2], [1.0, 3.0, 0.5]])
    ct = oracle.contacts_walls("spheres", pos, FLOOR, radius=np.ones(3), gap_abs=0.0, gap_rel=0.1)
    # z = 1.05: gap 0.05 < 0.1 (contact); z = 1.2: gap 0.2 (none); z = 0.5: overlap -0.5
    assert list(ct.i) == [0, 2] and list(ct.j) == [3, 3]
    np.testing.assert_allclose(ct.gap, [0.05, -0.5], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(ct.normal, [[0, 0, 1], [0, 0, 1]])
    # D column on the particle only: F = gamma n on body i, nothing else
    F = oracle.apply_D(3, ct, np.array([2.0, 3.0]))
    np.testing.assert_array_equal(F[0], [0, 0, 2, 0, 0, 0])
    np.testing.assert_array_equal(F[1], np.zeros(6))
    np.testing.assert_array_equal(F[2], [0, 0, 3, 0, 0, 0])
    # D^T U: the gap rate is the normal velocity of the particle (the wall is at rest)
    U = np.zeros((3, 6)); U[0, 2] = -1.5; U[2, :] = [7, 8, 9, 1, 1, 1]
    np.testing.assert_array_equal(oracle.apply_DT(3, ct, U), [-1.5, 9.0])


def test_box_corner_three_walls():
    box = 10.0
    walls = make_walls("box", box)
    pos = np.array([[0.5, 0.5, 0.5], [5.0, 5.0, 5.0], [9.95, 5.0, 0.98]])
    ct = oracle.contacts_walls("spheres", pos, walls, radius=np.ones(3), gap_abs=0.0, gap_rel=0.1)
    # body 0 overlaps the three low faces (x, y, z = 0); body 1 touches nothing; body 2 the x = box
    # face (gap -0.95) and the floor (gap -0.02)
    assert [(int(i), int(j) - 3) for i, j in zip(ct.i, ct.j)] == [(0, 0), (0, 2), (0, 4), (2, 1), (2, 4)]
    np.testing.assert_allclose(ct.gap, [-0.5, -0.5, -0.5, -0.95, -0.02], atol=1e-14)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_rod_plane_gap_brute_force(seed):
    """The rod's closest point to a plane is an endpoint (the signed distance is linear along the
    axis); checked against a dense sampling of the axis, and the lever arm against P - c."""
    rng = np.random.default_rng(seed)
    n = 300
    c = rng.uniform(-1, 1, size=(n, 3))
    t = rng.normal(size=(n, 3)); t /= np.linalg.norm(t, axis=1, keepdims=True)
    L = rng.uniform(2, 4, n)
    w = rng.normal(size=3); w /= np.linalg.norm(w)
    walls = np.array([[*w, rng.uniform(-3, -1)]])
    ct = oracle.contacts_walls("rods", c, walls, direction=t, length=L, b=0.5, gap_abs=1e9)
    assert ct.nc == n  # huge threshold: every rod reported
    s = np.linspace(-0.5, 0.5, 2001)
    for l in range(n):
        i = ct.i[l]
        pts = c[i][None, :] + (s * L[i])[:, None] * t[i][None, :]
        d = pts @ w - walls[0, 3] - 0.5
        assert abs(ct.gap[l] - d.min()) < 1e-12
        P = c[i] + ct.lever[l, 0]
        assert abs(P @ w - walls[0, 3] - 0.5 - ct.gap[l]) < 1e-12
        np.testing.assert_array_equal(ct.lever[l, 1], 0.0)
    # parallel rod: the centre
    ctp = oracle.contacts_walls("rods", np.zeros((1, 3)), np.array([[0.0, 0.0, 1.0, -0.6]]),
                                direction=np.array([[1.0, 0.0, 0.0]]), length=np.array([3.0]), b=0.5, gap_abs=0.2)
    np.testing.assert_array_equal(ctp.lever[0, 0], 0.0)
    assert abs(ctp.gap[0] - 0.1) < 1e-15


def _rot(t, w, h):
    th = np.linalg.norm(w, axis=1, keepdims=True) * h
    k = w / np.maximum(np.linalg.norm(w, axis=1, keepdims=True), 1e-300)
    return t * np.cos(th) + np.cross(k, t) * np.sin(th) + k * np.sum(k * t, axis=1, keepdims=True) * (1 - np.cos(th))


def test_fd_gap_rate_rod_walls():
    """Eq. Dtranspose for wall columns: the gap rate under a rigid motion (U, Omega) of each rod
    equals D^T U -- pins n, the sign and the lever arm r_i = P - c_i of the wall columns."""
    p = make_problem("C4", n=1500, walls="box")
    ct = oracle.contacts_walls("rods", p.pos, p.walls, direction=p.direction, length=p.length, b=0.5,
                               gap_abs=0.1)
    assert ct.nc > 100
    rng = np.random.default_rng(9)
    U = rng.normal(size=(p.n, 6))
    h = 1e-6

    def gaps(center, direction):
        g = oracle.contacts_walls("rods", center, p.walls, direction=direction, length=p.length, b=0.5,
                                  gap_abs=1e9)
        key = {(int(i), int(j)): v for i, j, v in zip(g.i, g.j, g.gap)}
        return np.array([key[(int(i), int(j))] for i, j in zip(ct.i, ct.j)])

    gp = gaps(p.pos + h * U[:, :3], _rot(p.direction, U[:, 3:], h))
    gm = gaps(p.pos - h * U[:, :3], _rot(p.direction, U[:, 3:], -h))
    fd = (gp - gm) / (2 * h)
    an = oracle.apply_DT(p.n, ct, U)
    np.testing.assert_allclose(an, fd, rtol=0, atol=1e-6)


@pytest.mark.parametrize("gap,F", [(0.05, 200.0), (0.05, 10.0), (0.0, 37.0), (-0.3, 0.0)])
def test_single_sphere_on_floor_closed_form(gap, F):
    """One sphere above the floor, pushed down by F: a 1-constraint LCP with
    A = 1/(6 pi mu a) (the self mobility, no other body), q = gap/dt - F A,
    gamma = max(0, -q/A) = max(0, F - gap/(dt A)); touching (gap 0) gives gamma = F exactly."""
    a, mu, dt = 1.0, 1.0, 0.01
    pos = np.array([[3.0, -2.0, a + gap]])
    ct = oracle.contacts_walls("spheres", pos, FLOOR, radius=np.ones(1), gap_abs=0.0, gap_rel=0.1)
    assert ct.nc == 1
    sysm = oracle.System(oracle.ORC_SPHERES, 1, ct, mu=mu, pos=pos, radius=np.ones(1))
    Fext = np.zeros((1, 6)); Fext[0, 2] = -F
    q = sysm.lcp_q(dt, sysm.mobility(Fext))
    A = 1.0 / (6 * math.pi * mu * a)
    assert abs(q[0] - (ct.gap[0] / dt - F * A)) <= 1e-13 * (1 + abs(q[0]))
    r = sysm.bbpgd(q, tol=1e-12, max_iter=50)
    want = max(0.0, F - ct.gap[0] / (dt * A))
    assert abs(r["gamma"][0] - want) <= 1e-10 * (1 + want)
    if gap == 0.0:
        assert r["gamma"][0] == pytest.approx(F, rel=1e-14)
        # the sphere comes to rest on the floor: U_z = (F_c - F) A = 0
        assert abs(r["Uc"][0, 2] + sysm.mobility(Fext)[0, 2]) < 1e-12


@pytest.mark.parametrize("n,seed", [(12, 0), (16, 0), (16, 2)])
def test_floor_lcp_vs_enumeration(n, seed):
    """Small clusters with floor contacts: BBPGD (oracle) vs brute-force active-set enumeration
    of the dense LCP D^T M D (independent solver), all 2^m supports."""
    p = make_problem("C1", n=n, seed=seed, walls="floor")
    sysm = oracle.system_for(p)
    ct = sysm.ct
    m = ct.nc
    assert (ct.j >= p.n).sum() > 0 and m <= 14, m
    A = np.stack([sysm.mvop(e) for e in np.eye(m)], axis=1)
    q = sysm.lcp_q(p.dt, sysm.mobility(p.force))
    best = None
    for mask in range(1 << m):
        S = [k for k in range(m) if mask >> k & 1]
        g = np.zeros(m)
        if S:
            AS = A[np.ix_(S, S)]
            try:
                g[S] = np.linalg.solve(AS, -q[S])
            except np.linalg.LinAlgError:
                continue
        w = A @ g + q
        if g.min() >= -1e-9 and w.min() >= -1e-7 * (1 + np.abs(q).max()):
            best = g
            break
    assert best is not None
    r = sysm.bbpgd(q, tol=1e-10, max_iter=20000)
    np.testing.assert_allclose(r["gamma"], best, rtol=0, atol=1e-6 * (1 + np.abs(best).max()))


# ------------------------------------------------------------------ moving boundaries
def test_moving_floor_single_sphere_closed_form():
    """A boundary may move with a prescribed velocity; D is unchanged and the gap
    rate becomes n.(U_i - V_k), so q = gap/dt + D^T U_ext - n.V.  One sphere (a = mu = 1) at
    height z above a floor n = e_z moving with V, pushed down by F: A = 1/(6 pi), q = (z - 1)/dt
    - F/(6 pi) - V_z, gamma = max(0, -q/A) = max(0, F + 6 pi (V_z - (z - 1)/dt)).  Tangential
    floor velocity does not enter (n.V = 0)."""
    dt = 0.01
    walls = np.array([[0.0, 0.0, 1.0, 0.0]])
    for z, F, V in [(1.05, 0.0, 10.0), (1.05, 0.0, 3.0), (0.98, 1.0, -1.0), (1.0, 0.0, 0.0),
                    (1.02, 5.0, 0.5), (1.05, 2.0, -20.0)]:
        pos = np.array([[0.3, -0.2, z]])
        ct = oracle.contacts_walls("spheres", pos, walls, radius=np.ones(1), gap_abs=0.0, gap_rel=0.1)
        assert ct.nc == 1
        sysm = oracle.System(oracle.ORC_SPHERES, 1, ct, pos=pos, radius=np.ones(1))
        FT = np.zeros((1, 6))
        FT[0, 2] = -F
        U = sysm.mobility(FT)
        for vel, vz in (([0.0, 0.0, V], V), ([2.0, -1.5, V], V)):
            q = sysm.lcp_q_moving_walls(dt, U, [vel])
            assert q[0] == pytest.approx((z - 1.0) / dt - F / (6 * np.pi) - vz, rel=1e-14, abs=1e-12)
            r = sysm.bbpgd(q, tol=1e-10, max_iter=50)
            expect = max(0.0, F + 6 * np.pi * (vz - (z - 1.0) / dt))
            assert r["gamma"][0] == pytest.approx(expect, rel=1e-12, abs=1e-12)
        # static wall: the moving-wall q with V = 0 is the static q
        np.testing.assert_array_equal(sysm.lcp_q_moving_walls(dt, U, [[0.0, 0.0, 0.0]]), sysm.lcp_q(dt, U))


def test_moving_walls_only_shift_wall_rows_of_q():
    """Pair constraints are untouched by wall velocities; each wall row moves by -n_k.V_k."""
    p = make_problem("C2", n=600, walls="box")
    sysm = oracle.system_for(p)
    U = sysm.mobility(p.force)
    q0 = sysm.lcp_q(p.dt, U)
    rng = np.random.default_rng(4)
    V = rng.normal(size=(len(p.walls), 3))
    q1 = sysm.lcp_q_moving_walls(p.dt, U, V)
    ct = sysm.ct
    wall = ct.j >= p.n
    assert wall.sum() > 0
    np.testing.assert_array_equal(q1[~wall], q0[~wall])
    k = ct.j[wall] - p.n
    np.testing.assert_allclose(q1[wall], q0[wall] - np.einsum("lc,lc->l", ct.normal[wall], V[k]), rtol=0,
                               atol=1e-12 * np.abs(q0).max())
