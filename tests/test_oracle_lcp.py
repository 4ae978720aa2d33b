"""Pins for the oracle's LCP setup and BBPGD.

* closed form: two-sphere head-on LCP (tests/golden/headon_two_sphere.txt);
* touching spheres: gamma = F exactly, independent of the mobility;
* scalar / diagonal textbook LCPs; q >= 0 exits after 1 MVOP;
* brute-force active-set enumeration on random SPD LCPs and on real contact
  clusters (n_c <= 10);
* active-set polish (exact gamma* by a dense solve) on C1 and the a-priori
  error bound Eq. abserrcqp;
* MVOP accounting 2 + iterations.
The exact iteration count is "parity unpinned".
"""
import itertools
import os

import mpmath as mp
import numpy as np
import pytest

import oracle
from paper_1909_06623_b200.synthetic import make_problem

GOLD = os.path.join(os.path.dirname(__file__), "golden", "headon_two_sphere.txt")


def _headon_closed_form(r, F, dt=0.01):
    mp.mp.dps = 30
    r = mp.mpf(str(r))
    s = 1 / (6 * mp.pi)
    m = (1 / (8 * mp.pi * r)) * (2 - mp.mpf(4) / (3 * r ** 2)) if r >= 2 else s * (1 - 3 * r / 16)
    A = 2 * (s - m)
    gap = r - 2
    q = gap / dt - F * A
    return A, q, max(mp.mpf(0), -q / A)


def _headon_system(r, F, dt=0.01):
    pos = np.array([[0.0, 0, 0], [r, 0, 0]])
    ct = oracle.contacts_spheres(pos, np.ones(2), 0.0, 0.1)
    sysm = oracle.System(oracle.ORC_SPHERES, 2, ct, pos=pos, radius=np.ones(2))
    Fext = np.zeros((2, 6)); Fext[0, 0] = F; Fext[1, 0] = -F
    q = sysm.lcp_q(dt, sysm.mobility(Fext))
    return sysm, q


def test_headon_golden_table():
    rows = [l.split() for l in open(GOLD) if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r, F, A, q, gam in rows:
        r, F = float(r), float(F)
        A_cf, q_cf, g_cf = _headon_closed_form(r, F)
        assert float(q_cf) == pytest.approx(float(q), rel=1e-15, abs=1e-15)
        assert float(g_cf) == pytest.approx(float(gam), rel=1e-15, abs=1e-15)
        if A != "":
            assert float(A_cf) == pytest.approx(float(A), rel=1e-15)
        sysm, qo = _headon_system(r, F)
        assert qo[0] == pytest.approx(float(q_cf), rel=1e-13, abs=1e-13)
        assert sysm.mvop(np.array([1.0]))[0] == pytest.approx(float(A_cf), rel=1e-14)
        res = sysm.bbpgd(qo, tol=1e-8)
        assert res["gamma"][0] == pytest.approx(float(g_cf), rel=1e-12, abs=1e-12)
        # the scalar LCP converges in at most one GD step
        assert res["iters"] <= 1
        assert res["mvops"] == (1 if float(g_cf) == 0 else 3)


def test_touching_spheres_gamma_equals_force():
    for F in (0.5, 3.0, 17.0):
        sysm, q = _headon_system(2.0, F)
        assert sysm.bbpgd(q, tol=1e-10)["gamma"][0] == pytest.approx(F, rel=1e-12)


def test_scalar_and_diagonal_textbook_cases():
    r = oracle.bbpgd_dense(np.array([[2.0]]), np.array([-4.0]))
    assert r["gamma"][0] == pytest.approx(2.0, rel=1e-15) and r["residual"] == 0.0
    r = oracle.bbpgd_dense(np.diag([2.0, 3.0]), np.array([-2.0, 6.0]))
    np.testing.assert_allclose(r["gamma"], [1.0, 0.0], atol=1e-12)
    # q >= 0 with gamma_0 = 0: solved after 1 MVOP, 0 GD steps
    r = oracle.bbpgd_dense(np.diag([2.0, 3.0]), np.array([0.5, 6.0]))
    assert r["mvops"] == 1 and r["iters"] == 0 and np.all(r["gamma"] == 0)
    # min-map residual examples
    assert oracle.minmap_residual(np.array([1.0, 2.0]), np.array([3.0, 0.5])) == pytest.approx(np.sqrt(1.25))
    assert oracle.minmap_residual(np.zeros(3), np.array([1.0, 0.0, 2.0])) == 0.0


def _enumerate_lcp(M, q):
    """All supports S: gamma_S = -M_SS^{-1} q_S >= 0, (M gamma + q) >= 0 off S."""
    n = len(q)
    sols = []
    for k in range(n + 1):
        for S in itertools.combinations(range(n), k):
            S = list(S)
            g = np.zeros(n)
            if S:
                try:
                    g[S] = np.linalg.solve(M[np.ix_(S, S)], -q[S])
                except np.linalg.LinAlgError:
                    continue
            w = M @ g + q
            tol = 1e-10 * (1 + np.abs(q).max() + np.abs(M).max() * (1 + np.abs(g).max()))
            if np.all(g >= -tol) and np.all(w >= -tol):
                sols.append(np.maximum(g, 0))
    return sols


def test_random_spd_vs_enumeration():
    rng = np.random.default_rng(2024)
    for trial in range(200):
        n = int(rng.integers(1, 11))
        A = rng.normal(size=(n, n))
        M = A @ A.T + 0.1 * np.eye(n)
        q = rng.normal(size=n) * 3
        sols = _enumerate_lcp(M, q)
        assert sols
        ref = sols[0]
        for s in sols[1:]:
            np.testing.assert_allclose(s, ref, atol=1e-8)  # unique for SPD M
        r = oracle.bbpgd_dense(M, q, tol=1e-10, max_iter=20000)
        assert r["status"] == 0
        assert np.abs(r["gamma"] - ref).max() <= 1e-7, (trial, r["gamma"], ref)
        assert r["mvops"] == r["iters"] + 2 or r["mvops"] == 1
        # BB2 and alternating steps reach the same solution
        for mode in (1, 2):
            r2 = oracle.bbpgd_dense(M, q, tol=1e-10, max_iter=20000, bb_mode=mode)
            assert np.abs(r2["gamma"] - ref).max() <= 1e-7


def _dense_lcp(sysm):
    nc = sysm.ct.nc
    return np.stack([sysm.mvop(e) for e in np.eye(nc)], axis=1)


def test_contact_clusters_vs_enumeration():
    """Small real clusters (3-7 spheres, n_c <= 10): oracle BBPGD == enumeration."""
    rng = np.random.default_rng(77)
    done = 0
    while done < 25:
        k = int(rng.integers(3, 8))
        pos = rng.uniform(0, 2.2 * k ** (1 / 3), size=(k, 3))
        radius = rng.uniform(0.5, 1.0, k)
        try:
            ct = oracle.contacts_spheres(pos, radius, 0.0, 0.1)
        except oracle.OracleError:
            continue
        if not 1 <= ct.nc <= 10:
            continue
        sysm = oracle.System(oracle.ORC_SPHERES, k, ct, pos=pos, radius=radius)
        F = np.zeros((k, 6)); F[:, :3] = rng.normal(size=(k, 3))
        q = sysm.lcp_q(0.01, sysm.mobility(F))
        M = _dense_lcp(sysm)
        np.testing.assert_allclose(M, M.T, atol=1e-14 * np.abs(M).max())
        sols = _enumerate_lcp(M, q)
        assert sols
        r = sysm.bbpgd(q, tol=1e-10, max_iter=20000)
        assert r["status"] == 0
        # gamma* is unique a.s. even when D is rank-deficient (reading A19); D gamma always is
        Fr = oracle.apply_D(k, ct, r["gamma"])
        for s in sols:
            np.testing.assert_allclose(oracle.apply_D(k, ct, s), Fr, atol=1e-7 * (1 + np.abs(Fr).max()))
        assert np.abs(r["gamma"] - sols[0]).max() <= 1e-6 * (1 + np.abs(sols[0]).max())
        done += 1


def test_c1_active_set_polish_and_error_bound():
    p = make_problem("C1")
    res = oracle.solve_problem(p)
    sysm, q, gam = res["system"], res["q"], res["gamma"]
    assert res["status"] == 0 and res["residual"] < 1e-8
    assert res["mvops"] == res["iters"] + 2
    M = _dense_lcp(sysm)
    S = np.flatnonzero(gam > 0)
    ex = np.zeros_like(gam)
    ex[S] = np.linalg.lstsq(M[np.ix_(S, S)], -q[S], rcond=None)[0]
    w = M @ ex + q
    scale = np.abs(q).max()
    assert ex[S].min() >= 0 and np.delete(w, S).min() >= -1e-9 * scale
    rel = np.linalg.norm(gam - ex) / np.linalg.norm(ex)
    assert rel < 1e-9, rel
    # the returned g equals M gamma + q
    np.testing.assert_allclose(res["g"], M @ gam + q, rtol=0, atol=1e-9 * scale)
    # Newton's third law on F_c and the complementarity certificate
    assert np.abs(res["Fc"][:, :3].sum(0)).max() < 1e-9 * np.abs(res["Fc"]).sum()
    assert oracle.minmap_residual(gam, M @ gam + q) < 1e-8


def test_error_bound_abserrcqp():
    """||gamma - gamma*|| <= (||M|| + 1)/lambda_min * phi on an SPD case."""
    rng = np.random.default_rng(5)
    A = rng.normal(size=(8, 8)); M = A @ A.T + np.eye(8); q = rng.normal(size=8) * 4
    ref = _enumerate_lcp(M, q)[0]
    lam = np.linalg.eigvalsh(M)
    for tol in (1e-2, 1e-4, 1e-6):
        r = oracle.bbpgd_dense(M, q, tol=tol)
        bound = (lam.max() + 1) / lam.min() * r["residual"]
        assert np.linalg.norm(r["gamma"] - ref) <= bound


def test_fixed_iteration_mode_runs_exactly_j_max():
    p = make_problem("C1")
    sysm = oracle.system_for(p)
    q = sysm.lcp_q(p.dt, sysm.mobility(p.force))
    r = sysm.bbpgd(q, tol=1e-8, max_iter=7, fixed_iters=1)
    assert r["iters"] == 7 and r["mvops"] == 9 and r["status"] == 0
    r2 = sysm.bbpgd(q, tol=1e-8, max_iter=7)
    np.testing.assert_array_equal(r["gamma"], r2["gamma"])  # same 7 steps
    assert r2["status"] == 1  # not converged at j_max (reading A7)


def test_torques_are_inert_for_spheres():
    """C3's rotor torques cannot change gamma (reading A18)."""
    p = make_problem("C3", n=400)
    r1 = oracle.solve_problem(p, max_iter=30, fixed_iters=1)
    p.force[:, 3:] = 0.0
    r2 = oracle.solve_problem(p, max_iter=30, fixed_iters=1)
    np.testing.assert_array_equal(r1["gamma"], r2["gamma"])


# ---------------------------------------------------------------- reading A5 (BB breakdown)
def test_bb_breakdown_step_in_null_space_closed_form():
    """Reading A5 pinned by a closed form.  M = [[1,-1,0],[-1,1,0],[0,0,1]] is SPSD with null
    vector z = (1,1,0); q = (-1,-1,1).  Step 6: alpha_0 = |q|^2 / q^T M q = 3/1 = 3.  Step 8-9:
    gamma_1 = max(0, -3q) = (3,3,0) = 3z, so s = 3z lies in null(M): y = M s = 0 and s^T y = 0 --
    a BB breakdown (BB1 3/0 and BB2 0/0 are both undefined).  Rule A5 keeps alpha = 3, so
    g_j = q for every j and gamma_j = 3j (1,1,0) exactly (integers), phi_j = |(-1,-1,0)| = sqrt 2
    (the LCP is infeasible: q^T z < 0), and every iteration, the last included (Steps 14-15 are in
    the loop body of Alg. 1), counts one breakdown.  A slip (accepting the undefined
    step, not counting it, or skipping the rule) changes gamma, the status or the count."""
    M = np.array([[1.0, -1.0, 0.0], [-1.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    q = np.array([-1.0, -1.0, 1.0])
    for bb_mode in (0, 1, 2):
        for J in (1, 2, 7):
            r = oracle.bbpgd_dense(M, q, tol=1e-8, max_iter=J, bb_mode=bb_mode)
            assert r["status"] == 1 and r["converged"] == 0
            np.testing.assert_array_equal(r["gamma"], [3.0 * J, 3.0 * J, 0.0])
            np.testing.assert_array_equal(r["g"], q)
            assert r["bb_breakdowns"] == J and r["iters"] == J and r["mvops"] == J + 2
            assert r["residual"] == pytest.approx(np.sqrt(2.0), rel=1e-15)


def test_bb_breakdown_negative_curvature_keeps_alpha():
    """Reading A5 on s^T y < 0 (a plausible slip would accept the negative BB1 step).
    M = diag(1, -2), q = (3, -1) (M indefinite: a unit pin of the rule, not a physical system).
    alpha_0 = |q|^2 / q^T M q = 10/7; gamma_1 = max(0, -alpha_0 q) = (0, 10/7); s = gamma_1,
    y = M s = (0, -20/7), s^T y = -200/49 < 0: breakdown, alpha stays 10/7; g_1 = (3, -27/7);
    gamma_2 = max(0, gamma_1 - (10/7) g_1) = (0, 340/49); again s^T y < 0: 2 breakdowns."""
    M = np.diag([1.0, -2.0])
    q = np.array([3.0, -1.0])
    r = oracle.bbpgd_dense(M, q, tol=1e-12, max_iter=2)
    assert r["bb_breakdowns"] == 2 and r["iters"] == 2
    np.testing.assert_allclose(r["gamma"], [0.0, 340.0 / 49.0], rtol=1e-14, atol=0)
    r1 = oracle.bbpgd_dense(M, q, tol=1e-12, max_iter=1)
    np.testing.assert_allclose(r1["gamma"], [0.0, 10.0 / 7.0], rtol=1e-15, atol=0)
    np.testing.assert_allclose(r1["g"], [3.0, -27.0 / 7.0], rtol=1e-15, atol=0)
    assert r1["bb_breakdowns"] == 1
