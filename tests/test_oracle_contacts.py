"""Pins for the oracle's contact detection (Sec. 3.2).

The oracle's sphere contacts are pinned by (1) hand examples, (2) an
independent library enumeration (scipy cKDTree) and (3) agreement of the
oracle's two independent searches (brute force and grid).  Rod contacts are
pinned by brute-force minimisation of the segment distance, special cases
with known distances, and the prefilter against the unfiltered all-pairs scan.
"""
import math

import numpy as np
import pytest
from scipy.optimize import minimize
from scipy.spatial import cKDTree

import oracle
from paper_1909_06623_b200.synthetic import make_problem


def _pairs(ct):
    return list(zip(ct.i.tolist(), ct.j.tolist()))


def test_hand_examples_threshold_A1():
    # unit spheres at distance 2.05: gap 0.05 < 0.1a -> contact
    ct = oracle.contacts_spheres(np.array([[0., 0, 0], [2.05, 0, 0]]), np.ones(2), 0.0, 0.1)
    assert _pairs(ct) == [(0, 1)]
    assert ct.gap[0] == pytest.approx(0.05, abs=1e-15)
    # normal from j to i (reading A13): i=0 at x=0, j=1 at x=2.05 -> (-1,0,0)
    np.testing.assert_array_equal(ct.normal[0], [-1.0, 0.0, 0.0])
    # distance 2.5: gap 0.5 >= 0.1 -> no contact under BASELINE's threshold
    ct = oracle.contacts_spheres(np.array([[0., 0, 0], [2.5, 0, 0]]), np.ones(2), 0.0, 0.1)
    assert ct.nc == 0
    # ... but a contact under the paper's 30%-of-summed-radii rule: delta = 0.6
    ct = oracle.contacts_spheres(np.array([[0., 0, 0], [2.5, 0, 0]]), np.ones(2), 0.6, 0.0)
    assert _pairs(ct) == [(0, 1)] and ct.gap[0] == 0.5
    # three collinear spheres: only neighbours
    ct = oracle.contacts_spheres(np.array([[0., 0, 0], [2.05, 0, 0], [4.1, 0, 0]]), np.ones(3), 0.0, 0.1)
    assert _pairs(ct) == [(0, 1), (1, 2)]
    # overlap allowed (reading A14): a=1 and a=2 at distance 2.5 -> gap -0.5
    ct = oracle.contacts_spheres(np.array([[0., 0, 0], [2.5, 0, 0]]), np.array([1.0, 2.0]), 0.0, 0.1)
    assert ct.gap[0] == -0.5


def test_empty_and_single():
    ct = oracle.contacts_spheres(np.zeros((0, 3)), np.zeros(0), 0.0, 0.1, method="brute")
    assert ct.nc == 0
    ct = oracle.contacts_spheres(np.zeros((1, 3)), np.ones(1), 0.0, 0.1)
    assert ct.nc == 0


def test_coincident_centres_are_an_error():
    with pytest.raises(oracle.OracleError):
        oracle.contacts_spheres(np.zeros((2, 3)), np.ones(2), 0.0, 0.1, method="brute")
    with pytest.raises(oracle.OracleError):
        oracle.contacts_spheres(np.zeros((2, 3)), np.ones(2), 0.0, 0.1, method="grid")


def _kdtree_pairs(pos, radius, gap_abs, gap_rel):
    rmax = 2 * radius.max() + gap_abs + gap_rel * radius.max()
    cand = cKDTree(pos).query_pairs(rmax * 1.0001, output_type="ndarray")
    out = set()
    for i, j in cand:
        i, j = min(i, j), max(i, j)
        d = math.dist(pos[i], pos[j]) - radius[i] - radius[j]
        thr = gap_abs + gap_rel * min(radius[i], radius[j])
        if d < thr - 1e-12:
            out.add((i, j))
        elif d < thr + 1e-12:
            out.add((i, j, "edge"))
    return out


@pytest.mark.parametrize("name,n", [("C1", 512), ("C2", 3000), ("C3", 4000), ("C5", 4000)])
def test_sphere_sets_vs_kdtree_and_brute(name, n):
    p = make_problem(name, n=n)
    g = oracle.contacts_spheres(p.pos, p.radius, p.gap_abs, p.gap_rel, method="grid")
    b = oracle.contacts_spheres(p.pos, p.radius, p.gap_abs, p.gap_rel, method="brute")
    # two independent searches in the oracle agree bit for bit
    np.testing.assert_array_equal(g.i, b.i)
    np.testing.assert_array_equal(g.j, b.j)
    np.testing.assert_array_equal(g.gap, b.gap)
    np.testing.assert_array_equal(g.normal, b.normal)
    # sorted by (i, j), i < j
    assert np.all(g.i < g.j)
    key = g.i.astype(np.int64) * n + g.j
    assert np.all(np.diff(key) > 0)
    # the set agrees with a library enumeration (pairs within 1e-12 of the threshold may go either way)
    ref = _kdtree_pairs(p.pos, p.radius, p.gap_abs, p.gap_rel)
    sure = {x for x in ref if len(x) == 2}
    edge = {(x[0], x[1]) for x in ref if len(x) == 3}
    got = set(_pairs(g))
    assert sure <= got and got <= sure | edge
    # normals are unit and point from j to i
    np.testing.assert_allclose(np.linalg.norm(g.normal, axis=1), 1.0, atol=1e-15)
    d = p.pos[g.i] - p.pos[g.j]
    assert np.all(np.einsum("ij,ij->i", d, g.normal) > 0)
    # overlapped fraction is the paper-shaped 80-90%
    if g.nc > 50:
        assert 0.7 < np.mean(g.gap < 0) < 0.95


# ------------------------------------------------------------------ rods
def _brute_segdist(c1, t1, L1, c2, t2, L2):
    p1 = c1 - 0.5 * L1 * t1
    p2 = c2 - 0.5 * L2 * t2
    d1, d2 = L1 * t1, L2 * t2
    f = lambda x: float(np.sum((p1 + x[0] * d1 - p2 - x[1] * d2) ** 2))
    s = np.linspace(0, 1, 201)
    S, T = np.meshgrid(s, s, indexing="ij")
    P = p1[None, None] + S[..., None] * d1 - p2[None, None] - T[..., None] * d2
    D = np.sum(P ** 2, axis=-1)
    k = np.unravel_index(np.argmin(D), D.shape)
    r = minimize(f, [S[k], T[k]], bounds=[(0, 1), (0, 1)], method="L-BFGS-B",
                 options={"ftol": 1e-20, "gtol": 1e-14})
    return math.sqrt(min(r.fun, D[k]))


def test_segment_closest_vs_brute_force():
    rng = np.random.default_rng(11)
    for _ in range(200):
        c1, c2 = rng.uniform(-2, 2, 3), rng.uniform(-2, 2, 3)
        t1 = rng.normal(size=3); t1 /= np.linalg.norm(t1)
        t2 = rng.normal(size=3); t2 /= np.linalg.norm(t2)
        L1, L2 = rng.uniform(2, 4, 2)
        P1, P2 = oracle.segment_closest(c1, t1, L1, c2, t2, L2)
        d = np.linalg.norm(P1 - P2)
        ref = _brute_segdist(c1, t1, L1, c2, t2, L2)
        assert d <= ref + 1e-12 and d >= ref - 1e-7
        # closest points lie on the segments
        for P, c, t, L in ((P1, c1, t1, L1), (P2, c2, t2, L2)):
            s = np.dot(P - c, t)
            assert abs(s) <= 0.5 * L + 1e-12
            np.testing.assert_allclose(P, c + s * t, atol=1e-12)


def test_segment_special_cases():
    ex, ey, ez = np.eye(3)
    # parallel side by side at separation 1.5: distance 1.5, s = 0 rule (reading A15)
    P1, P2 = oracle.segment_closest(np.zeros(3), ex, 2.0, 1.5 * ey, ex, 2.0)
    assert np.linalg.norm(P1 - P2) == pytest.approx(1.5, abs=1e-15)
    # crossing perpendicular axes 1 apart in z: distance 1 at the centres
    P1, P2 = oracle.segment_closest(np.zeros(3), ex, 2.0, ez, ey, 2.0)
    np.testing.assert_allclose(P1, [0, 0, 0], atol=1e-15)
    np.testing.assert_allclose(P2, [0, 0, 1], atol=1e-15)
    # collinear end to end: gap between the ends
    P1, P2 = oracle.segment_closest(np.zeros(3), ex, 2.0, 3.5 * ex, ex, 2.0)
    assert np.linalg.norm(P1 - P2) == pytest.approx(1.5, abs=1e-15)
    # T configuration: the end of one against the middle of the other
    P1, P2 = oracle.segment_closest(np.zeros(3), ex, 2.0, 2.0 * ey, ey, 2.0)
    assert np.linalg.norm(P1 - P2) == pytest.approx(1.0, abs=1e-15)


def test_rod_crossing_axes_normal():
    # axes intersect: dist = 0, normal = +-(t_i x t_j) oriented by the centres (reading A15)
    center = np.array([[0.0, 0, 0.0], [0, 0, 0.0]])
    center[0, 2] = 0.0
    center[1] = [0.5, -0.5, 0.0]
    d = np.array([[1.0, 0, 0], [0, 1.0, 0]])
    ct = oracle.contacts_rods(center, d, np.array([2.0, 2.0]), 0.5, 0.1)
    assert ct.nc == 1 and ct.gap[0] == -1.0
    assert abs(abs(ct.normal[0, 2]) - 1.0) < 1e-15


@pytest.mark.parametrize("n", [500, 2000])
def test_rod_prefilter_is_exact(n):
    p = make_problem("C4", n=n)
    a = oracle.contacts_rods(p.pos, p.direction, p.length, 0.5, 0.1, brute=False)
    b = oracle.contacts_rods(p.pos, p.direction, p.length, 0.5, 0.1, brute=True)
    np.testing.assert_array_equal(a.i, b.i)
    np.testing.assert_array_equal(a.j, b.j)
    np.testing.assert_array_equal(a.gap, b.gap)
    assert a.nc > n // 2
    # every emitted gap agrees with the brute-force segment distance
    for l in range(0, a.nc, max(1, a.nc // 40)):
        i, j = a.i[l], a.j[l]
        ref = _brute_segdist(p.pos[i], p.direction[i], p.length[i], p.pos[j], p.direction[j], p.length[j])
        assert a.gap[l] == pytest.approx(ref - 1.0, abs=1e-7)
        # lever arms are the closest points relative to the centres, perpendicular offsets along t
        ri, rj = a.lever[l]
        assert abs(np.linalg.norm(np.cross(ri, p.direction[i]))) < 1e-12
        assert abs(np.linalg.norm(np.cross(rj, p.direction[j]))) < 1e-12
