"""NEXT row f4(i): the fast O(N) RPY summation (csrc/fmm.cu) against the oracle's direct apply.

The fast summation approximates the BASELINE RPY operator; the parity bar is a stated relative L2
error per interpolation order (from the measured errors in
profiles/r02/fmm_scaling.jsonl, with margin), measured against the oracle's long-double direct sum
-- nothing of the GPU direct path enters the reference.  Near field (27 leaves, every overlapping
pair) is exact, so two spheres in one leaf must match the direct formula to rounding."""
import numpy as np
import pytest
import torch

import oracle
from paper_1909_06623_b200 import Context, ScError
from paper_1909_06623_b200.synthetic import make_problem

pytestmark = pytest.mark.gpu

TOL = {4: 2e-3, 6: 6e-5, 8: 3e-6}  # stated rel. L2 bars of the apply


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    c = Context(0)
    yield c
    c.close()


def _cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def _relL2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("order", [4, 6, 8])
@pytest.mark.parametrize("n,leaf_level", [(6000, 0), (20000, 0), (20000, 3)])
def test_fmm_apply_vs_oracle(ctx, order, n, leaf_level):
    p = make_problem("C5", n=n)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    ctx.set_mobility_model("rpy_fmm")
    ctx.set_fmm_params(order, leaf_level)
    rng = np.random.default_rng(1)
    FT = rng.normal(size=(p.n, 6))
    U = ctx.mobility_apply(_cuda(FT)).cpu().numpy()
    info = ctx.fmm_info()
    ctx.set_mobility_model("rpy")
    Uo = oracle.rpy_apply(p.pos, p.radius, p.mu, FT)
    assert info["ready"] == 1 and info["leaf_level"] >= 2 and (leaf_level == 0 or info["leaf_level"] == leaf_level)
    assert info["compression_mode"] == 2 and info["compressed"] == 0  # (auto: direct M2L below 2^15)
    err = _relL2(U[:, :3], Uo[:, :3])
    assert err <= TOL[order], (order, n, info, err)
    np.testing.assert_allclose(U[:, 3:], Uo[:, 3:], rtol=1e-13, atol=0)  # self rotation (exact)


def test_fmm_error_decreases_with_order_and_is_deterministic(ctx):
    p = make_problem("C5", n=12000)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    FT = np.random.default_rng(2).normal(size=(p.n, 6))
    Uo = oracle.rpy_apply(p.pos, p.radius, p.mu, FT)[:, :3]
    ctx.set_mobility_model("rpy_fmm")
    errs = []
    for order in (4, 6, 8):
        ctx.set_fmm_params(order, 3)
        U1 = ctx.mobility_apply(_cuda(FT))
        U2 = ctx.mobility_apply(_cuda(FT))
        assert torch.equal(U1, U2)  # fixed summation orders: bitwise repeatable
        errs.append(_relL2(U1.cpu().numpy()[:, :3], Uo))
    ctx.set_mobility_model("rpy")
    assert errs[0] > errs[1] > errs[2], errs


def test_fmm_near_field_exact_and_far_pair(ctx):
    """Overlapping and touching pairs are in the near field (exact formula); a pair far apart goes
    through P2M -> M2L -> L2P and must match the far branch to the interpolation accuracy."""
    rng = np.random.default_rng(3)
    pos = np.concatenate([np.array([[0.0, 0.0, 0.0], [1.5, 0.0, 0.0], [2.0, 2.0, 0.0]]),
                          rng.uniform(0, 60, size=(3000, 3)) + np.array([10.0, 0.0, 0.0])])
    pos = pos[np.r_[0:3, 3 + np.flatnonzero(np.min(np.linalg.norm(pos[3:, None, :] - pos[None, :3, :], axis=2), 1) > 2.5)]]
    FT = np.zeros((len(pos), 6))
    FT[:3, :3] = rng.normal(size=(3, 3))
    FT[-1, :3] = [1.0, -2.0, 0.5]
    ctx.build_contacts_spheres(_cuda(pos), None, 0.0, 0.1)
    ctx.set_mobility_model("rpy_fmm")
    ctx.set_fmm_params(8, 0)
    U = ctx.mobility_apply(_cuda(FT)).cpu().numpy()
    ctx.set_mobility_model("rpy")
    Uo = oracle.rpy_apply(pos, np.ones(len(pos)), 1.0, FT)
    np.testing.assert_allclose(U[:3, :3], Uo[:3, :3], rtol=1e-6, atol=1e-8 * np.abs(Uo).max())
    assert _relL2(U[:, :3], Uo[:, :3]) <= TOL[8]


def test_fmm_converged_solve_certified_by_oracle(ctx):
    """BBPGD with the fast summation as the mobility (order 8): the converged gamma satisfies the
    oracle's (direct) LCP to the accuracy of the operator -- phi(gamma, g_oracle) small next to
    |q| -- and is close to the direct solve's gamma."""
    p = make_problem("C5", n=20000, fixed_iters=0)
    t = _cuda
    rs = {}
    for model in ("rpy", "rpy_fmm"):
        ctx.set_mobility_model(model)
        ctx.set_fmm_params(8, 0)
        ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
        ctx.assemble_D()
        ctx.lcp_q(p.dt, ctx.mobility_apply(t(p.force), mu=p.mu))
        rs[model] = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    ctx.set_mobility_model("rpy")
    rf, rd = rs["rpy_fmm"], rs["rpy"]
    assert rf["status"] == 0 and rf["residual"] < p.tol
    gf, gd = rf["gamma"].cpu().numpy(), rd["gamma"].cpu().numpy()
    assert _relL2(gf, gd) <= 1e-3
    sysm = oracle.system_for(p)
    F = oracle.apply_D(p.n, sysm.ct, gf) + p.force
    go = sysm.lcp_q(p.dt, sysm.mobility(F))
    q = sysm.lcp_q(p.dt, sysm.mobility(p.force))
    phi = float(np.linalg.norm(np.minimum(gf, go)))
    assert phi <= 1e-5 * float(np.linalg.norm(q)), phi


def test_fmm_rejects_bad_params(ctx):
    with pytest.raises(ScError):
        ctx.set_fmm_params(5, 0)
    with pytest.raises(ScError):
        ctx.set_fmm_params(6, 11)


@pytest.mark.parametrize("order", [4, 6, 8])
@pytest.mark.parametrize("n,leaf_level", [(6000, 0), (8192, 3)])
def test_fmm_polydisperse_apply_vs_oracle(ctx, order, n, leaf_level):
    """C2 recipe (radii U[0.5, 1], phi = 0.4): the radius-split far field (m2l_poly_kernel, 9 node
    components) and the exact near field with abar = (a_i + a_j)/2 against the oracle's direct
    polydisperse sum, at the same stated bars as the monodisperse apply."""
    p = make_problem("C2", n=n)
    assert p.radius.min() < 0.6 and p.radius.max() > 0.9
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    ctx.set_mobility_model("rpy_fmm")
    ctx.set_fmm_params(order, leaf_level)
    FT = np.random.default_rng(11).normal(size=(p.n, 6))
    U = ctx.mobility_apply(_cuda(FT), mu=p.mu).cpu().numpy()
    U2 = ctx.mobility_apply(_cuda(FT), mu=p.mu).cpu().numpy()
    info = ctx.fmm_info()
    ctx.set_mobility_model("rpy")
    Uo = oracle.rpy_apply(p.pos, p.radius, p.mu, FT)
    assert info["ready"] == 1 and (leaf_level == 0 or info["leaf_level"] == leaf_level)
    np.testing.assert_array_equal(U, U2)
    err = _relL2(U[:, :3], Uo[:, :3])
    assert err <= TOL[order], (order, n, info, err)
    np.testing.assert_allclose(U[:, 3:], Uo[:, 3:], rtol=1e-13, atol=0)


def test_fmm_polydisperse_far_field_needs_all_three_fields(ctx):
    """A pair of very different radii far apart (through P2M -> M2L -> L2P only): the far branch
    with abar = (a_i + a_j)/2 is reproduced, and it differs from the far branch with either radius
    alone by far more than the interpolation error -- a dropped L_B or L_C field fails."""
    rng = np.random.default_rng(4)
    bulk = rng.uniform(0, 40, size=(2500, 3)) + np.array([12.0, 0.0, 0.0])
    pos = np.concatenate([np.array([[0.0, 0.0, 0.0], [20.0, 10.0, 10.0]]), bulk])
    keep = np.min(np.linalg.norm(pos[2:, None, :] - pos[None, :2, :], axis=2), 1) > 6.0
    pos = np.concatenate([pos[:2], pos[2:][keep]])
    radius = np.full(len(pos), 0.5)
    radius[0], radius[1] = 3.0, 0.25
    FT = np.zeros((len(pos), 6))
    FT[0, :3] = [0.3, -1.0, 2.0]
    FT[1, :3] = [1.0, 0.5, -0.7]
    ctx.build_contacts_spheres(_cuda(pos), _cuda(radius), 0.0, 0.1)
    ctx.set_mobility_model("rpy_fmm")
    ctx.set_fmm_params(8, 0)
    U = ctx.mobility_apply(_cuda(FT)).cpu().numpy()
    ctx.set_mobility_model("rpy")
    Uo = oracle.rpy_apply(pos, radius, 1.0, FT)
    cross = Uo[1, :3] - FT[1, :3] / (6 * np.pi * 0.25)  # the far contribution of body 0 at body 1
    for a_wrong in (3.0, 0.25):
        rw = radius.copy()
        rw[:2] = a_wrong
        Uw = oracle.rpy_apply(pos, rw, 1.0, FT)
        crossw = Uw[1, :3] - FT[1, :3] / (6 * np.pi * a_wrong)
        assert np.linalg.norm(crossw - cross) > 2e-3 * np.linalg.norm(cross)
    got = U[1, :3] - FT[1, :3] / (6 * np.pi * 0.25)
    assert np.linalg.norm(got - cross) <= 1e-4 * np.linalg.norm(cross)
    assert _relL2(U[:, :3], Uo[:, :3]) <= TOL[8]


def test_fmm_polydisperse_converged_solve_certified_by_oracle(ctx):
    """Full-size C2 (8192 polydisperse spheres, volume fraction 0.4) solved with the fast summation
    (order 8) and with the direct kernel: the FMM gamma lies within 1e-3 of the direct one and the
    oracle's direct polydisperse LCP certifies it to phi(gamma, g_oracle) <= 5e-5 |q| (measured
    1.3e-5 |q|: the denser C2 packing amplifies the operator error more than C5's 1e-5 bar)."""
    p = make_problem("C2", fixed_iters=0)
    t = _cuda
    rs = {}
    for model in ("rpy", "rpy_fmm"):
        ctx.set_mobility_model(model)
        ctx.set_fmm_params(8, 0)
        ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
        ctx.assemble_D()
        ctx.lcp_q(p.dt, ctx.mobility_apply(t(p.force), mu=p.mu))
        rs[model] = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    ctx.set_mobility_model("rpy")
    r = rs["rpy_fmm"]
    assert r["status"] == 0 and r["residual"] < p.tol
    g = r["gamma"].cpu().numpy()
    assert _relL2(g, rs["rpy"]["gamma"].cpu().numpy()) <= 1e-3
    sysm = oracle.system_for(p)
    F = oracle.apply_D(p.n, sysm.ct, g) + p.force
    go = sysm.lcp_q(p.dt, sysm.mobility(F))
    q = sysm.lcp_q(p.dt, sysm.mobility(p.force))
    phi = float(np.linalg.norm(np.minimum(g, go)))
    assert phi <= 5e-5 * float(np.linalg.norm(q)), phi


@pytest.mark.parametrize("n", [1, 2, 5, 40])
def test_fmm_tiny_problems_exact_near_field(ctx, n):
    """Few bodies in a small cluster: the root cube is at least 4 leaves of side 2a per dimension,
    every pair that can overlap is in the near field; the result matches the oracle."""
    rng = np.random.default_rng(n)
    pos = rng.uniform(0, 2.0 * max(1.0, n ** (1 / 3)), size=(n, 3))
    if n == 2:
        pos = np.array([[0.0, 0.0, 0.0], [1.2, 0.3, 0.0]])  # overlapping
    FT = rng.normal(size=(n, 6))
    ctx.build_contacts_spheres(_cuda(pos), None, 0.0, 0.1)
    ctx.set_mobility_model("rpy_fmm")
    ctx.set_fmm_params(6, 0)
    U = ctx.mobility_apply(_cuda(FT)).cpu().numpy()
    ctx.set_mobility_model("rpy")
    Uo = oracle.rpy_apply(pos, np.ones(n), 1.0, FT)
    assert _relL2(U, Uo) <= TOL[6]


def test_fmm_two_contexts_different_orders():
    """Two contexts with different orders interleaved in one process: the interpolation tables of
    every order live in constant memory side by side, so neither context disturbs the other."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    p = make_problem("C5", n=15000)
    FT = np.random.default_rng(9).normal(size=(p.n, 6))
    ref = {}
    for order in (4, 8):
        c = Context(0)
        c.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
        c.set_mobility_model("rpy_fmm")
        c.set_fmm_params(order, 0)
        ref[order] = c.mobility_apply(_cuda(FT)).clone()
        c.close()
    a, b = Context(0), Context(0)
    for c, order in ((a, 4), (b, 8)):
        c.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
        c.set_mobility_model("rpy_fmm")
        c.set_fmm_params(order, 0)
    for _ in range(2):
        ua = a.mobility_apply(_cuda(FT))
        ub = b.mobility_apply(_cuda(FT))
        assert torch.equal(ua, ref[4]) and torch.equal(ub, ref[8])
    a.close()
    b.close()


# ------------------------------------------------ compressed M2L (sc_set_fmm_compression)
@pytest.mark.parametrize("order", [4, 6, 8])
@pytest.mark.parametrize("n,leaf_level", [(20000, 0), (40000, 3)])
def test_fmm_compressed_m2l_vs_oracle(ctx, order, n, leaf_level):
    """The compressed M2L (per-level orthonormal basis of the 316 M2L operators, rank kept at 3% of
    the order's bar) meets the same stated bars against the oracle's direct sum, and repeated
    applies are bitwise equal (fixed-order batched GEMMs)."""
    p = make_problem("C5", n=n)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    ctx.set_mobility_model("rpy_fmm")
    ctx.set_fmm_params(order, leaf_level)
    ctx.set_fmm_compression(1)
    try:
        FT = np.random.default_rng(21).normal(size=(p.n, 6))
        U = ctx.mobility_apply(_cuda(FT))
        U2 = ctx.mobility_apply(_cuda(FT))
        info = ctx.fmm_info()
    finally:
        ctx.set_fmm_compression("auto")
        ctx.set_mobility_model("rpy")
    assert info["compression_mode"] == 1 and info["compressed"] == 1
    assert 0 < info["rank"] < 3 * order ** 3 and info["rank_level"] == info["leaf_level"]
    assert torch.equal(U, U2)
    Uo = oracle.rpy_apply(p.pos, p.radius, p.mu, FT)
    err = _relL2(U.cpu().numpy()[:, :3], Uo[:, :3])
    assert err <= TOL[order], (order, n, err)


def test_fmm_compressed_converged_solve_certified_by_oracle(ctx):
    """BBPGD with the compressed order-8 operator (host-enqueued iterations: the compressed M2L calls
    cuBLAS) converges, and the oracle's direct LCP certifies its gamma as for the direct M2L."""
    p = make_problem("C5", n=20000, fixed_iters=0)
    t = _cuda
    ctx.set_mobility_model("rpy_fmm")
    ctx.set_fmm_params(8, 0)
    ctx.set_fmm_compression(1)
    try:
        ctx.build_contacts_spheres(t(p.pos), t(p.radius), p.gap_abs, p.gap_rel)
        ctx.assemble_D()
        ctx.lcp_q(p.dt, ctx.mobility_apply(t(p.force), mu=p.mu))
        r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    finally:
        ctx.set_fmm_compression("auto")
        ctx.set_mobility_model("rpy")
    assert r["status"] == 0 and r["residual"] < p.tol
    g = r["gamma"].cpu().numpy()
    sysm = oracle.system_for(p)
    F = oracle.apply_D(p.n, sysm.ct, g) + p.force
    go = sysm.lcp_q(p.dt, sysm.mobility(F))
    q = sysm.lcp_q(p.dt, sysm.mobility(p.force))
    phi = float(np.linalg.norm(np.minimum(g, go)))
    assert phi <= 1e-5 * float(np.linalg.norm(q)), phi


def test_fmm_compression_mode_errors(ctx):
    with pytest.raises(ScError):
        ctx.set_fmm_compression(3)


@pytest.mark.parametrize("n", [5, 300])
def test_fmm_compressed_tiny_problems(ctx, n):
    """Compression forced on a two-level tree (leaf level 2: the smallest interaction grids)."""
    rng = np.random.default_rng(n + 7)
    pos = rng.uniform(0, 2.0 * max(1.0, n ** (1 / 3)), size=(n, 3))
    FT = rng.normal(size=(n, 6))
    ctx.build_contacts_spheres(_cuda(pos), None, 0.0, 0.1)
    ctx.set_mobility_model("rpy_fmm")
    ctx.set_fmm_params(6, 0)
    ctx.set_fmm_compression(1)
    try:
        U = ctx.mobility_apply(_cuda(FT)).cpu().numpy()
    finally:
        ctx.set_fmm_compression("auto")
        ctx.set_mobility_model("rpy")
    Uo = oracle.rpy_apply(pos, np.ones(n), 1.0, FT)
    assert _relL2(U, Uo) <= TOL[6]


@pytest.mark.parametrize("order", [6, 8])
def test_fmm_compressed_polydisperse_vs_oracle(ctx, order):
    """Polydisperse compressed M2L (one basis for the radius-free parts O and D, four products per
    offset) on the C2 recipe: within the stated bars and bitwise-repeatable."""
    p = make_problem("C2", n=8192)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    ctx.set_mobility_model("rpy_fmm")
    ctx.set_fmm_params(order, 3)
    ctx.set_fmm_compression(1)
    try:
        FT = np.random.default_rng(31).normal(size=(p.n, 6))
        U = ctx.mobility_apply(_cuda(FT), mu=p.mu)
        U2 = ctx.mobility_apply(_cuda(FT), mu=p.mu)
    finally:
        ctx.set_fmm_compression("auto")
        ctx.set_mobility_model("rpy")
    assert torch.equal(U, U2)
    Uo = oracle.rpy_apply(p.pos, p.radius, p.mu, FT)
    err = _relL2(U.cpu().numpy()[:, :3], Uo[:, :3])
    assert err <= TOL[order], (order, err)


def test_fmm_tolerance_picks_order_and_meets_it(ctx):
    assert ctx.set_fmm_tolerance(1e-2) == 4
    assert ctx.set_fmm_tolerance(1e-4) == 6
    assert ctx.set_fmm_tolerance(5e-6) == 8
    with pytest.raises(ScError):
        ctx.set_fmm_tolerance(1e-7)
    p = make_problem("C5", n=20000)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    ctx.set_mobility_model("rpy_fmm")
    assert ctx.set_fmm_tolerance(1e-4) == 6 and ctx.fmm_info()["order"] == 6
    FT = np.random.default_rng(41).normal(size=(p.n, 6))
    U = ctx.mobility_apply(_cuda(FT)).cpu().numpy()
    ctx.set_mobility_model("rpy")
    Uo = oracle.rpy_apply(p.pos, p.radius, p.mu, FT)
    assert _relL2(U[:, :3], Uo[:, :3]) <= 1e-4
