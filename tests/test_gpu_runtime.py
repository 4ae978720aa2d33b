"""Runtime behaviour of the C ABI on the GPU: residual trace, j_max = 0, warm-start invalidation,
several contexts in one process, stream ordering of the Python binding, communicator info, and
the O(N) exact fixed-point RPY accumulation (bitwise determinism; memory)."""
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
    yield c
    c.close()


def _cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def _setup(c, p):
    c.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    c.assemble_D()
    U = c.mobility_apply(_cuda(p.force), mu=p.mu)
    c.lcp_q(p.dt, U)
    return U


@pytest.mark.parametrize("name,n", [("C1", None), ("C2", 6000), ("C5", 9000)])
def test_residual_trace(ctx, name, n):
    """phi_0 .. phi_J of the solve (Steps 3 and 11): the last entry is the returned residual, the
    trace has iters + 1 entries, and it matches the oracle's iterates' residuals (same Alg. 1)."""
    p = make_problem(name, n=n, fixed_iters=0)
    ctx.set_residual_trace(6000)
    _setup(ctx, p)
    r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    tr = ctx.residual_trace()
    ctx.set_residual_trace(0)
    assert tr.size == r["iters"] + 1
    assert tr[-1] == r["residual"] and tr[-1] < p.tol and np.all(tr[:-1] >= p.tol)
    o = oracle.solve_problem(p, max_iter=5)  # the first iterates agree to rounding
    q = o["q"]
    assert tr[0] == pytest.approx(np.linalg.norm(np.minimum(0.0, q)), rel=1e-12)
    o5 = oracle.solve_problem(p, max_iter=5)
    assert tr[min(5, r["iters"])] == pytest.approx(o5["residual"], rel=1e-6)


def test_max_iter_zero_matches_oracle(ctx):
    """j_max = 0: Steps 1-6 only (alpha_0 computed, no GD step) on every path, persistent included."""
    for n in (None, 3000):
        p = make_problem("C1" if n is None else "C2", n=n, fixed_iters=0)
        _setup(ctx, p)
        r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=0)
        o = oracle.solve_problem(p, max_iter=0)
        assert r["iters"] == 0 == o["iters"] and r["mvops"] == 2 == o["mvops"]
        assert r["status"] == 1 == o["status"]
        assert float(r["gamma"].abs().max()) == 0.0
        assert r["residual"] == pytest.approx(o["residual"], rel=1e-12)


def test_warm_start_not_taken_from_an_older_solve(ctx):
    """An empty solve (n_c = 0) between two solves invalidates the warm-start gamma: the third
    solve starts from 0 like a cold solve (bitwise the same result)."""
    p = make_problem("C2", n=3000, fixed_iters=0)
    _setup(ctx, p)
    cold = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    far = np.array([[0.0, 0.0, 0.0], [100.0, 0.0, 0.0]])
    ctx.build_contacts_spheres(_cuda(far), None, 0.0, 0.1)
    ctx.assemble_D()
    ctx.lcp_q(0.01, ctx.mobility_apply(_cuda(np.zeros((2, 6)))))
    e = ctx.bbpgd_solve(warm_from_previous=True)
    assert e["status"] == 0 and ctx.nc == 0
    _setup(ctx, p)
    w = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter, warm_from_previous=True)
    assert w["iters"] == cold["iters"] and torch.equal(w["gamma"], cold["gamma"])


def test_two_contexts_one_process():
    """Kernel attributes and grids are per device, set in sc_create: a second context (and one
    created after the first is destroyed) runs the 64-KB-shared-memory kernels correctly."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    p = make_problem("C2", n=1900, fixed_iters=0)  # npad 2048: the persistent loop (64 KB smem)
    q = make_problem("C5", n=5000)  # symmetric RPY kernel
    a = Context(0)
    b = Context(0)
    ra = (_setup(a, p), a.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter))
    rb = (_setup(b, q), b.bbpgd_solve(mu=q.mu, tol=q.tol, max_iter=40, fixed_iters=True))
    a.close()
    c = Context(0)
    rc = (_setup(c, p), c.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter))
    assert torch.equal(ra[1]["gamma"], rc[1]["gamma"]) and ra[1]["converged"] == 1
    rb2 = (_setup(c, q), c.bbpgd_solve(mu=q.mu, tol=q.tol, max_iter=40, fixed_iters=True))
    assert torch.equal(rb[0], rb2[0]) and torch.equal(rb[1]["gamma"], rb2[1]["gamma"])
    b.close()
    c.close()


def test_stream_ordering_of_the_binding(ctx):
    """Outputs are produced on the library stream and consumed on torch's current stream: the
    binding orders the two with events, so an immediate torch reduction on a fresh output (no
    explicit synchronisation) sees the library's values."""
    p = make_problem("C5", n=20000)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    ctx.assemble_D()
    F = _cuda(p.force)
    ref = ctx.mobility_apply(F, mu=p.mu).clone()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):  # a non-default caller stream
        for _ in range(3):
            F2 = F * 2.0  # produced on the caller's stream right before the call
            U = ctx.mobility_apply(F2, mu=p.mu)
            s = (U - 2.0 * ref).abs().max()  # consumed on the caller's stream right after
            assert float(s) <= 1e-12 * float(ref.abs().max())


def test_comm_info_one_gpu(ctx):
    info = ctx.comm_info()
    assert info["nranks"] == 1 and info["rank"] == 0 and info["device"] == 0 and info["nccl_version"] > 0


@pytest.mark.parametrize("n", [4096, 30000])
def test_symmetric_rpy_fixed_point_bitwise_repeatable(ctx, n):
    """The symmetric kernel's fixed-point accumulation is exact integer addition: repeated applies
    (different CTA completion orders) are bitwise identical, and equal the target-row kernel to
    rounding (rel. L2 <= 1e-13)."""
    p = make_problem("C5", n=n)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    ctx.assemble_D()
    F = _cuda(p.force * 1e6)  # large forces: the scale adapts
    ctx.set_rpy_kernel(2)
    U = [ctx.mobility_apply(F, mu=p.mu).clone() for _ in range(4)]
    ctx.set_rpy_kernel(1)
    Ur = ctx.mobility_apply(F, mu=p.mu)
    ctx.set_rpy_kernel(0)
    for u in U[1:]:
        assert torch.equal(u, U[0])
    assert float((U[0] - Ur).norm() / Ur.norm()) <= 1e-13


@pytest.mark.parametrize("name,n", [("C1", None), ("C2", 4096), ("C4", 20000), ("C5", 9000)])
def test_results_bitwise_stable_under_schedule_perturbation(ctx, name, n):
    """Race proxy (compute-sanitizer is closed on this pool): a concurrent SM-occupying workload on
    another stream changes which CTAs run when (persistent grid barriers, the symmetric kernel's
    shared reverse accumulators and RED limbs, the last-CTA finalize); every result must stay
    bitwise identical to an undisturbed solve."""
    p = make_problem(name, n=n, fixed_iters=0)

    def solve():
        if p.kind == "spheres":
            ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
        else:
            ctx.build_contacts_rods(_cuda(p.pos), _cuda(p.direction), _cuda(p.length), p.rod_radius, p.gap_abs)
        ctx.assemble_D()
        U = ctx.mobility_apply(_cuda(p.force), mu=p.mu)
        ctx.lcp_q(p.dt, U)
        r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=min(p.max_iter, 300))
        return U, r

    U0, r0 = solve()
    side = torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda", dtype=torch.float32)
    for k in range(3):
        with torch.cuda.stream(side):
            for _ in range(20 + 10 * k):
                a = torch.tanh(a @ a.T * 1e-3)  # keeps SMs busy while the solve is enqueued
        U1, r1 = solve()
        torch.cuda.synchronize()
        assert torch.equal(U0, U1)
        assert r1["iters"] == r0["iters"] and r1["residual"] == r0["residual"]
        for key in ("gamma", "g", "Fc", "Uc"):
            assert torch.equal(r0[key], r1[key]), (k, key)


def test_checked_build_flag_matches_the_loaded_library(ctx):
    """SC_LIB=.../libstokescol_checked.so runs the suite against the checked build (device-side
    bounds asserts); its flag says so, so a checked run cannot silently use the release build."""
    import os
    want = 1 if "checked" in os.environ.get("SC_LIB", "") else 0
    assert ctx.lib.sc_build_flags() & 1 == want


def test_residual_trace_truncated_and_off(ctx):
    p = make_problem("C2", n=3000, fixed_iters=0)
    ctx.set_residual_trace(10)
    _setup(ctx, p)
    r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    tr = ctx.residual_trace()
    assert r["iters"] > 10 and tr.size == 10 and np.all(tr > 0)
    ctx.set_residual_trace(0)
    _setup(ctx, p)
    ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=p.max_iter)
    assert ctx.residual_trace().size == 0
