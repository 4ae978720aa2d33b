"""The multi-GPU decomposition run on one GPU.

An emulated world of P ranks executes every rank's share of every step (own
constraints' projection, own RPY target rows, own reduction chunks) with the
collectives replaced by their shared-buffer equivalents.  The design claims the
results are BITWISE identical to P = 1 (nsplit, the chunking and every reduction
order depend on N only); these tests hold it to that.
"""
import numpy as np
import pytest
import torch

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


def _solve(ctx, p, world, max_iter, fixed):
    ctx.set_rpy_kernel(1)  # the target-row kernel is the multi-GPU sharding unit
    ctx.set_emulated_world(world)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    ctx.assemble_D()
    U = ctx.mobility_apply(_cuda(p.force), mu=p.mu)
    ctx.lcp_q(p.dt, U)
    r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=max_iter, fixed_iters=fixed)
    r["U_ext"] = U
    ctx.set_emulated_world(1)
    ctx.set_rpy_kernel(0)
    return r


@pytest.mark.parametrize("name,n,max_iter,fixed", [("C1", None, 2000, False), ("C2", 3000, 5000, False),
                                                    ("C5", 9000, 25, True), ("C3", 2500, 5000, False)])
def test_emulated_ranks_bitwise_equal(ctx, name, n, max_iter, fixed):
    p = make_problem(name, n=n)
    ref = _solve(ctx, p, 1, max_iter, fixed)
    for world in (2, 3, 8):
        r = _solve(ctx, p, world, max_iter, fixed)
        assert r["iters"] == ref["iters"] and r["mvops"] == ref["mvops"], world
        assert r["residual"] == ref["residual"]
        for k in ("gamma", "g", "Fc", "Uc", "U_ext"):
            assert torch.equal(r[k], ref[k]), (world, k)


def test_emulated_world_more_ranks_than_blocks(ctx):
    """P larger than the number of 256-row blocks: idle ranks own nothing."""
    p = make_problem("C1", n=300)  # 2 row blocks
    ref = _solve(ctx, p, 1, 2000, False)
    r = _solve(ctx, p, 5, 2000, False)
    assert torch.equal(r["gamma"], ref["gamma"]) and torch.equal(r["Uc"], ref["Uc"])


@pytest.mark.parametrize("name,n,max_iter,fixed", [("C5", 9000, 25, True), ("C3", 6000, 40, True),
                                                    ("C2", 5000, 5000, False)])
def test_emulated_ranks_symmetric_kernel_bitwise(ctx, name, n, max_iter, fixed):
    """The symmetric RPY kernel's multi-GPU unit: ranks evaluate disjoint super-block pairs into
    fixed-point row accumulators whose int64 limbs are summed (all-reduce): integer sums are exact
    and order-free, so U -- and the whole solve -- is BITWISE the one-GPU result for every P."""
    p = make_problem(name, n=n)

    def solve(world):
        ctx.set_rpy_kernel(2)
        ctx.set_emulated_world(world)
        ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
        ctx.assemble_D()
        U = ctx.mobility_apply(_cuda(p.force), mu=p.mu)
        ctx.lcp_q(p.dt, U)
        r = ctx.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=max_iter, fixed_iters=fixed)
        r["U_ext"] = U
        ctx.set_emulated_world(1)
        ctx.set_rpy_kernel(0)
        return r

    ref = solve(1)
    for world in (2, 3, 8):
        r = solve(world)
        assert r["iters"] == ref["iters"] and r["residual"] == ref["residual"], world
        for k in ("gamma", "g", "Fc", "Uc", "U_ext"):
            assert torch.equal(r[k], ref[k]), (world, k)


@pytest.mark.parametrize("name,n,max_iter,fixed,kernel", [("C5", 9000, 25, True, 0), ("C2", 5000, 5000, False, 0),
                                                           ("C3", 2500, 5000, False, 1), ("C1", None, 2000, False, 1)])
def test_one_rank_nccl_path_bitwise_equals_plain_context(ctx, name, n, max_iter, fixed, kernel):
    """sc_create_dist with world = 1 builds a one-rank NCCL communicator and runs the multi-GPU code
    path for real on this GPU -- the partition, grouped ncclBroadcast of the owned (gamma, g)
    slices, ncclAllReduce of the chunk partials (double) and of the RPY fixed-point limbs (int64),
    the host-batched loop -- and must equal the plain 1-GPU context bitwise."""
    from paper_1909_06623_b200 import nccl_unique_id
    p = make_problem(name, n=n)

    def solve(c):
        c.set_rpy_kernel(kernel)
        c.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
        c.assemble_D()
        U = c.mobility_apply(_cuda(p.force), mu=p.mu)
        c.lcp_q(p.dt, U)
        r = c.bbpgd_solve(mu=p.mu, tol=p.tol, max_iter=max_iter, fixed_iters=fixed)
        r["U_ext"] = U
        return r

    ref = solve(ctx)
    ctx.set_rpy_kernel(0)
    d = Context(0, nccl_id=nccl_unique_id(), rank=0, world=1)
    try:
        info = d.comm_info()
        assert info["nranks"] == 1 and info["nccl_version"] > 0
        r = solve(d)
    finally:
        d.close()
    assert r["iters"] == ref["iters"] and r["residual"] == ref["residual"]
    for k in ("gamma", "g", "Fc", "Uc", "U_ext"):
        assert torch.equal(r[k], ref[k]), k
