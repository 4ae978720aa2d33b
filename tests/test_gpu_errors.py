"""Error behaviour of the C ABI on the GPU (include/stokescol.h: every call returns an
sc_status; SPEC's hard errors for coincident centres, dimension misuse and non-finite
values; a soft SC_NOT_CONVERGED at the iteration cap, reading A7)."""
import numpy as np
import pytest
import torch

from paper_1909_06623_b200 import Context, ScError
from paper_1909_06623_b200.synthetic import make_problem

pytestmark = pytest.mark.gpu

EINVAL, EDEGENERATE, ENONFINITE = -1, -2, -3


@pytest.fixture()
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    c = Context(0)
    yield c
    c.close()


def _cuda(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def _code(fn):
    with pytest.raises(ScError) as e:
        fn()
    return e.value.code


def test_calls_out_of_order(ctx):
    assert _code(lambda: ctx.assemble_D()) == EINVAL
    assert _code(lambda: ctx.mobility_apply(_cuda(np.zeros((0, 6))))) == EINVAL  # before build_contacts
    pos = np.array([[0.0, 0, 0], [2.05, 0, 0]])
    ctx.build_contacts_spheres(_cuda(pos), None, 0.0, 0.1)
    assert _code(lambda: ctx.bbpgd_solve()) == EINVAL  # needs assemble_D and lcp_q first
    ctx.assemble_D()
    assert _code(lambda: ctx.bbpgd_solve()) == EINVAL  # still no q


def test_bad_arguments(ctx):
    pos = np.array([[0.0, 0, 0], [2.05, 0, 0]])
    assert _code(lambda: ctx.build_contacts_spheres(_cuda(pos), None, 0.0, -0.1)) == EINVAL  # gap_rel < 0
    assert _code(lambda: ctx.build_contacts_rods(_cuda(pos), _cuda(np.eye(3)[:2]), _cuda([3.0, 3.0]), -0.5,
                                                 0.1)) == EINVAL  # b <= 0
    # rod shorter than its diameter: ln(L/2b) <= 0 makes the drag undefined
    assert _code(lambda: ctx.build_contacts_rods(_cuda(pos), _cuda(np.eye(3)[:2]), _cuda([0.5, 3.0]), 0.5,
                                                 0.1)) == EINVAL
    ctx.build_contacts_spheres(_cuda(pos), None, 0.0, 0.1)
    ctx.assemble_D()
    ctx.lcp_q(0.01, _cuda(np.zeros((2, 6))))
    assert _code(lambda: ctx.bbpgd_solve(mu=-1.0)) == EINVAL
    assert _code(lambda: ctx.bbpgd_solve(bb_mode=7)) == EINVAL
    assert _code(lambda: ctx.set_mobility_model(5)) == EINVAL
    assert _code(lambda: ctx.set_rpy_kernel(9)) == EINVAL


def test_non_finite_inputs(ctx):
    pos = np.array([[0.0, 0, 0], [2.05, 0, 0], [np.nan, 1.0, 1.0]])
    assert _code(lambda: ctx.build_contacts_spheres(_cuda(pos), None, 0.0, 0.1)) == ENONFINITE
    # a NaN external force reaches the gradient: hard error (SPEC), not a silent result
    pos = np.array([[0.0, 0, 0], [2.05, 0, 0]])
    ctx.build_contacts_spheres(_cuda(pos), None, 0.0, 0.1)
    ctx.assemble_D()
    F = np.zeros((2, 6)); F[0, 0] = np.nan
    ctx.lcp_q(0.01, ctx.mobility_apply(_cuda(F)))
    assert _code(lambda: ctx.bbpgd_solve()) == ENONFINITE


def test_coincident_centres_rods(ctx):
    c = np.array([[0.0, 0, 0], [0.0, 0, 0]])
    t = np.array([[1.0, 0, 0], [1.0, 0, 0]])  # identical segments: no defined normal
    assert _code(lambda: ctx.build_contacts_rods(_cuda(c), _cuda(t), _cuda([3.0, 3.0]), 0.5, 0.1)) == EDEGENERATE


def test_iteration_cap_is_soft(ctx):
    """j_max reached without convergence: SC_NOT_CONVERGED with the last iterate (reading A7)."""
    p = make_problem("C2", n=2048, fixed_iters=0)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    ctx.assemble_D()
    ctx.lcp_q(p.dt, ctx.mobility_apply(_cuda(p.force)))
    r = ctx.bbpgd_solve(tol=1e-8, max_iter=5)
    assert r["status"] == 1 and r["converged"] == 0 and r["iters"] == 5 and r["mvops"] == 7
    assert float(r["gamma"].min()) >= 0.0 and np.isfinite(r["residual"])


def test_minmap_residual_entry_point(ctx):
    """sc_minmap_residual (SPEC's min_map_residual) equals the solver's phi and numpy's."""
    p = make_problem("C1", fixed_iters=0)
    ctx.build_contacts_spheres(_cuda(p.pos), _cuda(p.radius), p.gap_abs, p.gap_rel)
    ctx.assemble_D()
    ctx.lcp_q(p.dt, ctx.mobility_apply(_cuda(p.force)))
    r = ctx.bbpgd_solve(tol=p.tol, max_iter=p.max_iter)
    phi = ctx.minmap_residual(r["gamma"], r["g"])
    gm, g = r["gamma"].cpu().numpy(), r["g"].cpu().numpy()
    assert phi == pytest.approx(float(np.linalg.norm(np.minimum(gm, g))), rel=1e-12)
    assert phi == pytest.approx(r["residual"], rel=1e-10)
    # host buffers through the same entry point
    assert ctx.minmap_residual(gm, g) == pytest.approx(phi, rel=1e-15)
    with pytest.raises(ValueError):
        ctx.minmap_residual(r["gamma"], r["g"][:-1])
