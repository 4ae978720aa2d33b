"""Pins for the oracle's APGD comparison solver (NEXT row f3).

APGD must reach the same unique CQP solution as brute-force enumeration and as BBPGD, and --
the paper's qualitative finding -- BBPGD needs fewer MVOPs ("BBPGD significantly outperforms
APGD").
"""
import numpy as np
import pytest

import oracle
from paper_1909_06623_b200.synthetic import make_problem
from test_oracle_lcp import _enumerate_lcp


def test_apgd_scalar_and_trivial():
    r = oracle.apgd_dense(np.array([[2.0]]), np.array([-4.0]), tol=1e-12)
    assert r["gamma"][0] == pytest.approx(2.0, rel=1e-10)
    r = oracle.apgd_dense(np.diag([2.0, 3.0]), np.array([0.5, 6.0]))
    assert r["mvops"] == 1 and r["iters"] == 0 and np.all(r["gamma"] == 0)


def test_apgd_random_spd_vs_enumeration():
    rng = np.random.default_rng(7)
    for trial in range(60):
        n = int(rng.integers(1, 9))
        A = rng.normal(size=(n, n))
        M = A @ A.T + 0.1 * np.eye(n)
        q = rng.normal(size=n) * 3
        ref = _enumerate_lcp(M, q)[0]
        r = oracle.apgd_dense(M, q, tol=1e-10, max_iter=200000)
        assert r["status"] == 0, trial
        assert np.abs(r["gamma"] - ref).max() <= 1e-6 * (1 + np.abs(ref).max()), trial


def test_apgd_matches_bbpgd_and_costs_more_mvops_on_c1():
    p = make_problem("C1")
    sysm = oracle.system_for(p)
    q = sysm.lcp_q(p.dt, sysm.mobility(p.force))
    b = sysm.bbpgd(q, tol=1e-8)
    a = sysm.apgd(q, tol=1e-8, max_iter=20000)
    assert a["status"] == 0 and a["residual"] < 1e-8
    rel = np.linalg.norm(a["gamma"] - b["gamma"]) / np.linalg.norm(b["gamma"])
    assert rel < 1e-6, rel
    assert a["mvops"] > b["mvops"], (a["mvops"], b["mvops"])
