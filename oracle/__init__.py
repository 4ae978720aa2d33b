"""CPU FP64 oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product (``paper_1909_06623_b200``) never imports it, and it never imports
the product.  It wraps ``oracle.c`` (plain C, ``-O2 -fopenmp
-ffp-contract=off``) with ctypes + numpy; every arithmetic step of the method
lives in ``oracle.c`` and cites PAPER.md there.

Parity pins: see tests/test_oracle_*.py and DESIGN.md "Oracle pins".  The
only function without an independent pin is the exact BBPGD iteration count
("parity unpinned").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

ORC_SPHERES, ORC_RODS, ORC_SPHERES_RPY6 = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, no FMA contraction)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
        _declare(_lib)
    return _lib


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class _Sys(C.Structure):
    _fields_ = [("kind", C.c_int), ("n", C.c_int64), ("pos", C.c_void_p), ("radius", C.c_void_p),
                ("dir", C.c_void_p), ("length", C.c_void_p), ("b", C.c_double), ("mu", C.c_double),
                ("nc", C.c_int64), ("ci", C.c_void_p), ("cj", C.c_void_p), ("normal", C.c_void_p),
                ("lever", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("mvops", C.c_int32), ("converged", C.c_int32),
                ("bb_breakdowns", C.c_int32), ("active", C.c_int32), ("residual", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _declare(L):
    i64, i32, d = C.c_int64, C.c_int32, C.c_double
    vp = C.c_void_p
    L.orc_contacts_spheres_brute.restype = i64
    L.orc_contacts_spheres_brute.argtypes = [i64, vp, vp, d, d, i64, vp, vp, vp, vp]
    L.orc_contacts_spheres_grid.restype = i64
    L.orc_contacts_spheres_grid.argtypes = [i64, vp, vp, d, d, i64, vp, vp, vp, vp]
    L.orc_contacts_rods.restype = i64
    L.orc_contacts_rods.argtypes = [i64, vp, vp, vp, d, d, C.c_int, i64, vp, vp, vp, vp, vp]
    L.orc_contacts_walls.restype = i64
    L.orc_contacts_walls.argtypes = [C.c_int, i64, vp, vp, vp, vp, d, C.c_int, vp, d, d, i64, vp, vp, vp, vp, vp]
    L.orc_segment_closest.restype = None
    L.orc_segment_closest.argtypes = [vp, vp, d, vp, vp, d, vp, vp]
    L.orc_apply_D.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp]
    L.orc_apply_DT.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp]
    L.orc_rpy_apply.argtypes = [i64, vp, vp, d, vp, vp]
    L.orc_rpy_apply_rows.argtypes = [i64, vp, vp, d, vp, i64, i64, vp]
    L.orc_rpy_block.restype = None
    L.orc_rpy_block.argtypes = [vp, d, vp, d, d, C.c_int, vp]
    L.orc_rod_drag_apply.argtypes = [i64, vp, vp, d, d, vp, vp]
    L.orc_rpy6_block.restype = None
    L.orc_rpy6_block.argtypes = [vp, d, vp, d, d, C.c_int, vp]
    L.orc_rpy6_apply_rows.argtypes = [i64, vp, vp, d, vp, i64, i64, vp]
    L.orc_lcp_q.argtypes = [C.POINTER(_Sys), vp, d, vp, vp]
    L.orc_lcp_q_moving_walls.argtypes = [C.POINTER(_Sys), vp, d, vp, C.c_int, vp, vp]
    L.orc_mvop.argtypes = [C.POINTER(_Sys), vp, vp]
    L.orc_bbpgd.argtypes = [C.POINTER(_Sys), vp, d, i32, i32, i32, vp, vp, vp, vp, C.POINTER(Stats)]
    L.orc_bbpgd_dense.argtypes = [i64, vp, vp, d, i32, i32, vp, vp, C.POINTER(Stats)]
    L.orc_minmap_residual.restype = d
    L.orc_minmap_residual.argtypes = [i64, vp, vp]
    L.orc_euler_update.argtypes = [i64, d, vp, vp, vp, vp]
    L.orc_apgd.argtypes = [C.POINTER(_Sys), vp, d, i32, vp, vp, C.POINTER(Stats)]
    L.orc_apgd_dense.argtypes = [i64, vp, vp, d, i32, vp, vp, C.POINTER(Stats)]


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    pass


def _check(st, what):
    if st < 0:
        raise OracleError(f"{what}: status {st}")
    return st


# ----------------------------------------------------------------- contacts
class Contacts:
    """Constraint list sorted by (i, j), i < j; normal from j to i."""

    def __init__(self, ci, cj, gap, normal, lever=None):
        self.i, self.j, self.gap, self.normal, self.lever = ci, cj, gap, normal, lever

    @property
    def nc(self):
        return int(self.i.shape[0])


def contacts_spheres(pos, radius, gap_abs, gap_rel, method="grid"):
    pos, radius = _f64(pos), _f64(radius)
    n = pos.shape[0]
    fn = lib().orc_contacts_spheres_grid if method == "grid" else lib().orc_contacts_spheres_brute
    cap = max(16, 8 * n)
    while True:
        ci = np.empty(cap, np.int32); cj = np.empty(cap, np.int32)
        gap = np.empty(cap); nrm = np.empty((cap, 3))
        nc = _check(fn(n, _p(pos), _p(radius), gap_abs, gap_rel, cap, _p(ci), _p(cj), _p(gap), _p(nrm)),
                    "contacts_spheres")
        if nc <= cap:
            return Contacts(ci[:nc].copy(), cj[:nc].copy(), gap[:nc].copy(), nrm[:nc].copy())
        cap = nc


def contacts_rods(center, direction, length, b, gap_thresh, brute=False):
    center, direction, length = _f64(center), _f64(direction), _f64(length)
    n = center.shape[0]
    cap = max(16, 8 * n)
    while True:
        ci = np.empty(cap, np.int32); cj = np.empty(cap, np.int32)
        gap = np.empty(cap); nrm = np.empty((cap, 3)); lev = np.empty((cap, 2, 3))
        nc = _check(lib().orc_contacts_rods(n, _p(center), _p(direction), _p(length), b, gap_thresh,
                                            int(bool(brute)), cap, _p(ci), _p(cj), _p(gap), _p(nrm),
                                            _p(lev)), "contacts_rods")
        if nc <= cap:
            return Contacts(ci[:nc].copy(), cj[:nc].copy(), gap[:nc].copy(), nrm[:nc].copy(),
                            lev[:nc].copy())
        cap = nc


def contacts_walls(kind, pos, walls, radius=None, direction=None, length=None, b=0.5, gap_abs=0.0,
                   gap_rel=0.1):
    """Particle-wall constraints (i, n + k) in body order (oracle.c orc_contacts_walls)."""
    pos, walls = _f64(pos), _f64(walls)
    radius, direction, length = _f64(radius), _f64(direction), _f64(length)
    n, nw = pos.shape[0], walls.shape[0]
    rods = kind == "rods"
    cap = max(16, n * nw)
    ci = np.empty(cap, np.int32); cj = np.empty(cap, np.int32)
    gap = np.empty(cap); nrm = np.empty((cap, 3)); lev = np.empty((cap, 2, 3))
    m = _check(lib().orc_contacts_walls(int(rods), n, _p(pos), _p(radius), _p(direction), _p(length), float(b),
                                        nw, _p(walls), float(gap_abs), float(gap_rel), cap, _p(ci), _p(cj),
                                        _p(gap), _p(nrm), _p(lev) if rods else None), "contacts_walls")
    return Contacts(ci[:m].copy(), cj[:m].copy(), gap[:m].copy(), nrm[:m].copy(), lev[:m].copy() if rods else None)


def merge_contacts(a: Contacts, b: Contacts) -> Contacts:
    """Union of two constraint lists, sorted by (i, j) (walls j = n + k sort last per i)."""
    ci = np.concatenate([a.i, b.i]); cj = np.concatenate([a.j, b.j])
    order = np.lexsort((cj, ci))
    lev = None if a.lever is None else np.concatenate([a.lever, b.lever])[order]
    return Contacts(ci[order], cj[order], np.concatenate([a.gap, b.gap])[order],
                    np.concatenate([a.normal, b.normal])[order], lev)


def segment_closest(c1, t1, L1, c2, t2, L2):
    P1 = np.empty(3); P2 = np.empty(3)
    c1, t1, c2, t2 = _f64(c1), _f64(t1), _f64(c2), _f64(t2)
    lib().orc_segment_closest(_p(c1), _p(t1), float(L1), _p(c2), _p(t2), float(L2), _p(P1), _p(P2))
    return P1, P2


# -------------------------------------------------------------- D and D^T
def apply_D(n, ct: Contacts, gamma):
    gamma = _f64(gamma)
    FT = np.empty((n, 6))
    _check(lib().orc_apply_D(n, ct.nc, _p(ct.i), _p(ct.j), _p(ct.normal), _p(ct.lever), _p(gamma),
                             _p(FT)), "apply_D")
    return FT


def apply_DT(n, ct: Contacts, UW):
    UW = _f64(UW)
    out = np.empty(ct.nc)
    _check(lib().orc_apply_DT(n, ct.nc, _p(ct.i), _p(ct.j), _p(ct.normal), _p(ct.lever), _p(UW),
                              _p(out)), "apply_DT")
    return out


# --------------------------------------------------------------- mobility
def rpy_apply(pos, radius, mu, FT):
    pos, radius, FT = _f64(pos), _f64(radius), _f64(FT)
    UW = np.empty((pos.shape[0], 6))
    _check(lib().orc_rpy_apply(pos.shape[0], _p(pos), _p(radius), mu, _p(FT), _p(UW)), "rpy_apply")
    return UW


def rpy_apply_rows(pos, radius, mu, FT, row0, row1):
    pos, radius, FT = _f64(pos), _f64(radius), _f64(FT)
    UW = np.empty((row1 - row0, 6))
    _check(lib().orc_rpy_apply_rows(pos.shape[0], _p(pos), _p(radius), mu, _p(FT), row0, row1, _p(UW)),
           "rpy_apply_rows")
    return UW


def rpy_block(xi, ai, xj, aj, mu, self_block=False):
    M = np.empty(9)
    xi, xj = _f64(xi), _f64(xj)  # (keep the converted arrays alive across the call)
    lib().orc_rpy_block(_p(xi), float(ai), _p(xj), float(aj), float(mu), int(self_block), _p(M))
    return M.reshape(3, 3)


def rpy6_apply(pos, radius, mu, FT, row0=0, row1=None):
    """Full 6N RPY grand mobility (NEXT row f4(ii), oracle.c orc_rpy6_block)."""
    pos, radius, FT = _f64(pos), _f64(radius), _f64(FT)
    n = pos.shape[0]
    row1 = n if row1 is None else row1
    UW = np.empty((row1 - row0, 6))
    _check(lib().orc_rpy6_apply_rows(n, _p(pos), _p(radius), mu, _p(FT), row0, row1, _p(UW)), "rpy6_apply")
    return UW


def rpy6_block(xi, ai, xj, aj, mu, self_block=False):
    M = np.empty(36)
    xi, xj = _f64(xi), _f64(xj)
    lib().orc_rpy6_block(_p(xi), float(ai), _p(xj), float(aj), float(mu), int(self_block), _p(M))
    return M.reshape(6, 6)


def rod_drag_apply(direction, length, b, mu, FT):
    direction, length, FT = _f64(direction), _f64(length), _f64(FT)
    UW = np.empty((direction.shape[0], 6))
    _check(lib().orc_rod_drag_apply(direction.shape[0], _p(direction), _p(length), b, mu, _p(FT), _p(UW)),
           "rod_drag_apply")
    return UW


# ------------------------------------------------------------ LCP + BBPGD
class System:
    """Holds numpy arrays alive for an ``orc_system`` struct."""

    def __init__(self, kind, n, ct: Contacts, mu=1.0, pos=None, radius=None, direction=None,
                 length=None, b=0.5):
        self.kind, self.n, self.ct, self.mu, self.b = kind, n, ct, mu, b
        self.pos, self.radius = _f64(pos), _f64(radius)
        self.direction, self.length = _f64(direction), _f64(length)
        self.s = _Sys(kind, n, _p(self.pos), _p(self.radius), _p(self.direction), _p(self.length),
                      b, mu, ct.nc, _p(ct.i), _p(ct.j), _p(ct.normal), _p(ct.lever))

    def mobility(self, FT):
        if self.kind == ORC_SPHERES:
            return rpy_apply(self.pos, self.radius, self.mu, FT)
        if self.kind == ORC_SPHERES_RPY6:
            return rpy6_apply(self.pos, self.radius, self.mu, FT)
        return rod_drag_apply(self.direction, self.length, self.b, self.mu, FT)

    def lcp_q(self, dt, U_nc):
        U_nc = _f64(U_nc)
        q = np.empty(self.ct.nc)
        _check(lib().orc_lcp_q(C.byref(self.s), _p(self.ct.gap), dt, _p(U_nc), _p(q)), "lcp_q")
        return q

    def lcp_q_moving_walls(self, dt, U_nc, wall_vel):
        """q with walls moving at the prescribed velocities wall_vel (k x 3)."""
        U_nc, wv = _f64(U_nc), _f64(np.asarray(wall_vel, dtype=np.float64).reshape(-1, 3))
        q = np.empty(self.ct.nc)
        _check(lib().orc_lcp_q_moving_walls(C.byref(self.s), _p(self.ct.gap), dt, _p(U_nc), wv.shape[0], _p(wv),
                                            _p(q)), "lcp_q_moving_walls")
        return q

    def mvop(self, x):
        x = _f64(x)
        w = np.empty(self.ct.nc)
        _check(lib().orc_mvop(C.byref(self.s), _p(x), _p(w)), "mvop")
        return w

    def apgd(self, q, tol=1e-8, max_iter=20000):
        q = _f64(q)
        nc = self.ct.nc
        gamma = np.zeros(nc); g = np.empty(nc); st = Stats()
        rc = _check(lib().orc_apgd(C.byref(self.s), _p(q), tol, max_iter, _p(gamma), _p(g), C.byref(st)), "apgd")
        return {"gamma": gamma, "g": g, "status": rc, **st.as_dict()}

    def bbpgd(self, q, tol=1e-8, max_iter=5000, bb_mode=0, fixed_iters=0, gamma0=None):
        q = _f64(q)
        nc = self.ct.nc
        gamma = np.zeros(nc) if gamma0 is None else _f64(gamma0).copy()
        g = np.empty(nc); Fc = np.empty((self.n, 6)); Uc = np.empty((self.n, 6))
        st = Stats()
        rc = _check(lib().orc_bbpgd(C.byref(self.s), _p(q), tol, max_iter, bb_mode, int(fixed_iters),
                                    _p(gamma), _p(g), _p(Fc), _p(Uc), C.byref(st)), "bbpgd")
        return {"gamma": gamma, "g": g, "Fc": Fc, "Uc": Uc, "status": rc, **st.as_dict()}


def apgd_dense(M, q, tol=1e-8, max_iter=20000):
    M, q = _f64(M), _f64(q)
    n = q.shape[0]
    gamma = np.zeros(n); g = np.empty(n); st = Stats()
    rc = _check(lib().orc_apgd_dense(n, _p(M), _p(q), tol, max_iter, _p(gamma), _p(g), C.byref(st)), "apgd_dense")
    return {"gamma": gamma, "g": g, "status": rc, **st.as_dict()}


def bbpgd_dense(M, q, tol=1e-8, max_iter=5000, bb_mode=0):
    M, q = _f64(M), _f64(q)
    n = q.shape[0]
    gamma = np.zeros(n); g = np.empty(n); st = Stats()
    rc = _check(lib().orc_bbpgd_dense(n, _p(M), _p(q), tol, max_iter, bb_mode, _p(gamma), _p(g),
                                      C.byref(st)), "bbpgd_dense")
    return {"gamma": gamma, "g": g, "status": rc, **st.as_dict()}


def minmap_residual(gamma, g):
    gamma, g = _f64(gamma), _f64(g)
    return float(lib().orc_minmap_residual(gamma.shape[0], _p(gamma), _p(g)))


def euler_update(dt, UW, pos, quat=None, direction=None):
    """Step 4: returns updated copies (pos, quat, direction)."""
    UW = _f64(UW)
    pos = _f64(pos).copy()
    quat = None if quat is None else _f64(quat).copy()
    direction = None if direction is None else _f64(direction).copy()
    _check(lib().orc_euler_update(pos.shape[0], dt, _p(UW), _p(pos), _p(quat), _p(direction)), "euler_update")
    return pos, quat, direction


def warm_gamma(prev_ct, prev_gamma, ct):
    """gamma_0 for a new constraint list: the previous gamma of the same pair (i, j), else 0."""
    if prev_ct is None:
        return None
    prev = {(int(i), int(j)): g for i, j, g in zip(prev_ct.i, prev_ct.j, prev_gamma)}
    return np.array([prev.get((int(i), int(j)), 0.0) for i, j in zip(ct.i, ct.j)])


def time_step(problem, quat=None, max_iter=None, warm=None):
    """The four steps of P:L480-L489 on the CPU: U_nc, contacts + D, LCP, Euler update.
    warm = (prev contacts, prev gamma): Step 1's gamma_0 from the previous step's gamma."""
    res = solve_problem(problem, max_iter=max_iter, fixed_iters=0, warm=warm)
    U = res["U_ext"] + res["Uc"]
    pos, quat, direction = euler_update(problem.dt, U, problem.pos, quat,
                                        problem.direction if problem.kind == "rods" else None)
    res.update(pos=pos, quat=quat, direction=direction, U=U)
    return res


# ------------------------------------------------------ one-call pipeline
def system_for(problem, method="grid"):
    """Contacts (+ wall constraints, if the problem has walls) + System for a synthetic
    ``Problem`` (spheres or rods)."""
    walls = getattr(problem, "walls", None)
    if problem.kind == "spheres":
        ct = contacts_spheres(problem.pos, problem.radius, problem.gap_abs, problem.gap_rel, method)
        if walls is not None and len(walls):
            ct = merge_contacts(ct, contacts_walls("spheres", problem.pos, walls, radius=problem.radius,
                                                   gap_abs=problem.gap_abs, gap_rel=problem.gap_rel))
        kind = ORC_SPHERES_RPY6 if getattr(problem, "mobility", "rpy") == "rpy6" else ORC_SPHERES
        return System(kind, problem.n, ct, mu=problem.mu, pos=problem.pos, radius=problem.radius)
    ct = contacts_rods(problem.pos, problem.direction, problem.length, problem.rod_radius, problem.gap_abs)
    if walls is not None and len(walls):
        ct = merge_contacts(ct, contacts_walls("rods", problem.pos, walls, direction=problem.direction,
                                               length=problem.length, b=problem.rod_radius,
                                               gap_abs=problem.gap_abs))
    return System(ORC_RODS, problem.n, ct, mu=problem.mu, direction=problem.direction,
                  length=problem.length, b=problem.rod_radius)


def solve_problem(problem, max_iter=None, fixed_iters=None, bb_mode=0, warm=None):
    """The whole per-step path on the CPU: contacts, D, U_ext, q, BBPGD."""
    sysm = system_for(problem)
    U_ext = sysm.mobility(problem.force)
    q = sysm.lcp_q(problem.dt, U_ext)
    fixed = problem.fixed_iters if fixed_iters is None else fixed_iters
    jmax = (fixed if fixed else problem.max_iter) if max_iter is None else max_iter
    g0 = warm_gamma(warm[0], warm[1], sysm.ct) if warm is not None else None
    res = sysm.bbpgd(q, tol=problem.tol, max_iter=jmax, bb_mode=bb_mode, fixed_iters=int(bool(fixed)), gamma0=g0)
    res.update(system=sysm, q=q, U_ext=U_ext)
    return res
