"""Seeded synthetic inputs shaped like the paper's workloads.

This module is the ONLY code shared by the oracle side (tests/, bench cpu
baseline) and the CUDA side. It holds no arithmetic of the method: it draws
positions, radii, rod geometry and external forces with
``numpy.random.default_rng(seed)`` and nothing else (the
recipe restated in DESIGN.md "Input recipe").

Workloads (BASELINE.json ``configs``; numbered 1-5 in order):

* C1: 512 monodisperse spheres a=1, volume fraction 0.2, F ~ N(0,1)^3,
  contact threshold gap < 0.1a, dt = 0.01, tol 1e-8, j_max 2000.
* C2: 8,192 spheres, radii U[0.5, 1], volume fraction 0.4,
  F = (0,0,-a_i^3) + N(0, 0.1)^3 (std 0.1, reading A16), threshold
  0.1*min(a_i, a_j), dt = 0.005.
* C3: 65,536 spheres a=1, volume fraction 0.5, F ~ N(0,1)^3, torques (0,0,+-1)
  with a random sign, dt = 0.002, j_max 5000.
* C4: 200,000 spherocylinders, b = 0.5, L ~ U[2,4], directions uniform on the
  sphere, volume fraction 0.3, F ~ N(0,1)^3, gap < 0.1, dt = 0.01 (reading A15).
* C5: 262,144 spheres a=1, volume fraction 0.3, F ~ N(0,1)^3, dt = 0.005;
  fixed 50 BBPGD iterations for timing plus a converged run.

Draw order (fixed): radii, rod lengths, rod directions,
centres U[0, Lbox)^3 with Lbox from the realised volumes (reading A17), forces,
torque signs. ``n`` overrides the body count with the same recipe (same volume
fraction, so the box shrinks), which is how the parity tests get small cases of
every config.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = ["Problem", "CONFIGS", "make_problem"]


@dataclasses.dataclass
class Problem:
    name: str
    kind: str                 # "spheres" or "rods"
    n: int
    pos: np.ndarray           # (n,3) float64 centres
    radius: np.ndarray | None  # (n,) float64 sphere radii (spheres)
    direction: np.ndarray | None  # (n,3) unit axes (rods)
    length: np.ndarray | None     # (n,) cylinder lengths (rods)
    rod_radius: float             # b (rods)
    force: np.ndarray         # (n,6) external force/torque, per body (Fx,Fy,Fz,Tx,Ty,Tz)
    mu: float
    dt: float
    gap_abs: float            # contact iff gap < gap_abs + gap_rel * min(a_i, a_j)
    gap_rel: float
    tol: float
    max_iter: int
    fixed_iters: int          # >0: run exactly this many iterations (C5 timing mode)
    box: float
    monodisperse: bool
    walls: np.ndarray | None = None  # (k,4) planes n.x = h, unit n into the fluid (NEXT row f2)
    mobility: str = "rpy"            # "rpy" (BASELINE) or "rpy6" (full grand mobility, NEXT row f4(ii))

    def nbytes_inputs(self) -> int:
        arrs = [self.pos, self.radius, self.direction, self.length, self.force]
        return int(sum(a.nbytes for a in arrs if a is not None))


# name: (kind, N, volume fraction, dt, gap_abs, gap_rel, j_max, fixed_iters)
CONFIGS = {
    "C1": ("spheres", 512, 0.2, 0.01, 0.0, 0.1, 2000, 0),
    "C2": ("spheres", 8192, 0.4, 0.005, 0.0, 0.1, 5000, 0),
    "C3": ("spheres", 65536, 0.5, 0.002, 0.0, 0.1, 5000, 0),
    "C4": ("rods", 200000, 0.3, 0.01, 0.1, 0.0, 5000, 0),
    "C5": ("spheres", 262144, 0.3, 0.005, 0.0, 0.1, 5000, 50),
}
_SEED = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5}


def make_walls(kind: str | None, box: float) -> np.ndarray | None:
    """Static planar boundaries (NEXT row f2): "floor" = the plane z = 0 (the
    bottom face of the placement cube, normal +z); "box" = the six faces of [0, box]^3 with
    inward normals.  Centres are drawn inside the cube, so bodies near a face overlap it."""
    if kind is None:
        return None
    if kind == "floor":
        return np.array([[0.0, 0.0, 1.0, 0.0]])
    if kind == "box":
        return np.array([[1.0, 0.0, 0.0, 0.0], [-1.0, 0.0, 0.0, -box], [0.0, 1.0, 0.0, 0.0],
                         [0.0, -1.0, 0.0, -box], [0.0, 0.0, 1.0, 0.0], [0.0, 0.0, -1.0, -box]])
    raise ValueError(f"unknown walls {kind!r}")


def make_problem(name: str, n: int | None = None, seed: int | None = None,
                 fixed_iters: int | None = None, walls: str | None = None) -> Problem:
    """Draw the seeded synthetic instance of config ``name`` (C1..C5); ``walls`` adds the
    static planes of :func:`make_walls` (no extra random draws)."""
    kind, n_full, phi, dt, gap_abs, gap_rel, jmax, fixed = CONFIGS[name]
    n = n_full if n is None else int(n)
    rng = np.random.default_rng(_SEED[name] if seed is None else seed)
    radius = direction = length = None
    b = 0.5
    mono = True
    # 1. radii
    if name == "C2":
        radius = rng.uniform(0.5, 1.0, size=n)
        mono = False
    elif kind == "spheres":
        radius = np.ones(n)
    # 2./3. rod lengths and directions
    if kind == "rods":
        length = rng.uniform(2.0, 4.0, size=n)
        d = rng.normal(size=(n, 3))
        direction = d / np.linalg.norm(d, axis=1, keepdims=True)
        vol = float(np.sum(math.pi * b * b * length + 4.0 / 3.0 * math.pi * b ** 3))
    else:
        vol = float(np.sum(4.0 / 3.0 * math.pi * radius ** 3))
    box = (vol / phi) ** (1.0 / 3.0)
    # 4. centres
    pos = rng.uniform(0.0, box, size=(n, 3))
    # 5. forces
    force = np.zeros((n, 6))
    if name == "C2":
        force[:, 2] = -radius ** 3
        force[:, :3] += rng.normal(0.0, 0.1, size=(n, 3))
    else:
        force[:, :3] = rng.normal(size=(n, 3))
    # 6. torque signs (C3 rotors)
    if name == "C3":
        sign = np.where(rng.random(n) < 0.5, -1.0, 1.0)
        force[:, 5] = sign
    return Problem(name=name, kind=kind, n=n, pos=np.ascontiguousarray(pos),
                   radius=radius, direction=direction, length=length, rod_radius=b,
                   force=force, mu=1.0, dt=dt, gap_abs=gap_abs, gap_rel=gap_rel,
                   tol=1e-8, max_iter=jmax,
                   fixed_iters=fixed if fixed_iters is None else fixed_iters,
                   box=box, monodisperse=mono, walls=make_walls(walls, box))
