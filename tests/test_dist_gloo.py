"""CPU test (world size 2, gloo) of the multi-GPU decomposition.

Each process plays one rank of the NCCL design with torch.distributed/gloo standing in
for NCCL and the oracle standing in for the kernels (test infrastructure):
  * rank r owns the RPY target rows plan_partition(n, P, r) gives it and the
    constraints whose first body it owns (the paper's smaller-index rule);
  * per iteration: projection of own constraints -> broadcast of every rank's slice;
    F = D gamma locally; RPY of own rows -> all-gather of the rows; D^T + chunk partials
    of own 256-body chunks -> all-reduce of the zero-padded partial vector; fixed-order
    final sums -> identical alpha / phi / stop decision on every rank.
The distributed BBPGD must reach the single-process oracle's gamma.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1909_06623_b200 import plan_partition
from paper_1909_06623_b200.synthetic import make_problem

WORLD = 2
CHUNK = 256


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _first_ptr(ct, n):
    fp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(fp, ct.i.astype(np.int64) + 1, 1)
    return np.cumsum(fp)


def _rank_main(rank, world, port, name, n, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = make_problem(name, n=n)
    n = p.n
    ct = oracle.contacts_spheres(p.pos, p.radius, p.gap_abs, p.gap_rel)
    fp = _first_ptr(ct, n)
    parts = [plan_partition(n, world, r) for r in range(world)]
    me = parts[rank]
    npad, nch = me["npad"], me["npad"] // CHUNK
    clip = lambda b: min(b, n)
    lo, hi = clip(me["row_lo"]), clip(me["row_hi"])
    l0, l1 = fp[lo], fp[hi]
    slices = [(fp[clip(q["row_lo"])], fp[clip(q["row_hi"])]) for q in parts]

    def bcast_slices(v):
        for r, (a, b) in enumerate(slices):
            t = torch.from_numpy(v[a:b].copy())
            dist.broadcast(t, src=r)
            v[a:b] = t.numpy()

    def rpy_rows_allgather(FT):
        own = oracle.rpy_apply_rows(p.pos, p.radius, p.mu, FT, lo, hi) if hi > lo else np.zeros((0, 6))
        rpr = me["rows_per_rank"]
        buf = np.zeros((rpr, 6))
        buf[: hi - lo] = own
        out = [torch.zeros(rpr, 6, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, torch.from_numpy(buf))
        return torch.cat(out).numpy()[:n]

    def chunk_sums(vals):  # vals: (nc, k) own rows valid -> fixed-order global sums
        part = np.zeros((nch, vals.shape[1]))
        for c in range(me["chunk_lo"], me["chunk_hi"]):
            a, b = fp[clip(c * CHUNK)], fp[clip(c * CHUNK + CHUNK)]
            part[c] = vals[a:b].sum(0)
        t = torch.from_numpy(part)
        dist.all_reduce(t)
        return t.numpy().sum(0)

    # U_ext and q (own constraints)
    U = rpy_rows_allgather(p.force)
    q = np.zeros(ct.nc)
    q[l0:l1] = (ct.gap / p.dt + oracle.apply_DT(n, ct, U))[l0:l1]
    bcast_slices(q)  # (for the final comparison only)

    def grad_own(gam_full):  # own slice of M gamma (no q)
        F = oracle.apply_D(n, ct, gam_full)
        Ufull = rpy_rows_allgather(F)
        return oracle.apply_DT(n, ct, Ufull)

    gam = np.zeros(ct.nc)
    g = q.copy()  # gamma_0 = 0: g_0 = q (Step 2, one counted MVOP)
    phi = np.sqrt(chunk_sums(np.minimum(gam, g)[:, None] ** 2)[0])
    iters = 0
    if not phi < p.tol:
        bcast_slices(g)
        w = grad_own(g)
        s2 = chunk_sums(np.stack([g * g, g * w], 1))
        alpha = s2[0] / s2[1]  # Step 6
        for j in range(1, p.max_iter + 1):
            gnew = np.zeros(ct.nc)
            gnew[l0:l1] = np.maximum(gam[l0:l1] - alpha * g[l0:l1], 0.0)  # Steps 8-9 (own)
            bcast_slices(gnew)
            gg = np.zeros(ct.nc)
            gg[l0:l1] = grad_own(gnew)[l0:l1] + q[l0:l1]  # Step 10 (own)
            s = gnew - gam
            y = gg - g
            sums = chunk_sums(np.stack([s * s, s * y, y * y, np.minimum(gnew, gg) ** 2], 1))
            gam, g = gnew, gg
            iters = j
            phi = np.sqrt(sums[3])
            if phi < p.tol:
                break
            if sums[1] > 0:
                alpha = sums[0] / sums[1]  # BB1, Step 15
    bcast_slices(g)
    np.save(os.path.join(outdir, f"gamma{rank}.npy"), gam)
    np.save(os.path.join(outdir, f"meta{rank}.npy"), np.array([iters, phi, l0, l1]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,n", [("C1", 512), ("C2", 700)])
def test_gloo_world2_bbpgd_matches_oracle(tmp_path, name, n):
    port = _free_port()
    mp.spawn(_rank_main, args=(WORLD, port, name, n, str(tmp_path)), nprocs=WORLD, join=True)
    g0 = np.load(tmp_path / "gamma0.npy")
    g1 = np.load(tmp_path / "gamma1.npy")
    m0, m1 = np.load(tmp_path / "meta0.npy"), np.load(tmp_path / "meta1.npy")
    # every rank ends with the same full gamma and took the same decisions
    np.testing.assert_array_equal(g0, g1)
    assert m0[0] == m1[0] and m0[1] == m1[1] and m0[1] < 1e-8
    # ownership: the two ranks' constraint slices tile [0, n_c) with no overlap
    assert m0[2] == 0 and m0[3] == m1[2]
    ref = oracle.solve_problem(make_problem(name, n=n))
    assert m1[3] == ref["system"].ct.nc
    rel = np.linalg.norm(g0 - ref["gamma"]) / np.linalg.norm(ref["gamma"])
    assert rel < 1e-8, rel


# ------------------------------------------------------------- symmetric RPY decomposition
SB = 512


def _fx_scale(force, radius, npad):
    """The fixed-point shift s of rpy.cu (fx_shift): |row sum| * 2^s < 2^100."""
    mf = float(np.abs(force[:, :3]).max())
    mi = float((1.0 / radius).max())
    B = 2.0 * mf * mi * npad
    if not B > 0:
        return 0
    return int(100 - (np.floor(np.log2(B)) + 1))


def _to_fixed(v, s):
    """round(v 2^s) (ties away from zero) as a Python int, split in 3 limbs of 43 bits."""
    from fractions import Fraction
    x = Fraction(v) * (Fraction(2) ** s)
    X = int(abs(x) + Fraction(1, 2)) * (1 if x >= 0 else -1)
    m = (1 << 43) - 1
    return X & m, (X >> 43) & m, X >> 86


def _sym_rank_main(rank, world, port, name, n, outdir):
    """Rank r evaluates its super-block pairs (the library's own table), rounds each (pair, row)
    partial sum to the fixed-point limbs and the limbs are all-reduced (int64 sum) -- the design
    of rpy.cu; the oracle's RPY rows stand in for the kernel."""
    from paper_1909_06623_b200 import sym_pair_table
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = make_problem(name, n=n)
    n = p.n
    npad = -(-n // SB) * SB
    nsb = npad // SB
    rng = np.random.default_rng(3)
    FT = np.zeros((n, 6))
    FT[:, :3] = rng.normal(size=(n, 3)) * 10.0 ** rng.uniform(-3, 3, size=(n, 1))
    s = _fx_scale(FT, p.radius, npad)
    limbs = np.zeros((npad, 3, 3), dtype=np.int64)

    def add(rows, vals):
        for r, v in zip(rows, vals):
            for c in range(3):
                x0, x1, x2 = _to_fixed(float(v[c]), s)
                limbs[r, c, 0] += x0
                limbs[r, c, 1] += x1
                limbs[r, c, 2] += x2

    def block(ti, sj):  # rows of super-block ti from the sources of super-block sj
        r0, r1 = ti * SB, min(n, ti * SB + SB)
        s0, s1 = sj * SB, min(n, sj * SB + SB)
        if r1 <= r0 or s1 <= s0:
            return np.arange(0), np.zeros((0, 3))
        F = np.zeros_like(FT)
        F[s0:s1] = FT[s0:s1]
        return np.arange(r0, r1), oracle.rpy_apply_rows(p.pos, p.radius, p.mu, F, r0, r1)[:, :3]

    for si, sj in sym_pair_table(nsb, world, rank):
        add(*block(si, sj))  # forward
        if si != sj:
            add(*block(sj, si))  # reverse
    t = torch.from_numpy(limbs.reshape(-1).copy())
    dist.all_reduce(t)  # exact int64 sum
    L = t.numpy().reshape(npad, 3, 3)[:n]
    # carry-normalise and convert (rpy.cu fx_value), exact to one rounding
    U = np.zeros((n, 3))
    for i in range(n):
        for c in range(3):
            X = int(L[i, c, 0]) + (int(L[i, c, 1]) << 43) + (int(L[i, c, 2]) << 86)
            U[i, c] = float(X) * 2.0 ** (-s)
    np.save(os.path.join(outdir, f"Usym_w{world}_r{rank}.npy"), U)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,n", [("C5", 1400), ("C2", 1900)])
def test_gloo_symmetric_rpy_decomposition(tmp_path, name, n):
    """The default multi-GPU RPY split (symmetric super-block pairs, cyclic-half table per rank,
    fixed-point limbs, int64 all-reduce): every rank's U equals the full oracle apply to rounding,
    and is BITWISE the same for world 1, 2 and 3 (integer sums are order-free)."""
    from paper_1909_06623_b200 import sym_pair_table
    npad = -(-n // SB) * SB
    nsb = npad // SB
    for world in (1, 2, 3):  # the tables tile every unordered super-block pair exactly once
        allp = np.concatenate([sym_pair_table(nsb, world, r) for r in range(world)])
        key = {(min(a, b), max(a, b)) for a, b in allp}
        assert len(allp) == len(key) == nsb * (nsb + 1) // 2
    res = {}
    for world in (1, 2, 3):
        mp.spawn(_sym_rank_main, args=(world, _free_port(), name, n, str(tmp_path)), nprocs=world, join=True)
        Us = [np.load(tmp_path / f"Usym_w{world}_r{r}.npy") for r in range(world)]
        for u in Us[1:]:
            np.testing.assert_array_equal(u, Us[0])
        res[world] = Us[0]
    np.testing.assert_array_equal(res[2], res[1])
    np.testing.assert_array_equal(res[3], res[1])
    p = make_problem(name, n=n)
    rng = np.random.default_rng(3)
    FT = np.zeros((n, 6))
    FT[:, :3] = rng.normal(size=(n, 3)) * 10.0 ** rng.uniform(-3, 3, size=(n, 1))
    ref = oracle.rpy_apply(p.pos, p.radius, p.mu, FT)[:, :3]
    assert np.linalg.norm(res[1] - ref) / np.linalg.norm(ref) < 1e-13
