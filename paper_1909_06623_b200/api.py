"""Thin Python binding of the C ABI (same names as include/stokescol.h).

Argument marshalling only: every step of the hot path runs in libstokescol's
CUDA kernels.  Arrays may be torch tensors (CUDA or CPU) or numpy arrays;
CPU arrays are staged by the library itself (host pointers are accepted by
every entry point).  Outputs are allocated as torch CUDA tensors unless the
caller passes buffers.
"""
from __future__ import annotations

import contextlib
import ctypes as C

import numpy as np

from . import _lib

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None


class ScError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_lib.STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def _ptr(a):
    """Data pointer of a contiguous float64/int32 torch tensor or numpy array (None -> NULL)."""
    if a is None:
        return None
    if torch is not None and isinstance(a, torch.Tensor):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    raise TypeError(f"unsupported array type {type(a)}")


def _check_dtype(a, dt):
    if a is None:
        return a
    if torch is not None and isinstance(a, torch.Tensor):
        want = torch.float64 if dt == "f64" else torch.int32
        if a.dtype != want:
            raise TypeError(f"expected {want}, got {a.dtype}")
    elif isinstance(a, np.ndarray):
        want = np.float64 if dt == "f64" else np.int32
        if a.dtype != want:
            raise TypeError(f"expected {want}, got {a.dtype}")
    return a


def _f64(a, shape, what):
    """dtype float64 and the expected shape (None entries: any); None passes through.  The C ABI
    takes plain pointers, so a mis-sized buffer must be caught here."""
    if a is None:
        return None
    _check_dtype(a, "f64")
    got = tuple(a.shape)
    if len(got) != len(shape) or any(w is not None and g != w for g, w in zip(got, shape)):
        raise ValueError(f"{what}: expected shape {shape}, got {got}")
    return a


class Context:
    """One sc_ctx (one GPU).  ``world > 1``: NCCL communicator over ranks."""

    def __init__(self, device: int = 0, stream=None, nccl_id: bytes | None = None, rank: int = 0,
                 world: int = 1):
        self.lib = _lib.load()
        self._h = C.c_void_p()
        s = None
        if stream is not None:
            s = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        if world > 1 or nccl_id is not None:  # (world 1 with an id: a one-rank communicator)
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
            rc = self.lib.sc_create_dist(C.byref(self._h), device, s, idbuf, rank, world)
        else:
            rc = self.lib.sc_create(C.byref(self._h), device, s)
        if rc != 0:
            raise ScError(rc, f"sc_create failed on device {device}")
        self.device = device
        self.n = 0
        self.nc = 0
        self.kind = None
        self._ext = None  # torch view of the library stream (created on first use)

    # ------------------------------------------------------------- plumbing
    def close(self):
        if self._h:
            self.lib.sc_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _rc(self, rc, allow=(0,)):
        if rc not in allow:
            raise ScError(rc, self.lib.sc_last_error(self._h).decode())
        return rc

    @property
    def stream_ptr(self) -> int:
        return self.lib.sc_stream(self._h) or 0

    def torch_stream(self):
        return torch.cuda.ExternalStream(self.stream_ptr, device=self.device)

    @contextlib.contextmanager
    def _ordered(self):
        """Stream ordering across the boundary: the library works on its own stream, the caller's
        tensors are produced and consumed on torch's current stream.  Entry: the library stream
        waits for the caller's stream; exit: the caller's stream waits for the library stream
        (CUDA events only; no host synchronisation)."""
        if torch is None or not torch.cuda.is_available():
            yield
            return
        if self._ext is None:
            self._ext = self.torch_stream()
        cur = torch.cuda.current_stream(self.device)
        same = cur.cuda_stream == self._ext.cuda_stream
        if not same:
            self._ext.wait_stream(cur)
        try:
            yield
        finally:
            if not same:
                cur.wait_stream(self._ext)

    def _dev(self, shape, dtype=None):
        return torch.empty(shape, dtype=dtype or torch.float64, device=f"cuda:{self.device}")

    # ------------------------------------------------------- NEXT row f2
    def set_walls(self, walls):
        """Static planar walls n.x = h (rows (nx, ny, nz, h), unit n into the fluid) for every
        later contact build on this context; wall k appears as body n + k in the constraint
        list (include/stokescol.h sc_set_walls).  walls=None or empty removes them."""
        import numpy as np
        w = np.ascontiguousarray(np.zeros((0, 4)) if walls is None else np.asarray(walls, dtype=np.float64))
        if w.ndim != 2 or w.shape[1] != 4:
            raise ValueError("walls must be k x 4")
        self._rc(self.lib.sc_set_walls(self._h, int(w.shape[0]), w.ctypes.data if w.size else None))
        self._walls = w

    def set_wall_velocities(self, vel):
        """Prescribed velocities (k x 3) of the walls of the last set_walls call (moving
        boundaries): they enter q as -n_k . V_k; time_step advances the planes."""
        v = np.ascontiguousarray(np.asarray(vel, dtype=np.float64).reshape(-1, 3))
        self._rc(self.lib.sc_set_wall_velocities(self._h, int(v.shape[0]), v.ctypes.data if v.size else None))

    def get_walls(self):
        """The current planes (k x 4), moved by time_step for walls with a velocity."""
        k = int(getattr(self, "_walls", np.zeros((0, 4))).shape[0])
        out = np.zeros((max(k, 1), 4))
        self._rc(self.lib.sc_get_walls(self._h, out.ctypes.data))
        return out[:k]

    # --------------------------------------------------- NEXT row f4(ii)
    def set_mobility_model(self, model):
        """"rpy" (BASELINE: translational RPY + self rotation), "rpy6" (full 6N RPY grand
        mobility with the translation-rotation and rotation-rotation pair blocks) or "rpy_fmm"
        (the "rpy" operator by the fast O(N) summation, NEXT row f4(i))."""
        m = {"rpy": 0, "rpy6": 1, "rpy_fmm": 2}[model] if isinstance(model, str) else int(model)
        self._rc(self.lib.sc_set_mobility_model(self._h, m))

    # --------------------------------------------------- NEXT row f4(i)
    def set_fmm_params(self, order=6, leaf_level=0):
        """Order (Chebyshev nodes per dimension: 4, 6 or 8) and leaf level (0: automatic) of the
        fast RPY summation used with set_mobility_model("rpy_fmm")."""
        self._rc(self.lib.sc_set_fmm_params(self._h, int(order), int(leaf_level)))

    def set_fmm_tolerance(self, rel_err) -> int:
        """Pick the lowest fast-summation order whose stated error bar meets rel_err; returns it."""
        o = C.c_int32()
        self._rc(self.lib.sc_set_fmm_tolerance(self._h, float(rel_err), C.byref(o)))
        return int(o.value)

    def set_fmm_compression(self, mode=1):
        """Compressed M2L of the fast summation (one orthonormal basis per level for its M2L
        operators, include/stokescol.h sc_set_fmm_compression): 0 / False off, 1 / True on,
        2 / "auto" (the default: on at orders 6 and 8)."""
        m = 2 if mode == "auto" else int(mode)
        self._rc(self.lib.sc_set_fmm_compression(self._h, m))

    def fmm_info(self) -> dict:
        out = (C.c_int32 * 3)()
        self._rc(self.lib.sc_get_fmm_info(self._h, out))
        info = dict(zip(["order", "leaf_level", "ready"], list(out)))
        c4 = (C.c_int32 * 4)()
        self._rc(self.lib.sc_get_fmm_compression_info(self._h, c4))
        info.update(zip(["compression_mode", "compressed", "rank", "rank_level"], list(c4)))
        return info

    # ------------------------------------------------------------- (a1)
    def build_contacts_spheres(self, pos, radius=None, gap_abs=0.0, gap_rel=0.1) -> int:
        n = int(pos.shape[0])
        nc = C.c_int64()
        _f64(pos, (n, 3), "pos"); _f64(radius, (n,), "radius")
        with self._ordered():
            self._rc(self.lib.sc_build_contacts_spheres(self._h, n, _ptr(_check_dtype(pos, "f64")),
                                                        _ptr(_check_dtype(radius, "f64")), float(gap_abs),
                                                        float(gap_rel), C.byref(nc)))
        self.n, self.nc, self.kind = n, nc.value, "spheres"
        return self.nc

    def build_contacts_rods(self, center, direction, length, b, gap_thresh) -> int:
        n = int(center.shape[0])
        nc = C.c_int64()
        _f64(center, (n, 3), "center"); _f64(direction, (n, 3), "direction"); _f64(length, (n,), "length")
        with self._ordered():
            self._rc(self.lib.sc_build_contacts_rods(self._h, n, _ptr(_check_dtype(center, "f64")),
                                                     _ptr(_check_dtype(direction, "f64")),
                                                     _ptr(_check_dtype(length, "f64")), float(b),
                                                     float(gap_thresh), C.byref(nc)))
        self.n, self.nc, self.kind = n, nc.value, "rods"
        return self.nc

    def get_contacts(self, lever: bool = False):
        nc = self.nc
        ci = self._dev((nc,), torch.int32)
        cj = self._dev((nc,), torch.int32)
        gap = self._dev((nc,))
        nrm = self._dev((nc, 3))
        lev = self._dev((nc, 2, 3)) if lever else None
        with self._ordered():
            self._rc(self.lib.sc_get_contacts(self._h, _ptr(ci), _ptr(cj), _ptr(gap), _ptr(nrm), _ptr(lev)))
        out = {"i": ci, "j": cj, "gap": gap, "normal": nrm}
        if lever:
            out["lever"] = lev
        return out

    # ------------------------------------------------------------- (a2)
    def assemble_D(self):
        with self._ordered():
            self._rc(self.lib.sc_assemble_D(self._h))

    def apply_D(self, gamma, out=None):
        out = self._dev((self.n, 6)) if out is None else out
        _f64(gamma, (self.nc,), "gamma"); _f64(out, (self.n, 6), "out")
        with self._ordered():
            self._rc(self.lib.sc_apply_D(self._h, _ptr(_check_dtype(gamma, "f64")), _ptr(_check_dtype(out, "f64"))))
        return out

    def apply_DT(self, UW, out=None):
        out = self._dev((self.nc,)) if out is None else out
        _f64(UW, (self.n, 6), "UW"); _f64(out, (self.nc,), "out")
        with self._ordered():
            self._rc(self.lib.sc_apply_DT(self._h, _ptr(_check_dtype(UW, "f64")), _ptr(_check_dtype(out, "f64"))))
        return out

    # ------------------------------------------------------------- (a4)
    def mobility_apply(self, FT, mu=1.0, out=None):
        out = self._dev((self.n, 6)) if out is None else out
        _f64(FT, (self.n, 6), "FT"); _f64(out, (self.n, 6), "out")
        with self._ordered():
            self._rc(self.lib.sc_mobility_apply(self._h, float(mu), _ptr(_check_dtype(FT, "f64")),
                                                _ptr(_check_dtype(out, "f64"))))
        return out

    # ------------------------------------------------------------- q, (a6)
    def lcp_q(self, dt, U_nc, out=None):
        out = self._dev((self.nc,)) if out is None else out
        _f64(U_nc, (self.n, 6), "U_nc"); _f64(out, (self.nc,), "out")
        with self._ordered():
            self._rc(self.lib.sc_lcp_q(self._h, float(dt), _ptr(_check_dtype(U_nc, "f64")),
                                       _ptr(_check_dtype(out, "f64"))))
        return out

    def bbpgd_solve(self, mu=1.0, tol=1e-8, max_iter=5000, bb_mode=0, fixed_iters=False, gamma0=None,
                    want_g=True, want_Fc=True, want_Uc=True, out=None, warm_from_previous=False):
        warm = 1 if gamma0 is not None else (2 if warm_from_previous else 0)
        opts = _lib.BbpgdOpts(float(mu), float(tol), int(max_iter), int(bb_mode), int(bool(fixed_iters)), warm)
        out = out or {}
        gamma = out.get("gamma")
        if gamma is None:
            gamma = self._dev((self.nc,))
        if gamma0 is not None:
            gamma.copy_(torch.as_tensor(gamma0, dtype=torch.float64))
        g = out.get("g", self._dev((self.nc,)) if want_g else None)
        Fc = out.get("Fc", self._dev((self.n, 6)) if want_Fc else None)
        Uc = out.get("Uc", self._dev((self.n, 6)) if want_Uc else None)
        st = _lib.BbpgdStats()
        with self._ordered():
            rc = self._rc(self.lib.sc_bbpgd_solve(self._h, C.byref(opts), _ptr(gamma), _ptr(g), _ptr(Fc), _ptr(Uc),
                                                  C.byref(st)), allow=(0, 1))
        return {"gamma": gamma, "g": g, "Fc": Fc, "Uc": Uc, "status": rc, **st.as_dict()}

    def collision_step(self, kind, pos, F_ext, radius=None, direction=None, length=None, b=0.5,
                       gap_abs=0.0, gap_rel=0.1, mu=1.0, dt=0.01, tol=1e-8, max_iter=5000, bb_mode=0,
                       fixed_iters=False, Fc_out=None, Uc_out=None):
        """The whole per-step path in one C call (any pointer may be host or device)."""
        n = int(pos.shape[0])
        _f64(pos, (n, 3), "pos"); _f64(F_ext, (n, 6), "F_ext"); _f64(radius, (n,), "radius")
        _f64(direction, (n, 3), "direction"); _f64(length, (n,), "length")
        prob = _lib.Problem(0 if kind == "spheres" else 1, 0, n, _ptr(pos), _ptr(radius), _ptr(direction),
                            _ptr(length), float(b), float(gap_abs), float(gap_rel), float(mu), float(dt),
                            _ptr(F_ext))
        opts = _lib.BbpgdOpts(float(mu), float(tol), int(max_iter), int(bb_mode), int(bool(fixed_iters)), 0)
        nc = C.c_int64()
        st = _lib.BbpgdStats()
        _f64(Fc_out, (n, 6), "Fc_out"); _f64(Uc_out, (n, 6), "Uc_out")
        with self._ordered():
            rc = self._rc(self.lib.sc_collision_step(self._h, C.byref(prob), C.byref(opts), _ptr(Fc_out),
                                                     _ptr(Uc_out), C.byref(nc), C.byref(st)), allow=(0, 1))
        self.n, self.nc, self.kind = n, nc.value, kind
        return {"status": rc, "nc": nc.value, **st.as_dict()}

    def apgd_solve(self, mu=1.0, tol=1e-8, max_iter=20000):
        """APGD comparison solver on the same CQP (NEXT row f3); stats['bb_breakdowns'] = restarts."""
        opts = _lib.BbpgdOpts(float(mu), float(tol), int(max_iter), 0, 0, 0)
        gamma = self._dev((self.nc,))
        g = self._dev((self.nc,))
        st = _lib.BbpgdStats()
        with self._ordered():
            rc = self._rc(self.lib.sc_apgd_solve(self._h, C.byref(opts), _ptr(gamma), _ptr(g), C.byref(st)),
                          allow=(0, 1))
        return {"gamma": gamma, "g": g, "status": rc, **st.as_dict()}

    def time_step(self, kind, pos, F_ext, radius=None, direction=None, length=None, b=0.5, gap_abs=0.0,
                  gap_rel=0.1, mu=1.0, dt=0.01, tol=1e-8, max_iter=5000, bb_mode=0, quat=None, want_U=True,
                  warm_start=False):
        """One whole time step: returns the next centres (and rod axes),
        updates `quat` (n x 4) in place, and the total velocity U_nc + U_c."""
        n = int(pos.shape[0])
        _f64(pos, (n, 3), "pos"); _f64(F_ext, (n, 6), "F_ext"); _f64(radius, (n,), "radius")
        _f64(direction, (n, 3), "direction"); _f64(length, (n,), "length")
        prob = _lib.Problem(0 if kind == "spheres" else 1, 0, n, _ptr(pos), _ptr(radius), _ptr(direction),
                            _ptr(length), float(b), float(gap_abs), float(gap_rel), float(mu), float(dt),
                            _ptr(F_ext))
        opts = _lib.BbpgdOpts(float(mu), float(tol), int(max_iter), int(bb_mode), 0, 2 if warm_start else 0)
        _f64(quat, (n, 4), "quat")
        pos_out = self._dev((n, 3))
        dir_out = self._dev((n, 3)) if kind == "rods" else None
        U = self._dev((n, 6)) if want_U else None
        nc = C.c_int64()
        st = _lib.BbpgdStats()
        with self._ordered():
            rc = self._rc(self.lib.sc_time_step(self._h, C.byref(prob), C.byref(opts), _ptr(pos_out), _ptr(dir_out),
                                                _ptr(_check_dtype(quat, "f64")), _ptr(U), C.byref(nc), C.byref(st)),
                          allow=(0, 1))
        self.n, self.nc, self.kind = n, nc.value, kind
        return {"pos": pos_out, "dir": dir_out, "U": U, "status": rc, "nc": nc.value, **st.as_dict()}

    def minmap_residual(self, gamma, g) -> float:
        """phi = || min(gamma, g) ||_2 on the GPU."""
        nc = int(gamma.shape[0])
        _f64(gamma, (nc,), "gamma"); _f64(g, (nc,), "g")
        out = np.zeros(1)
        with self._ordered():
            self._rc(self.lib.sc_minmap_residual(self._h, nc, _ptr(gamma), _ptr(g), _ptr(out)))
        return float(out[0])

    # ------------------------------------------------------------- residual trace
    def set_residual_trace(self, capacity: int):
        """Record phi_0, phi_1, ... of the next solves (up to `capacity` values; 0 = off)."""
        self._rc(self.lib.sc_set_residual_trace(self._h, int(capacity)))
        self._trace_cap = int(capacity)

    def residual_trace(self):
        """phi_0, phi_1, ..., phi_iters of the last solve (numpy; empty if tracing is off)."""
        cap = getattr(self, "_trace_cap", 0)
        out = np.zeros(max(cap, 1))
        cnt = C.c_int32()
        self._rc(self.lib.sc_get_residual_trace(self._h, out.ctypes.data, int(cap), C.byref(cnt)))
        return out[:min(cap, cnt.value)].copy()

    def comm_info(self) -> dict:
        """{nranks, rank, device, nccl_version} of this context's communicator."""
        out = (C.c_int32 * 4)()
        self._rc(self.lib.sc_comm_info(self._h, out))
        return dict(zip(["nranks", "rank", "device", "nccl_version"], list(out)))

    # ------------------------------------------------------------- measurement
    def set_timing(self, enable=True):
        self._rc(self.lib.sc_set_timing(self._h, int(bool(enable))))

    def reset_timing(self):
        self._rc(self.lib.sc_reset_timing(self._h))

    def get_timing(self):
        out = {}
        for k, name in enumerate(_lib.K_FAMILIES):
            ms = C.c_double()
            cnt = C.c_int64()
            self._rc(self.lib.sc_get_timing(self._h, k, C.byref(ms), C.byref(cnt)))
            out[name] = (ms.value, cnt.value)
        return out

    def set_emulated_world(self, world: int):
        """Testing hook: run the multi-GPU decomposition of `world` ranks on this one GPU."""
        self._rc(self.lib.sc_set_emulated_world(self._h, int(world)))

    def set_rpy_kernel(self, mode: int):
        """0 automatic, 1 target-row kernel (multi-GPU unit), 2 symmetric pair-tile kernel."""
        self._rc(self.lib.sc_set_rpy_kernel(self._h, int(mode)))

    def launch_count(self) -> int:
        return int(self.lib.sc_launch_count(self._h))


def nccl_unique_id() -> bytes:
    lib = _lib.load()
    buf = C.create_string_buffer(128)
    rc = lib.sc_nccl_unique_id(buf)
    if rc != 0:
        raise ScError(rc, "ncclGetUniqueId failed")
    return buf.raw


def plan_partition(n: int, world: int, rank: int) -> dict:
    """Host-only: the row/chunk partition of a world-sized context (no GPU needed)."""
    lib = _lib.load()
    out = (C.c_int64 * 7)()
    rc = lib.sc_plan_partition(int(n), int(world), int(rank), out)
    if rc != 0:
        raise ScError(rc, "plan_partition: bad arguments")
    keys = ["npad", "rows_per_rank", "row_lo", "row_hi", "chunk_lo", "chunk_hi", "nsplit"]
    return dict(zip(keys, list(out)))


def sym_pair_table(nsb: int, world: int, rank: int) -> np.ndarray:
    """Host-only: the (SI, SJ) super-block pairs rank `rank` of `world` evaluates in the
    symmetric RPY kernel (include/stokescol.h sc_sym_pair_table)."""
    lib = _lib.load()
    cnt = C.c_int64()
    rc = lib.sc_sym_pair_table(int(nsb), int(world), int(rank), None, C.byref(cnt))
    if rc != 0:
        raise ScError(rc, "sym_pair_table: bad arguments")
    out = np.zeros((max(cnt.value, 1), 2), dtype=np.int32)
    rc = lib.sc_sym_pair_table(int(nsb), int(world), int(rank), out.ctypes.data, C.byref(cnt))
    if rc != 0:
        raise ScError(rc, "sym_pair_table: bad arguments")
    return out[:cnt.value]
