"""Python face of the C-ABI (include/scaletrack.h): same names, marshalling only.

Arrays may be numpy arrays (host) or torch tensors (host or CUDA); the library
detects the pointer kind.  Every step of the particle path runs in the CUDA
kernels of libscaletrack.so — nothing here computes.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


def _ptr(a):
    """Raw address of a contiguous numpy array or torch tensor (or None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


def _numel(a) -> int:
    if a is None:
        return 0
    return int(a.size) if isinstance(a, np.ndarray) else int(a.numel())


def _need(a, n: int, what: str):
    """The C side copies fixed sizes: a wrong shape would read or write out of bounds."""
    if a is not None and _numel(a) != n:
        raise ValueError(f"{what}: expected {n} elements, got {_numel(a)}")


def _default_stream(device: int):
    """torch's current stream on `device` (None for the legacy default stream, which the
    library orders against by creating a blocking stream of its own)."""
    try:
        import torch
        if torch.cuda.is_available():
            h = torch.cuda.current_stream(device).cuda_stream
            return h or None
    except Exception:
        pass
    return None


def _as_f32(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=np.float32)
    import torch
    return a.to(torch.float32).contiguous()


@dataclass
class Config:
    """Python mirror of st_config (defaults = st_config_default)."""

    dims: tuple = (16, 16, 16)
    origin: tuple = (0.0, 0.0, 0.0)
    cell_size: tuple = (1 / 16, 1 / 16, 1 / 16)
    chunk_cells: int = 8
    bc: tuple = (N.BC_PERIODIC,) * 3
    rho_f: float = 1.2
    nu_f: float = 1.5e-5
    rho_p: float = 1000.0
    gravity: tuple = (0.0, 0.0, 0.0)
    drag_law: int = N.DRAG_SCHILLER_NAUMANN
    integrator: int = N.INT_EXPONENTIAL
    coupling: int = N.TWO_WAY
    rebin_interval: int = 1
    capacity: int = 1_000_000
    device: int = 0
    rank: int = 0
    nranks: int = 1
    decomposition: int = 0       # N.DECOMP_SLAB | N.DECOMP_SHARDED
    slab_planes: tuple | None = None   # nranks+1 chunk-plane boundaries (plan_partition), None = equal

    def to_c(self, stream=None, unique_id: bytes | None = None) -> N.StConfig:
        c = N.StConfig()
        N.load().st_config_default(ctypes.byref(c))
        for a in range(3):
            c.dims[a] = int(self.dims[a])
            c.origin[a] = float(self.origin[a])
            c.cell_size[a] = float(self.cell_size[a])
            c.bc[a] = int(self.bc[a])
            c.gravity[a] = float(self.gravity[a])
        c.chunk_cells = int(self.chunk_cells)
        c.rho_f, c.nu_f, c.rho_p = float(self.rho_f), float(self.nu_f), float(self.rho_p)
        c.drag_law, c.integrator, c.coupling = int(self.drag_law), int(self.integrator), int(self.coupling)
        c.rebin_interval = int(self.rebin_interval)
        c.capacity = int(self.capacity)
        c.device = int(self.device)
        c.stream = stream
        c.rank, c.nranks = int(self.rank), int(self.nranks)
        c.decomposition = int(self.decomposition)
        c.nccl_unique_id = None
        if self.slab_planes is not None:
            arr = (ctypes.c_int32 * len(self.slab_planes))(*[int(v) for v in self.slab_planes])
            c._keep_slab_planes = arr   # alive as long as the struct
            c.slab_planes = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int32))
        return c

    @property
    def ncell(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])


def plan_layout(cfg: Config) -> N.StLayout:
    """Host-only layout of cfg.rank (st_plan_layout): no GPU needed."""
    lib = N.load()
    o = N.StLayout()
    c = cfg.to_c()
    if cfg.nranks > 1:
        c.nccl_unique_id = 1   # only checked for non-NULL by the validator
    rc = lib.st_plan_layout(ctypes.byref(c), ctypes.byref(o))
    if rc:
        raise N.StError(rc, lib.st_last_error(None).decode())
    return o


def plan_partition(cfg: Config, plane_counts) -> tuple:
    """st_plan_partition: count-balanced slab boundaries (chunk planes) for cfg.nranks
    ranks from the particle count of every chunk plane.  Host-only."""
    lib = N.load()
    c = cfg.to_c()
    counts = np.ascontiguousarray(plane_counts, dtype=np.int64)
    out = np.empty(int(cfg.nranks) + 1, np.int32)
    rc = lib.st_plan_partition(ctypes.byref(c), counts.ctypes.data, out.ctypes.data)
    if rc:
        raise N.StError(rc, lib.st_last_error(None).decode())
    return tuple(int(v) for v in out)


def hilbert_index(order: int, xyz) -> np.ndarray:
    """st_hilbert_index: 3-D Hilbert index of integer cells xyz [n][3] on a 2^order cube."""
    lib = N.load()
    xyz = np.ascontiguousarray(xyz, dtype=np.int32).reshape(-1, 3)
    out = np.empty(xyz.shape[0], np.uint64)
    rc = lib.st_hilbert_index(int(order), xyz.shape[0], xyz.ctypes.data, out.ctypes.data)
    if rc:
        raise N.StError(rc, "st_hilbert_index: coordinate out of range or bad order")
    return out


def plan_hilbert(cfg: Config, chunk_counts) -> np.ndarray:
    """st_plan_hilbert: owner rank of every chunk, contiguous along the Hilbert curve of the
    chunk coordinates and balanced by chunk_counts.  Host-only."""
    lib = N.load()
    c = cfg.to_c()
    counts = np.ascontiguousarray(chunk_counts, dtype=np.int64)
    out = np.empty(counts.size, np.int32)
    rc = lib.st_plan_hilbert(ctypes.byref(c), counts.ctypes.data, out.ctypes.data)
    if rc:
        raise N.StError(rc, "st_plan_hilbert failed")
    return out


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = N.load().st_nccl_unique_id(buf)
    if rc:
        raise N.StError(rc, "ncclGetUniqueId failed")
    return buf.raw


class ScaleTrack:
    """One st_ctx: the particle store, fields and sources of one rank / GPU."""

    def __init__(self, cfg: Config, stream=None, unique_id: bytes | None = None):
        self.lib = N.load()
        self.cfg = cfg
        if stream is None:
            stream = _default_stream(int(cfg.device))
        c = cfg.to_c(stream=stream)
        self._uid = None
        if unique_id is not None:
            self._uid = ctypes.create_string_buffer(unique_id, 128)
            c.nccl_unique_id = ctypes.cast(self._uid, ctypes.c_void_p)
        h = ctypes.c_void_p()
        rc = self.lib.st_init(ctypes.byref(c), ctypes.byref(h))
        if rc:
            raise N.StError(rc, self.lib.st_last_error(None).decode())
        self.h = h
        self.layout = self.get_layout()

    # -- lifecycle --
    def close(self):
        if getattr(self, "h", None):
            self.lib.st_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc:
            raise N.StError(rc, self.lib.st_last_error(self.h).decode())

    # -- st_* --
    def _owned_cells(self) -> int:
        nx, ny, _ = self.cfg.dims
        return int(nx) * int(ny) * int(self.layout.z1 - self.layout.z0)

    def set_fluid_field(self, u):
        u = _as_f32(u)
        _need(u, 3 * self._owned_cells(), "set_fluid_field u [3][z1-z0][ny][nx]")
        self._check(self.lib.st_set_fluid_field(self.h, _ptr(u)))
        self._keep = u   # device inputs stay alive until stream-ordered consumption

    def inject(self, x, u, d, w=None, ids=None):
        x, u, d, w = _as_f32(x), _as_f32(u), _as_f32(d), _as_f32(w)
        n = int(d.shape[0])
        if ids is not None and isinstance(ids, np.ndarray):
            ids = np.ascontiguousarray(ids, dtype=np.uint64)
        _need(x, 3 * n, "inject x [3][n]")
        _need(u, 3 * n, "inject u [3][n]")
        _need(w, n, "inject w [n]")
        _need(ids, n, "inject ids [n]")
        self._check(self.lib.st_inject(self.h, n, _ptr(x), _ptr(u), _ptr(d), _ptr(w), _ptr(ids)))

    def advance(self, dt: float, nsteps: int = 1):
        self._check(self.lib.st_advance(self.h, float(dt), int(nsteps)))

    def get_sources(self, out=None):
        """S [3][z1-z0][ny][nx] fp32 (N/m^3) and the interval T_acc."""
        if out is None:
            nx, ny, _ = self.cfg.dims
            out = np.empty((3, self.layout.z1 - self.layout.z0, ny, nx), np.float32)
        _need(out, 3 * self._owned_cells(), "get_sources out [3][z1-z0][ny][nx]")
        T = ctypes.c_double()
        self._check(self.lib.st_get_sources(self.h, _ptr(out), ctypes.byref(T)))
        return out, T.value

    def request_sources(self):
        self._check(self.lib.st_request_sources(self.h))

    def wait_sources(self, out=None):
        if out is None:
            nx, ny, _ = self.cfg.dims
            out = np.empty((3, self.layout.z1 - self.layout.z0, ny, nx), np.float32)
        _need(out, 3 * self._owned_cells(), "wait_sources out [3][z1-z0][ny][nx]")
        T = ctypes.c_double()
        self._check(self.lib.st_wait_sources(self.h, _ptr(out), ctypes.byref(T)))
        return out, T.value

    def count(self) -> int:
        n = ctypes.c_int64()
        self._check(self.lib.st_get_count(self.h, ctypes.byref(n)))
        return n.value

    def get_particles(self) -> dict:
        n = self.count()
        x = np.empty((3, n), np.float32)
        u = np.empty((3, n), np.float32)
        d = np.empty(n, np.float32)
        w = np.empty(n, np.float32)
        ids = np.empty(n, np.uint64)
        cell = np.empty(n, np.int32)
        chunk = np.empty(n, np.int32)
        no = ctypes.c_int64()
        self._check(self.lib.st_get_particles(self.h, n, ctypes.byref(no), _ptr(x), _ptr(u), _ptr(d), _ptr(w),
                                              _ptr(ids), _ptr(cell), _ptr(chunk)))
        return dict(x=x, u=u, d=d, w=w, id=ids, cell=cell, chunk=chunk)

    def locate(self, x):
        x = _as_f32(x)
        n = int(x.shape[1])
        _need(x, 3 * n, "locate x [3][n]")
        cell = np.empty(n, np.int32)
        chunk = np.empty(n, np.int32)
        self._check(self.lib.st_locate(self.h, n, _ptr(x), _ptr(cell), _ptr(chunk)))
        return cell, chunk

    def migration_counts(self) -> np.ndarray:
        row = np.zeros(self.cfg.nranks, np.int64)
        self._check(self.lib.st_get_migration_counts(self.h, _ptr(row)))
        return row

    def get_layout(self) -> N.StLayout:
        o = N.StLayout()
        self._check(self.lib.st_get_layout(self.h, ctypes.byref(o)))
        return o

    def stats(self) -> dict:
        o = N.StStats()
        self._check(self.lib.st_get_stats(self.h, ctypes.byref(o)))
        return {k: getattr(o, k) for k, _ in N.StStats._fields_}

    def sync(self):
        self._check(self.lib.st_sync(self.h))

    def rebalance(self, tolerance: float = 0.05):
        """st_rebalance (collective, ST_DECOMP_SHARDED): (sent, received) particles."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self._check(self.lib.st_rebalance(self.h, float(tolerance), ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def trace(self, k: int) -> np.ndarray:
        """st_trace: [k-th copy in begin, end, k-th step begin, end, k-th readout begin,
        end] in ms since st_init (-1: not recorded / too old)."""
        t = np.empty(6, np.float64)
        self._check(self.lib.st_trace(self.h, int(k), t.ctypes.data))
        return t

    def last_timings(self):
        a, r = ctypes.c_float(), ctypes.c_float()
        self._check(self.lib.st_last_timings(self.h, ctypes.byref(a), ctypes.byref(r)))
        return a.value, r.value


class Extrapolator:
    """st_ec_*: the extrapolator-corrector of the asynchronous coupling (SURVEY §8(f1),
    PAPER.md §2.4 Eq. 14-16) over source fields of `n` values.  Marshalling only: the
    estimator runs in libscaletrack.so (csrc/st_ec.cu)."""

    MODES = {"zero": N.EC_ZERO, "constant": N.EC_CONSTANT, "linear": N.EC_LINEAR}

    def __init__(self, mode: str, n: int, max_backlog: int = 8, device: int = 0, stream=None):
        self.lib = N.load()
        c = N.StEcConfig()
        c.abi_version = N.ST_ABI_VERSION
        c.mode = self.MODES[mode]
        c.n = int(n)
        c.max_backlog = int(max_backlog)
        c.device = int(device)
        c.stream = stream
        h = ctypes.c_void_p()
        rc = self.lib.st_ec_init(ctypes.byref(c), ctypes.byref(h))
        if rc:
            raise N.StError(rc, self.lib.st_ec_last_error(None).decode())
        self.h = h
        self.n = int(n)

    def _check(self, rc: int):
        if rc:
            raise N.StError(rc, self.lib.st_ec_last_error(self.h).decode())

    def step(self, received=None, dt_ratio: float = 1.0, out=None):
        """received: None, or k true fields stacked as [k, n] (numpy or torch, host or
        CUDA), oldest first.  Returns S^n_est as float32 [n] (numpy unless `out`)."""
        k = 0
        if received is not None:
            received = _as_f32(received)
            k = int(received.shape[0]) if received.ndim > 1 else 1
            numel = received.size if isinstance(received, np.ndarray) else received.numel()
            if numel != k * self.n:
                raise ValueError(f"received must hold k*n = {k}*{self.n} values")
        if out is None:
            out = np.empty(self.n, dtype=np.float32)
        _need(out, self.n, "Extrapolator.step out [n]")
        self._check(self.lib.st_ec_step(self.h, k, _ptr(received) if k else None, float(dt_ratio), _ptr(out)))
        return out

    def ledger(self):
        """(Σ true received, Σ emitted, Σ pending) per value (fp64) and their totals."""
        ct, ce, pe = (np.empty(self.n, dtype=np.float64) for _ in range(3))
        tot = np.empty(3, dtype=np.float64)
        self._check(self.lib.st_ec_ledger(self.h, _ptr(ct), _ptr(ce), _ptr(pe), _ptr(tot)))
        return ct, ce, pe, tot

    def backlog(self) -> int:
        b = ctypes.c_int32()
        self._check(self.lib.st_ec_backlog(self.h, ctypes.byref(b)))
        return b.value

    def close(self):
        if getattr(self, "h", None):
            self.lib.st_ec_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class MicroConfig:
    """Python mirror of st_micro_config (defaults = st_micro_config_default, C-30)."""

    dims: tuple = (1, 1, 1)
    origin: tuple = (0.0, 0.0, 0.0)
    cell_size: tuple = (1.0, 1.0, 1.0)
    bc: tuple = (N.BC_REFLECT,) * 3
    rho_f: float = 1.2
    nu_f: float = 1.5e-5
    rho_p: float = 1000.0
    gravity: tuple = (0.0, 0.0, -9.81)
    drag_law: int = N.DRAG_SCHILLER_NAUMANN
    D_v: float = 2.5e-5
    kappa_f: float = 0.025
    cp_p: float = 4186.0
    latent: float = 2.45e6
    nusselt: float = 2.0
    s_vp: float = 1.0
    device: int = 0
    stream: int | None = None
    arithmetic: str = "fp64"     # "fp64" (C-28, default) | "fp32" (C-36)

    def to_c(self) -> N.StMicroConfig:
        c = N.StMicroConfig()
        c.abi_version = N.ST_ABI_VERSION
        for k in range(3):
            c.dims[k], c.origin[k], c.cell_size[k] = int(self.dims[k]), float(self.origin[k]), float(self.cell_size[k])
            c.bc[k], c.gravity[k] = int(self.bc[k]), float(self.gravity[k])
        for f in ("rho_f", "nu_f", "rho_p", "D_v", "kappa_f", "cp_p", "latent", "nusselt", "s_vp"):
            setattr(c, f, float(getattr(self, f)))
        c.drag_law, c.device, c.stream = int(self.drag_law), int(self.device), self.stream
        if self.arithmetic not in ("fp64", "fp32"):
            raise ValueError(f"arithmetic must be 'fp64' or 'fp32', not {self.arithmetic!r}")
        c.arithmetic = N.ARITH_FP32 if self.arithmetic == "fp32" else N.ARITH_FP64
        return c


def micro_advance(cfg: MicroConfig, x, u, d, T, w, F, dt: float, nsteps: int, acc) -> int:
    """st_micro_advance: nsteps droplet sub-steps (PAPER Eq. 7-13) on CUDA
    tensors x, u [3, n], d, T, w [n] (fp32, x/u/d/T updated in place), F [5, nz, ny, nx]
    fp32, acc [5, nz, ny, nx] fp64 (added to).  Returns the number of mass-floor clamps."""
    lib = N.load()
    n = int(d.shape[0])
    ncell = int(cfg.dims[0]) * int(cfg.dims[1]) * int(cfg.dims[2])
    for a, k, what in ((x, 3 * n, "x"), (u, 3 * n, "u"), (T, n, "T"), (w, n, "w"), (F, 5 * ncell, "F"),
                       (acc, 5 * ncell, "acc")):
        _need(a, k, f"micro_advance {what}")
    c = cfg.to_c()
    nc = ctypes.c_int64()
    rc = lib.st_micro_advance(ctypes.byref(c), n, _ptr(x), _ptr(u), _ptr(d), _ptr(T), _ptr(w), _ptr(F),
                              float(dt), int(nsteps), _ptr(acc), ctypes.byref(nc))
    if rc:
        raise N.StError(rc, "st_micro_advance failed")
    return int(nc.value)
