"""ORACLE — plain CPU reference of the SCALE-TRACK particle step (arXiv 2603.26691).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It never imports the product package ``paper_2603_26691_b200`` and
shares no code with it (its C core is ``oracle/st_oracle.c``).

``Sim`` drives the C core the way a user drives ``st_*`` (include/scaletrack.h):
inject -> set fluid field -> advance(dt, nsteps) -> get sources, with

* the per-particle step of SURVEY §8(c1) / DESIGN.md §4 (C core, fp32 or fp64);
* the rebin rule C-15: after the last sub-step of every K-th ``advance`` call the
  store is stable-sorted by the bin key (chunk id, cell within the chunk)
  (``orc_bin_key_*`` + ``orc_stable_order``, a counting sort);
* the far-tail rule C-15b: at a rebin of a store that is already
  binned (no injection since its last rebin) with 8^3-cell chunks, a particle whose
  cell is more than one cell (per axis, periodic-aware) from the cell of its home bin
  (the bin it was sorted into at the previous rebin) is "far"; the sort key is then
  (bin key, far), i.e. within every bin the near particles in their prior order,
  then the far ones in their prior order (arrivals from other ranks after the kept,
  C-16).  At K = 1 in a multi-rank job a far particle whose cell is owned by another
  rank makes every rank take the plain sort;
* the R-rank emulation rule C-16: rank r owns chunk planes
  [floor(r*NCz/R), floor((r+1)*NCz/R)); at a rebin every rank keeps its own
  particles in order, appends arrivals in ascending source rank (each in the
  sender's order), then stable-sorts by bin key; M[src][dst] counts movers.
* source readout C-13: S = acc / (V_cell * T_acc) in N/m^3, acc in float64.

Parity status: every function here is pinned by tests/test_oracle_pins.py (the
C-15b rule by a pure-Python brute force, P-9b) except where DESIGN.md §5 says "parity
unpinned" (trajectory values in a non-uniform field beyond the invariants of pin P-10).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle_st.so")

BC_PERIODIC, BC_REFLECT = 0, 1
DRAG_STOKES, DRAG_SCHILLER_NAUMANN = 0, 1
INT_EXPONENTIAL, INT_SEMI_IMPLICIT = 0, 1
ONE_WAY, TWO_WAY = 0, 1
ERR_CFL = 5


class Params(ctypes.Structure):
    """Mirror of ``orc_params`` in oracle/st_oracle.c."""

    _fields_ = [
        ("dims", ctypes.c_int32 * 3),
        ("origin", ctypes.c_double * 3),
        ("cell_size", ctypes.c_double * 3),
        ("chunk_cells", ctypes.c_int32),
        ("bc", ctypes.c_int32 * 3),
        ("rho_f", ctypes.c_double),
        ("nu_f", ctypes.c_double),
        ("rho_p", ctypes.c_double),
        ("gravity", ctypes.c_double * 3),
        ("drag_law", ctypes.c_int32),
        ("integrator", ctypes.c_int32),
        ("coupling", ctypes.c_int32),
    ]


_lib = None


def build(quiet: bool = True) -> str:
    """Compile the oracle core with gcc (plain C, no FMA contraction)."""
    src = os.path.join(_HERE, "st_oracle.c")
    cmd = (f"gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared "
           f"-o {LIB_PATH} {src} -lm")
    rc = os.system(cmd + (" >/dev/null 2>&1" if quiet else ""))
    if rc != 0:
        raise RuntimeError(f"oracle build failed: {cmd}")
    return LIB_PATH


def lib():
    """Load (building if needed) the oracle shared library."""
    global _lib
    if _lib is not None:
        return _lib
    src = os.path.join(_HERE, "st_oracle.c")
    inc = os.path.join(_HERE, "st_oracle_step.inc")
    if (not os.path.exists(LIB_PATH)
            or os.path.getmtime(LIB_PATH) < max(os.path.getmtime(src), os.path.getmtime(inc))):
        build()
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER(Params)
    vp = ctypes.c_void_p
    for sfx in ("f32", "f64"):
        real = ctypes.c_float if sfx == "f32" else ctypes.c_double
        f = getattr(L, f"orc_advance_{sfx}")
        f.argtypes = [P, ctypes.c_int64, vp, vp, vp, vp, vp, ctypes.c_double, ctypes.c_int, vp]
        f.restype = ctypes.c_int
        f = getattr(L, f"orc_locate_{sfx}")
        f.argtypes = [P, ctypes.c_int64, vp, vp, vp]
        f.restype = ctypes.c_int
        f = getattr(L, f"orc_interpolate_{sfx}")
        f.argtypes = [P, ctypes.c_int64, vp, vp, vp]
        f.restype = ctypes.c_int
        f = getattr(L, f"orc_bin_key_{sfx}")
        f.argtypes = [P, ctypes.c_int64, vp, vp]
        f.restype = ctypes.c_int
        f = getattr(L, f"orc_drag_factor_{sfx}")
        f.argtypes = [ctypes.c_int, real]
        f.restype = real
    L.orc_stable_order.argtypes = [ctypes.c_int64, vp, ctypes.c_int64, vp, vp]
    L.orc_stable_order.restype = ctypes.c_int
    _lib = L
    return L


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def drag_factor(Re: float, law: int = DRAG_SCHILLER_NAUMANN, precision: str = "f64") -> float:
    """f(Re) = Cd*Re/24 of the oracle core (C-2)."""
    return float(getattr(lib(), f"orc_drag_factor_{precision}")(law, Re))


def stable_order(key: np.ndarray, nkeys: int) -> tuple[np.ndarray, np.ndarray]:
    """C-15: permutation of a stable counting sort by key, and the CSR offsets."""
    key = np.ascontiguousarray(key, dtype=np.int64)
    perm = np.empty(key.size, dtype=np.int64)
    off = np.empty(nkeys + 1, dtype=np.int64)
    rc = lib().orc_stable_order(key.size, _ptr(key), nkeys, _ptr(perm), _ptr(off))
    if rc != 0:
        raise ValueError(f"orc_stable_order failed ({rc})")
    return perm, off


@dataclass
class Mesh:
    dims: tuple
    origin: tuple = (0.0, 0.0, 0.0)
    cell_size: tuple = (1.0, 1.0, 1.0)
    chunk_cells: int = 8
    bc: tuple = (BC_PERIODIC, BC_PERIODIC, BC_PERIODIC)

    @property
    def ncell(self) -> int:
        return int(self.dims[0]) * int(self.dims[1]) * int(self.dims[2])

    @property
    def nchunk(self) -> tuple:
        c = self.chunk_cells
        return tuple((int(n) + c - 1) // c for n in self.dims)

    @property
    def n_chunks(self) -> int:
        a, b, c = self.nchunk
        return a * b * c

    @property
    def n_bins(self) -> int:
        return self.n_chunks * self.chunk_cells ** 3

    @property
    def cell_volume(self) -> float:
        return float(self.cell_size[0]) * float(self.cell_size[1]) * float(self.cell_size[2])


@dataclass
class Physics:
    rho_f: float = 1.2
    nu_f: float = 1.5e-5
    rho_p: float = 1000.0
    gravity: tuple = (0.0, 0.0, 0.0)
    drag_law: int = DRAG_SCHILLER_NAUMANN
    integrator: int = INT_EXPONENTIAL
    coupling: int = TWO_WAY


def make_params(mesh: Mesh, phys: Physics) -> Params:
    p = Params()
    for a in range(3):
        p.dims[a] = int(mesh.dims[a])
        p.origin[a] = float(mesh.origin[a])
        p.cell_size[a] = float(mesh.cell_size[a])
        p.bc[a] = int(mesh.bc[a])
        p.gravity[a] = float(phys.gravity[a])
    p.chunk_cells = int(mesh.chunk_cells)
    p.rho_f, p.nu_f, p.rho_p = float(phys.rho_f), float(phys.nu_f), float(phys.rho_p)
    p.drag_law, p.integrator, p.coupling = int(phys.drag_law), int(phys.integrator), int(phys.coupling)
    return p


@dataclass
class _Store:
    x: np.ndarray
    u: np.ndarray
    d: np.ndarray
    w: np.ndarray
    id: np.ndarray

    @property
    def n(self) -> int:
        return int(self.d.size)


def _empty_store(real) -> _Store:
    return _Store(np.zeros((3, 0), real), np.zeros((3, 0), real), np.zeros(0, real),
                  np.zeros(0, real), np.zeros(0, np.uint64))


@dataclass
class Sim:
    """One job of ``nranks`` logical ranks over one global mesh (C-16 emulation)."""

    mesh: Mesh
    phys: Physics = field(default_factory=Physics)
    rebin_interval: int = 1
    precision: str = "f32"
    nranks: int = 1
    plane_split: tuple | None = None   # C-16b: nranks+1 chunk-plane boundaries (None: equal split)

    def __post_init__(self):
        if self.precision not in ("f32", "f64"):
            raise ValueError("precision must be 'f32' or 'f64'")
        if self.mesh.nchunk[2] < self.nranks:
            raise ValueError("need at least one chunk plane per rank")
        self.real = np.float32 if self.precision == "f32" else np.float64
        self.params = make_params(self.mesh, self.phys)
        self._lib = lib()
        self.stores = [_empty_store(self.real) for _ in range(self.nranks)]
        self.field = None
        self.acc = np.zeros((3, self.mesh.ncell), np.float64)
        self.T_acc = 0.0
        self.calls = 0
        self.next_id = [0] * self.nranks
        self.M = np.zeros((self.nranks, self.nranks), np.int64)
        self.last_status = 0
        self.home = [None] * self.nranks    # C-15b: home bin key per particle (None: not binned)
        self.last_far = 0

    # ---- geometry (C-6, C-14, C-16) ----
    def plane_range(self, r: int) -> tuple:
        if self.plane_split is not None:
            return int(self.plane_split[r]), int(self.plane_split[r + 1])
        ncz = self.mesh.nchunk[2]
        return (r * ncz) // self.nranks, ((r + 1) * ncz) // self.nranks

    def owner_of_chunk(self, chunk: np.ndarray) -> np.ndarray:
        ncx, ncy, _ = self.mesh.nchunk
        kz = chunk // (ncx * ncy)
        own = np.full(chunk.shape, -1, np.int64)
        for r in range(self.nranks):
            lo, hi = self.plane_range(r)
            own[(kz >= lo) & (kz < hi)] = r
        return own

    def locate(self, x: np.ndarray):
        x = np.ascontiguousarray(x, dtype=self.real)
        n = x.shape[1]
        cell = np.empty(n, np.int32)
        chunk = np.empty(n, np.int32)
        getattr(self._lib, f"orc_locate_{self.precision}")(self.params, n, _ptr(x), _ptr(cell), _ptr(chunk))
        return cell, chunk

    def bin_key(self, x: np.ndarray) -> np.ndarray:
        """C-15 bin key = chunk * cc^3 + cell-within-chunk of each position."""
        x = np.ascontiguousarray(x, dtype=self.real)
        key = np.empty(x.shape[1], np.int64)
        getattr(self._lib, f"orc_bin_key_{self.precision}")(self.params, x.shape[1], _ptr(x), _ptr(key))
        return key

    def interpolate(self, x: np.ndarray, F: np.ndarray | None = None) -> np.ndarray:
        F = self.field if F is None else np.ascontiguousarray(F, dtype=self.real)
        x = np.ascontiguousarray(x, dtype=self.real)
        out = np.empty_like(x)
        getattr(self._lib, f"orc_interpolate_{self.precision}")(self.params, x.shape[1], _ptr(x), _ptr(F), _ptr(out))
        return out

    # ---- st_* mirror ----
    def set_fluid_field(self, F: np.ndarray):
        nx, ny, nz = self.mesh.dims
        F = np.ascontiguousarray(F, dtype=self.real).reshape(3, nz, ny, nx)
        self.field = F

    def inject(self, x, u, d, w=None, ids=None, rank: int = 0):
        x = np.asarray(x, self.real).reshape(3, -1)
        n = x.shape[1]
        u = np.asarray(u, self.real).reshape(3, n)
        d = np.asarray(d, self.real).reshape(n)
        w = np.ones(n, self.real) if w is None else np.asarray(w, self.real).reshape(n)
        if ids is None:
            ids = (np.uint64(rank) << np.uint64(40)) + np.arange(self.next_id[rank], self.next_id[rank] + n, dtype=np.uint64)
            self.next_id[rank] += n
        ids = np.asarray(ids, np.uint64).reshape(n)
        lo = np.array([self.real(o) for o in self.mesh.origin], self.real)
        hi = np.array([self.real(o + n_ * h) for o, n_, h in zip(self.mesh.origin, self.mesh.dims, self.mesh.cell_size)], self.real)
        if not (np.all(x >= lo[:, None]) and np.all(x <= hi[:, None])):
            raise ValueError("out of domain")
        s = self.stores[rank]
        # an injection leaves the store unbinned (every rank of a multi-rank job: the
        # call is collective); the next rebin is the plain stable sort (C-15b)
        if self.nranks > 1:
            self.home = [None] * self.nranks
        elif n > 0:
            self.home[rank] = None
        self.stores[rank] = _Store(np.concatenate([s.x, x], 1), np.concatenate([s.u, u], 1),
                                   np.concatenate([s.d, d]), np.concatenate([s.w, w]),
                                   np.concatenate([s.id, ids]))

    def advance(self, dt: float, nsteps: int = 1) -> int:
        if self.field is None:
            raise RuntimeError("advance before set_fluid_field")
        status = 0
        fn = getattr(self._lib, f"orc_advance_{self.precision}")
        for s in self.stores:
            if s.n == 0:
                continue
            x = np.ascontiguousarray(s.x)
            u = np.ascontiguousarray(s.u)
            rc = fn(self.params, s.n, _ptr(x), _ptr(u), _ptr(s.d), _ptr(s.w), _ptr(self.field),
                    float(dt), int(nsteps), _ptr(self.acc))
            s.x, s.u = x, u
            status = status or rc
        self.T_acc += nsteps * dt
        self.calls += 1
        if self.calls % self.rebin_interval == 0:
            self.rebin()
        self.last_status = status
        return status

    def home_cell(self, key: np.ndarray) -> np.ndarray:
        """Cell (x, y, z) of a bin key (C-15: chunk * cc^3 + (lz*cc + ly)*cc + lx)."""
        cc = int(self.mesh.chunk_cells)
        ncx, ncy, _ = self.mesh.nchunk
        key = np.asarray(key, np.int64)
        chunk, local = key // cc ** 3, key % cc ** 3
        kx, ky, kz = chunk % ncx, (chunk // ncx) % ncy, chunk // (ncx * ncy)
        lx, ly, lz = local % cc, (local // cc) % cc, local // (cc * cc)
        return np.stack([kx * cc + lx, ky * cc + ly, kz * cc + lz])

    def far_mask(self, home_key: np.ndarray, x: np.ndarray) -> np.ndarray:
        """C-15b: the particle's current cell is more than one cell from its home bin's
        cell along some axis (periodic axes: the shorter way round when n >= 3)."""
        nx, ny, _ = self.mesh.dims
        cell, _ = self.locate(x)
        cell = cell.astype(np.int64)
        cur = np.stack([cell % nx, (cell // nx) % ny, cell // (nx * ny)])
        hc = self.home_cell(home_key)
        far = np.zeros(cell.shape, bool)
        for a in range(3):
            n = int(self.mesh.dims[a])
            d = cur[a] - hc[a]
            if self.mesh.bc[a] == BC_PERIODIC and n >= 3:
                d = np.where(d == n - 1, -1, np.where(d == -(n - 1), 1, d))
            far |= np.abs(d) > 1
        return far

    def rebin(self):
        """C-15 / C-15b / C-16: migrate to owners, then stable sort on every rank by the
        bin key (plain), or by (bin key, far) when the store was binned (C-15b)."""
        R = self.nranks
        M = np.zeros((R, R), np.int64)
        parts = [[None] * R for _ in range(R)]   # parts[src][dst] = index array in src order
        owners, fars = [], []
        for src, s in enumerate(self.stores):
            _, chunk = self.locate(s.x)
            own = self.owner_of_chunk(chunk.astype(np.int64))
            owners.append(own)
            for dst in range(R):
                idx = np.nonzero(own == dst)[0]
                parts[src][dst] = idx
                M[src, dst] = idx.size
        # C-15b applies when every rank's store is binned; a far particle that changes rank
        # is placed in the receiver's far tail when the rebin's counts come from the
        # in-place step of the call that made it due (K >= 2); at K = 1 (counts from a
        # separate pass over the store) it makes every rank take the plain sort
        fused = int(self.mesh.chunk_cells) == 8 and all(h is not None for h in self.home)
        if fused:
            for src, s in enumerate(self.stores):
                f = self.far_mask(self.home[src], s.x) if s.n else np.zeros(0, bool)
                fars.append(f)
                if self.rebin_interval == 1 and np.any(f & (owners[src] != src)):
                    fused = False
        self.last_far = int(sum(int(f.sum()) for f in fars)) if fused else 0
        new, homes = [], []
        for dst in range(R):
            order = [dst] + [src for src in range(R) if src != dst]   # kept first, then arrivals by source rank
            xs, us, ds, ws, ids, fs = [], [], [], [], [], []
            for src in order:
                s, idx = self.stores[src], parts[src][dst]
                xs.append(s.x[:, idx]); us.append(s.u[:, idx]); ds.append(s.d[idx])
                ws.append(s.w[idx]); ids.append(s.id[idx])
                fs.append(fars[src][idx] if fused else np.zeros(idx.size, bool))
            st = _Store(np.concatenate(xs, 1), np.concatenate(us, 1), np.concatenate(ds),
                        np.concatenate(ws), np.concatenate(ids))
            key = self.bin_key(st.x)
            far = np.concatenate(fs)
            perm, _ = stable_order(2 * key + far.astype(np.int64), 2 * self.mesh.n_bins)
            new.append(_Store(np.ascontiguousarray(st.x[:, perm]), np.ascontiguousarray(st.u[:, perm]),
                              st.d[perm].copy(), st.w[perm].copy(), st.id[perm].copy()))
            homes.append(key[perm])
        self.stores = new
        self.home = homes
        self.M = M

    def get_sources(self):
        """C-13: S = acc/(V_cell*T_acc) [N/m^3] on the global mesh, then reset."""
        nx, ny, nz = self.mesh.dims
        T = self.T_acc
        S = np.zeros((3, nz, ny, nx), np.float64) if T == 0 else (self.acc / (self.mesh.cell_volume * T)).reshape(3, nz, ny, nx)
        self.acc = np.zeros_like(self.acc)
        self.T_acc = 0.0
        return S, T

    def particles(self, rank: int = 0) -> dict:
        s = self.stores[rank]
        cell, chunk = self.locate(s.x)
        return dict(x=s.x.copy(), u=s.u.copy(), d=s.d.copy(), w=s.w.copy(), id=s.id.copy(),
                    cell=cell, chunk=chunk)

    @property
    def n_total(self) -> int:
        return sum(s.n for s in self.stores)


def particle_mass(d, rho_p):
    """m_p = (pi/6) rho_p d^3 (C-18) — plain float64 helper for harness checks."""
    return math.pi / 6.0 * rho_p * d ** 3
