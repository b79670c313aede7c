"""Python binding of the C ABI in include/sph.h (ctypes; argument marshalling only).

Every step of the method runs in libsph.so's CUDA kernels.  There is no CPU
fallback: if the library is missing this module raises at import of the
library (``lib()``), and every call raises ``SphError`` on a non-OK status.
PyTorch owns the device memory (SoA fp64 tensors) and provides the stream.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPH_LIB selects another in-tree build of the same library (A/B runs of kernel variants)
LIB_PATH = os.environ.get("SPH_LIB") or os.path.join(_HERE, "libsph.so")

ABI_VERSION = 6
KERNEL_MODES = {"poly": 0, "table": 1, "sin": 2}
EOS = {"linear": 0, "ideal": 1}
STATUS = {0: "SPH_OK", 1: "SPH_ERR_NUMERIC", 2: "SPH_ERR_CONFIG", 3: "SPH_ERR_CAPACITY",
          4: "SPH_ERR_CUDA", 5: "SPH_ERR_COMM", 6: "SPH_ERR_STATE"}
PHASES = ("bbox", "keys", "sort", "permute", "cells", "neighbors", "density", "iad", "momentum",
          "update", "halo", "records")

STATE_FIELDS = ("x", "y", "z", "vx", "vy", "vz", "h", "m", "u", "vhx", "vhy", "vhz", "du_prev")
OUT_FIELDS = ("rho", "omega", "p", "c", "c11", "c12", "c13", "c22", "c23", "c33", "ax", "ay", "az",
              "du", "vsig")
ALL_FIELDS = STATE_FIELDS + OUT_FIELDS


def nccl_unique_id() -> bytes:
    """Rank 0's 128-byte NCCL id (sph_nccl_unique_id); broadcast it to all ranks."""
    buf = C.create_string_buffer(128)
    st = lib().sph_nccl_unique_id(buf, 128)
    if st != 0:
        raise SphError(st, "sph_nccl_unique_id failed (built without NCCL?)")
    return buf.raw


def local_comm_id(nranks: int) -> bytes:
    """128-byte id of a new in-process hub (sph_local_comm_id): pass it as ``unique_id`` to
    ``nranks`` Simulations of this process, one per rank, each driven by its own thread."""
    buf = C.create_string_buffer(128)
    st = lib().sph_local_comm_id(int(nranks), buf, 128)
    if st != 0:
        raise SphError(st, "sph_local_comm_id failed")
    return buf.raw


def decomp_splitters(hist: np.ndarray, G: int) -> np.ndarray:
    """split[G+1]: rank r owns key-prefix bins [split[r], split[r+1]) (host helper of the C ABI)."""
    h = np.ascontiguousarray(hist, dtype=np.int64)
    out = np.zeros(G + 1, dtype=np.int64)
    st = lib().sph_decomp_splitters(h.ctypes.data_as(C.POINTER(C.c_int64)), h.size, G,
                                    out.ctypes.data_as(C.POINTER(C.c_int64)))
    if st != 0:
        raise SphError(st, "sph_decomp_splitters")
    return out


def decomp_owner(split: np.ndarray, b: int) -> int:
    s = np.ascontiguousarray(split, dtype=np.int64)
    return lib().sph_decomp_owner(s.ctypes.data_as(C.POINTER(C.c_int64)), s.size - 1, int(b))


def measure_fp64_peak(stream=None) -> float:
    """Measured FP64 DFMA TFLOP/s of the current GPU (roofline denominator)."""
    import torch
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    v = C.c_double(0.0)
    st = lib().sph_measure_fp64_peak(C.c_void_p(stream), C.byref(v))
    if st != 0:
        raise SphError(st, "sph_measure_fp64_peak failed")
    return v.value


class SphError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Params(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int), ("sinc_n", C.c_double), ("alpha_av", C.c_double),
        ("eos", C.c_int), ("c0", C.c_double), ("rho0", C.c_double), ("gamma", C.c_double),
        ("omega_mode", C.c_int), ("courant", C.c_double), ("dt_growth", C.c_double),
        ("n_target", C.c_double), ("h_min", C.c_double), ("h_max", C.c_double),
        ("u_floor", C.c_double), ("max_neighbors", C.c_int), ("cell_factor", C.c_double),
        ("box_lo", C.c_double * 3), ("box_hi", C.c_double * 3), ("periodic", C.c_int * 3),
        ("rank", C.c_int), ("nranks", C.c_int), ("nccl_unique_id", C.c_void_p),
        ("stream", C.c_void_p),
        ("kernel_mode", C.c_int), ("table_size", C.c_int), ("symmetric", C.c_int),
        ("redecomp_every", C.c_int),
    ]


_P = C.POINTER(C.c_double)


class Particles(C.Structure):
    _fields_ = ([("n", C.c_int64), ("capacity", C.c_int64), ("id", C.POINTER(C.c_int64))] +
                [(k, _P) for k in ("x", "y", "z", "vx", "vy", "vz", "h", "m", "u")] +
                [(k, _P) for k in ("rho", "omega", "p", "c")] +
                [(k, _P) for k in ("c11", "c12", "c13", "c22", "c23", "c33")] +
                [(k, _P) for k in ("ax", "ay", "az", "du", "vsig")] +
                [(k, _P) for k in ("vhx", "vhy", "vhz", "du_prev")])


class Diag(C.Structure):
    _fields_ = ([(k, C.c_int64) for k in ("n_owned", "n_halo", "nbr_total", "nbr_max",
                                          "omega_clamped", "iad_singular", "coincident_pairs",
                                          "u_floored", "h_clamped", "steps", "first_bad_id")] +
                [("dt", C.c_double), ("dt_prev", C.c_double), ("time", C.c_double),
                 ("momentum", C.c_double * 3), ("ang_momentum", C.c_double * 3),
                 ("energy", C.c_double), ("grid", C.c_int * 3)])

    def as_dict(self):
        out = {}
        for k, _ in self._fields_:
            v = getattr(self, k)
            out[k] = list(v) if hasattr(v, "__len__") else v
        return out


_lib = None


def lib():
    """Load libsph.so (fails loudly: there is no CPU path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python __graft_entry__.py` (build) first")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.sph_abi_version.restype = C.c_int
        L.sph_error_string.restype = C.c_char_p
        L.sph_error_string.argtypes = [vp]
        L.sph_init.argtypes = [C.POINTER(Params), C.c_int64, C.POINTER(vp)]
        L.sph_attach.argtypes = [vp, C.POINTER(Particles)]
        for f in ("sph_find_neighbors", "sph_density", "sph_iad", "sph_advance", "sph_destroy"):
            getattr(L, f).argtypes = [vp]
        L.sph_get_neighbors.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int64]
        L.sph_momentum_energy.argtypes = [vp, _P]
        L.sph_step.argtypes = [vp, _P]
        L.sph_upload.argtypes = [vp, C.POINTER(Particles)]
        L.sph_download.argtypes = [vp, C.POINTER(Particles)]
        L.sph_diagnostics.argtypes = [vp, C.POINTER(Diag)]
        L.sph_set_profiling.argtypes = [vp, C.c_int]
        L.sph_phase_times.argtypes = [vp, _P, C.POINTER(C.c_int64), C.c_int]
        L.sph_measure_fp64_peak.argtypes = [vp, _P]
        L.sph_local_count.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.sph_local_count.restype = C.c_int
        L.sph_memory_bytes.argtypes = [vp, C.POINTER(C.c_int64)]
        L.sph_memory_bytes.restype = C.c_int
        L.sph_nccl_unique_id.argtypes = [vp, C.c_int]
        L.sph_nccl_unique_id.restype = C.c_int
        L.sph_local_comm_id.argtypes = [C.c_int, vp, C.c_int]
        L.sph_local_comm_id.restype = C.c_int
        L.sph_decomp_splitters.argtypes = [C.POINTER(C.c_int64), C.c_int64, C.c_int,
                                           C.POINTER(C.c_int64)]
        L.sph_decomp_splitters.restype = C.c_int
        L.sph_decomp_owner.argtypes = [C.POINTER(C.c_int64), C.c_int, C.c_int64]
        L.sph_decomp_owner.restype = C.c_int
        for f in ("sph_init", "sph_attach", "sph_find_neighbors", "sph_get_neighbors", "sph_density",
                  "sph_iad", "sph_momentum_energy", "sph_advance", "sph_step", "sph_upload",
                  "sph_download", "sph_diagnostics", "sph_set_profiling", "sph_phase_times",
                  "sph_destroy", "sph_measure_fp64_peak"):
            getattr(L, f).restype = C.c_int
        if L.sph_abi_version() != ABI_VERSION:
            raise RuntimeError("libsph.so ABI version mismatch")
        _lib = L
    return _lib


def make_params(d: dict, *, n: float = 6.0, alpha: float = 1.0, omega_mode: int = 0,
                courant: float = 0.3, dt_growth: float = 1.1, h_min: float = 0.0,
                h_max: float = 0.0, u_floor: float = -np.inf, max_neighbors: int = 0,
                cell_factor: float = 0.0, rank: int = 0, nranks: int = 1, stream=None,
                kernel_mode: int = 0, table_size: int = 0, symmetric: int = 0,
                redecomp_every: int = 1) -> Params:
    p = Params()
    p.abi_version = ABI_VERSION
    p.sinc_n = n
    p.alpha_av = alpha
    p.eos = EOS[d["eos"]]
    p.c0, p.rho0, p.gamma = float(d["c0"]), float(d["rho0"]), float(d["gamma"])
    p.omega_mode = omega_mode
    p.courant, p.dt_growth = courant, dt_growth
    p.n_target = float(d["n_target"])
    p.h_min, p.h_max, p.u_floor = h_min, h_max, u_floor
    p.max_neighbors = max_neighbors
    p.cell_factor = cell_factor
    for k in range(3):
        p.box_lo[k] = float(d["box_lo"][k])
        p.box_hi[k] = float(d["box_hi"][k])
        p.periodic[k] = int(d["periodic"][k])
    p.rank, p.nranks = rank, nranks
    p.nccl_unique_id = None
    p.stream = stream
    p.kernel_mode = kernel_mode
    p.table_size = table_size
    p.symmetric = int(symmetric)
    p.redecomp_every = int(redecomp_every)
    return p


class DeviceParticles:
    """SoA fp64 torch tensors on the GPU (caller-owned memory of the C ABI)."""

    def __init__(self, d: dict, capacity: int | None = None, device="cuda"):
        import torch
        n = int(d["x"].size)
        cap = int(capacity or n)
        self.capacity = cap
        self.n = n
        self.t = {}
        self.t["id"] = torch.zeros(cap, dtype=torch.int64, device=device)
        self.t["id"][:n] = torch.from_numpy(np.ascontiguousarray(d["id"], dtype=np.int64)).to(device)
        for k in ALL_FIELDS:
            self.t[k] = torch.zeros(cap, dtype=torch.float64, device=device)
        for k in ("x", "y", "z", "vx", "vy", "vz", "h", "m", "u"):
            self.t[k][:n] = torch.from_numpy(np.ascontiguousarray(d[k], dtype=np.float64)).to(device)
        for k in ("vhx", "vhy", "vhz", "du_prev"):
            if k in d:
                self.t[k][:n] = torch.from_numpy(np.ascontiguousarray(d[k], dtype=np.float64)).to(device)

    def cstruct(self) -> Particles:
        s = Particles()
        s.n = self.n
        s.capacity = self.capacity
        s.id = C.cast(self.t["id"].data_ptr(), C.POINTER(C.c_int64))
        for k in ALL_FIELDS:
            setattr(s, k, C.cast(self.t[k].data_ptr(), _P))
        return s

    def numpy(self, fields=None) -> dict:
        fields = fields or ("id",) + ALL_FIELDS
        return {k: self.t[k][:self.n].cpu().numpy() for k in fields}


class HostParticles:
    """Pinned host SoA buffers for sph_upload / sph_download (end-to-end path)."""

    def __init__(self, d: dict, capacity: int | None = None):
        import torch
        n = int(d["x"].size)
        cap = int(capacity or n)
        self.n, self.capacity = n, cap
        self.t = {"id": torch.zeros(cap, dtype=torch.int64).pin_memory()}
        self.t["id"][:n] = torch.from_numpy(np.ascontiguousarray(d["id"], dtype=np.int64))
        for k in STATE_FIELDS:
            self.t[k] = torch.zeros(cap, dtype=torch.float64).pin_memory()
            if k in d:
                self.t[k][:n] = torch.from_numpy(np.ascontiguousarray(d[k], dtype=np.float64))

    def cstruct(self) -> Particles:
        s = Particles()
        s.n, s.capacity = self.n, self.capacity
        s.id = C.cast(self.t["id"].data_ptr(), C.POINTER(C.c_int64))
        for k in STATE_FIELDS:
            setattr(s, k, C.cast(self.t[k].data_ptr(), _P))
        return s

    def nbytes(self) -> int:
        return self.n * (8 * len(STATE_FIELDS) + 8)


class Simulation:
    """One context of libsph bound to a DeviceParticles set."""

    def __init__(self, d: dict, capacity: int | None = None, device="cuda", stream=None,
                 unique_id: bytes | None = None, **kw):
        import torch
        self.dev = DeviceParticles(d, capacity, device)
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        self.params = make_params(d, stream=stream, **kw)
        if self.params.nranks > 1:  # NCCL communicator from rank 0's id (dist.py)
            self._uid = C.create_string_buffer(unique_id, 128)
            self.params.nccl_unique_id = C.cast(self._uid, C.c_void_p)
        self._ctx = C.c_void_p()
        st = lib().sph_init(C.byref(self.params), self.dev.capacity, C.byref(self._ctx))
        if st != 0:
            msg = lib().sph_error_string(self._ctx).decode() if self._ctx else "sph_init rejected params"
            self.close()
            raise SphError(st, msg)
        self._parts = self.dev.cstruct()
        self._check(lib().sph_attach(self._ctx, C.byref(self._parts)))

    # -- plumbing
    def _check(self, st: int):
        if st != 0:
            raise SphError(st, lib().sph_error_string(self._ctx).decode())

    def close(self):
        if getattr(self, "_ctx", None):
            lib().sph_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n(self) -> int:
        return self.dev.n

    def _sync_n(self):
        no, nh = C.c_int64(0), C.c_int64(0)
        self._check(lib().sph_local_count(self._ctx, C.byref(no), C.byref(nh)))
        self.dev.n = no.value
        self.n_halo = nh.value

    # -- the method
    def find_neighbors(self):
        st = lib().sph_find_neighbors(self._ctx)
        self._sync_n()
        self._check(st)

    def get_neighbors(self):
        n = self.dev.n
        off = np.zeros(n + 1, dtype=np.int64)
        st = lib().sph_get_neighbors(self._ctx, off.ctypes.data_as(C.POINTER(C.c_int64)), None, 0)
        if st not in (0, 3):
            self._check(st)
        tot = int(off[-1])
        ids = np.zeros(max(tot, 1), dtype=np.int64)
        self._check(lib().sph_get_neighbors(self._ctx, off.ctypes.data_as(C.POINTER(C.c_int64)),
                                            ids.ctypes.data_as(C.POINTER(C.c_int64)), tot))
        return off, ids[:tot]

    def density(self):
        self._check(lib().sph_density(self._ctx))

    def iad(self):
        self._check(lib().sph_iad(self._ctx))

    def momentum_energy(self, want_dt: bool = False):
        dt = C.c_double(0.0)
        self._check(lib().sph_momentum_energy(self._ctx, C.byref(dt) if want_dt else None))
        return dt.value if want_dt else None

    def advance(self):
        self._check(lib().sph_advance(self._ctx))

    def step(self, want_dt: bool = False):
        dt = C.c_double(0.0)
        st = lib().sph_step(self._ctx, C.byref(dt) if want_dt else None)
        if self.params.nranks > 1:
            self._sync_n()
        self._check(st)
        return dt.value if want_dt else None

    def upload(self, host: HostParticles):
        s = host.cstruct()
        self._check(lib().sph_upload(self._ctx, C.byref(s)))
        self.dev.n = host.n

    def download(self, host: HostParticles):
        s = host.cstruct()
        self._check(lib().sph_download(self._ctx, C.byref(s)))
        host.n = s.n

    def diagnostics(self, check: bool = True) -> dict:
        """Conserved sums and counters (sph_diagnostics).  check=False returns what the
        library reports even after a sticky error (first_bad_id, steps)."""
        d = Diag()
        st = lib().sph_diagnostics(self._ctx, C.byref(d))
        if check:
            self._check(st)
        out = d.as_dict()
        out["status"] = st
        return out

    def library_bytes(self) -> int:
        """Device memory held by the library for this context (sph_memory_bytes)."""
        b = C.c_int64(0)
        self._check(lib().sph_memory_bytes(self._ctx, C.byref(b)))
        return b.value

    def set_profiling(self, on: bool):
        self._check(lib().sph_set_profiling(self._ctx, int(on)))

    def phase_times(self, reset: bool = False):
        ms = (C.c_double * len(PHASES))()
        ln = (C.c_int64 * len(PHASES))()
        self._check(lib().sph_phase_times(self._ctx, ms, ln, int(reset)))
        return dict(zip(PHASES, list(ms))), dict(zip(PHASES, list(ln)))

    def state(self) -> dict:
        return self.dev.numpy()
