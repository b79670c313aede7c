"""ctypes front end of the fp64 CPU oracle (oracle/sph_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of bench.py may import this.  It
never imports the CUDA package and the CUDA package never imports it.

The step pipeline below follows SURVEY §8(c) "Pipeline order":
O1 neighbours -> O3-O5 density/Omega/EOS -> O6 IAD -> O7 momentum/energy ->
O8 dt -> O9 update -> O10 h.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sph_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
          "-shared", "-fPIC", "-Wall"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "sph_oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Params(C.Structure):
    _fields_ = [
        ("n", C.c_double), ("Bn", C.c_double), ("table_K", C.c_int),
        ("table", C.POINTER(C.c_double)), ("alpha", C.c_double), ("eos", C.c_int),
        ("c0", C.c_double), ("rho0", C.c_double), ("gamma", C.c_double),
        ("omega_mode", C.c_int), ("courant", C.c_double), ("dt_growth", C.c_double),
        ("n_target", C.c_double), ("h_min", C.c_double), ("h_max", C.c_double),
        ("u_floor", C.c_double), ("box_lo", C.c_double * 3), ("box_hi", C.c_double * 3),
        ("periodic", C.c_int * 3), ("symmetric", C.c_int),
    ]


class Counters(C.Structure):
    _fields_ = [("omega_clamped", C.c_int64), ("iad_singular", C.c_int64),
                ("coincident_pairs", C.c_int64), ("u_floored", C.c_int64),
                ("h_clamped", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int64)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        P = C.POINTER(_Params)
        L.orc_norm.restype = C.c_double
        L.orc_norm.argtypes = [C.c_double]
        L.orc_table_build.argtypes = [C.c_double, C.c_int, _D]
        for f in ("orc_S", "orc_vdS"):
            getattr(L, f).restype = C.c_double
            getattr(L, f).argtypes = [P, C.c_double]
        for f in ("orc_W", "orc_dWdh"):
            getattr(L, f).restype = C.c_double
            getattr(L, f).argtypes = [P, C.c_double, C.c_double]
        L.orc_neighbors.restype = C.c_int64
        L.orc_neighbors.argtypes = [P, C.c_int, C.c_int64, _D, _D, _D, _D, _I, _I, C.c_int64]
        L.orc_density.argtypes = [P, C.c_int64] + [_D] * 6 + [_I, _I] + [_D] * 5 + [C.POINTER(Counters)]
        L.orc_iad.argtypes = [P, C.c_int64] + [_D] * 6 + [_I, _I] + [_D] * 6 + [C.POINTER(Counters)]
        L.orc_momentum_energy.argtypes = ([P, C.c_int64] + [_D] * 18 + [_I, _I] + [_D] * 7 +
                                          [C.POINTER(Counters)])
        L.orc_timestep.restype = C.c_double
        L.orc_timestep.argtypes = [P, C.c_int64, _D, _D, C.c_double, C.c_int]
        L.orc_update.argtypes = ([P, C.c_int64, C.c_double, C.c_double, C.c_int] + [_D] * 15 +
                                 [C.POINTER(Counters)])
        L.orc_update_h.argtypes = [P, C.c_int64, _D, _I, C.POINTER(Counters)]
        L.orc_diagnostics.argtypes = [C.c_int64] + [_D] * 9
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(_D)


def _i(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_I)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Params:
    """Method constants (readings R7-R20)."""
    n: float = 6.0
    table_K: int = 0
    alpha: float = 1.0
    eos: str = "linear"
    c0: float = 1.0
    rho0: float = 1.0
    gamma: float = 5.0 / 3.0
    omega_mode: int = 0
    courant: float = 0.3
    dt_growth: float = 1.1
    n_target: float = 300.0
    h_min: float = 0.0
    h_max: float = 0.0
    u_floor: float = -np.inf
    box_lo: tuple = (0.0, 0.0, 0.0)
    box_hi: tuple = (1.0, 1.0, 1.0)
    periodic: tuple = (0, 0, 0)
    symmetric: int = 0

    @classmethod
    def from_inputs(cls, d: dict, **kw) -> "Params":
        p = cls(eos=d["eos"], c0=float(d["c0"]), rho0=float(d["rho0"]), gamma=float(d["gamma"]),
                n_target=float(d["n_target"]), box_lo=tuple(map(float, d["box_lo"])),
                box_hi=tuple(map(float, d["box_hi"])),
                periodic=tuple(int(v) for v in d["periodic"]))
        for k, v in kw.items():
            setattr(p, k, v)
        return p

    def cstruct(self):
        s = _Params()
        s.n = self.n
        s.Bn = norm(self.n)
        s.table_K = int(self.table_K)
        self._table = None
        if self.table_K > 0:
            self._table = table(self.n, self.table_K)
            s.table = _d(self._table)
        s.alpha = self.alpha
        s.eos = 0 if self.eos == "linear" else 1
        s.c0, s.rho0, s.gamma = self.c0, self.rho0, self.gamma
        s.omega_mode = self.omega_mode
        s.courant, s.dt_growth, s.n_target = self.courant, self.dt_growth, self.n_target
        s.h_min, s.h_max, s.u_floor = self.h_min, self.h_max, self.u_floor
        for k in range(3):
            s.box_lo[k] = self.box_lo[k]
            s.box_hi[k] = self.box_hi[k]
            s.periodic[k] = int(self.periodic[k])
        s.symmetric = int(self.symmetric)
        return s


_norm_cache: dict = {}


def norm(n: float) -> float:
    if n not in _norm_cache:
        _norm_cache[n] = lib().orc_norm(n)
    return _norm_cache[n]


def table(n: float, K: int) -> np.ndarray:
    t = np.empty(K)
    lib().orc_table_build(n, K, _d(t))
    return t


class Oracle:
    def __init__(self, params: Params):
        self.params = params
        self._s = params.cstruct()
        self.p = C.byref(self._s)
        self.counters = Counters()

    # ---- kernel ---------------------------------------------------------
    def S(self, v):
        return np.array([lib().orc_S(self.p, float(t)) for t in np.atleast_1d(v)])

    def vdS(self, v):
        return np.array([lib().orc_vdS(self.p, float(t)) for t in np.atleast_1d(v)])

    def W(self, r, h):
        return np.array([lib().orc_W(self.p, float(t), float(h)) for t in np.atleast_1d(r)])

    def dWdh(self, r, h):
        return np.array([lib().orc_dWdh(self.p, float(t), float(h)) for t in np.atleast_1d(r)])

    # ---- O1 ---------------------------------------------------------------
    def neighbors(self, d: dict, method: int = 1):
        """CSR (offsets[N+1], nbr) of particle positions, rows ascending."""
        x, y, z = (_f64(d[k]) for k in ("x", "y", "z"))
        h = _f64(d["h"])
        N = x.size
        off = np.zeros(N + 1, dtype=np.int64)
        cap = int(max(1, N) * 64)
        nbr = np.empty(cap, dtype=np.int64)
        tot = lib().orc_neighbors(self.p, method, N, _d(x), _d(y), _d(z), _d(h), _i(off),
                                  _i(nbr), cap)
        if tot > cap:
            nbr = np.empty(tot, dtype=np.int64)
            tot = lib().orc_neighbors(self.p, method, N, _d(x), _d(y), _d(z), _d(h), _i(off),
                                      _i(nbr), tot)
        return off, nbr[:tot].copy()

    # ---- O3-O5 --------------------------------------------------------------
    def density(self, d: dict, off, nbr):
        x, y, z, h, m, u = (_f64(d[k]) for k in ("x", "y", "z", "h", "m", "u"))
        N = x.size
        out = {k: np.empty(N) for k in ("rho", "omega", "p", "c", "omega_scale")}
        lib().orc_density(self.p, N, _d(x), _d(y), _d(z), _d(h), _d(m), _d(u), _i(off), _i(nbr),
                          _d(out["rho"]), _d(out["omega"]), _d(out["p"]), _d(out["c"]),
                          _d(out["omega_scale"]), C.byref(self.counters))
        return out

    # ---- O6 -------------------------------------------------------------------
    def iad(self, d: dict, rho, off, nbr):
        x, y, z, h, m = (_f64(d[k]) for k in ("x", "y", "z", "h", "m"))
        rho = _f64(rho)
        N = x.size
        out = {k: np.empty(N) for k in ("c11", "c12", "c13", "c22", "c23", "c33")}
        lib().orc_iad(self.p, N, _d(x), _d(y), _d(z), _d(h), _d(m), _d(rho), _i(off), _i(nbr),
                      *(_d(out[k]) for k in ("c11", "c12", "c13", "c22", "c23", "c33")),
                      C.byref(self.counters))
        return out

    # ---- O7 -------------------------------------------------------------------
    def momentum_energy(self, d: dict, dens: dict, iad: dict, off, nbr):
        f = [_f64(d[k]) for k in ("x", "y", "z", "vx", "vy", "vz", "h", "m")]
        g = [_f64(dens[k]) for k in ("rho", "omega", "p", "c")]
        cc = [_f64(iad[k]) for k in ("c11", "c12", "c13", "c22", "c23", "c33")]
        N = f[0].size
        out = {k: np.empty(N) for k in ("ax", "ay", "az", "du", "vsig", "scale_du")}
        out["scale_a"] = np.empty(3 * N)
        lib().orc_momentum_energy(self.p, N, *(_d(a) for a in f + g + cc), _i(off), _i(nbr),
                                  *(_d(out[k]) for k in ("ax", "ay", "az", "du", "vsig",
                                                         "scale_a", "scale_du")),
                                  C.byref(self.counters))
        out["scale_a"] = out["scale_a"].reshape(3, N)
        return out

    # ---- O8-O11 -----------------------------------------------------------------
    def timestep(self, h, vsig, dt_prev: float, first: bool) -> float:
        h, vsig = _f64(h), _f64(vsig)
        return lib().orc_timestep(self.p, h.size, _d(h), _d(vsig), float(dt_prev), int(first))

    def update(self, st: dict, acc: dict, dt: float, dt_prev: float, first: bool):
        """In place on st (x,y,z,vx,vy,vz,vhx,vhy,vhz,u,du_prev)."""
        N = st["x"].size
        lib().orc_update(self.p, N, float(dt), float(dt_prev), int(first),
                         *(_d(st[k]) for k in ("x", "y", "z", "vx", "vy", "vz", "vhx", "vhy", "vhz")),
                         *(_d(_f64(acc[k])) for k in ("ax", "ay", "az")),
                         _d(st["u"]), _d(_f64(acc["du"])), _d(st["du_prev"]),
                         C.byref(self.counters))

    def update_h(self, h: np.ndarray, off):
        lib().orc_update_h(self.p, h.size, _d(h), _i(off), C.byref(self.counters))

    @staticmethod
    def diagnostics(d: dict) -> np.ndarray:
        out = np.empty(7)
        f = [_f64(d[k]) for k in ("m", "x", "y", "z", "vx", "vy", "vz", "u")]
        lib().orc_diagnostics(f[0].size, *(_d(a) for a in f), _d(out))
        return out

    # ---- whole step --------------------------------------------------------------
    def step(self, st: dict, method: int = 1) -> dict:
        """One timestep on state dict ``st`` (copied).  ``st`` holds x..u, and
        optionally vhx/vhy/vhz/du_prev/dt_prev/first.  Returns the new state
        plus every intermediate (neighbours, density, IAD, rates, dt)."""
        s = {k: _f64(st[k]).copy() for k in ("x", "y", "z", "vx", "vy", "vz", "h", "m", "u")}
        N = s["x"].size
        for k in ("vhx", "vhy", "vhz", "du_prev"):
            s[k] = _f64(st[k]).copy() if k in st else np.zeros(N)
        first = bool(st.get("first", True))
        dt_prev = float(st.get("dt_prev", 0.0))
        off, nbr = self.neighbors(s, method)
        dens = self.density(s, off, nbr)
        iad = self.iad(s, dens["rho"], off, nbr)
        acc = self.momentum_energy(s, dens, iad, off, nbr)
        dt = self.timestep(s["h"], acc["vsig"], dt_prev, first)
        self.update(s, acc, dt, dt_prev, first)
        self.update_h(s["h"], off)
        s["dt_prev"] = dt
        s["first"] = False
        return {"state": s, "offsets": off, "nbr": nbr, "dens": dens, "iad": iad, "acc": acc,
                "dt": dt}
