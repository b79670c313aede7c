"""Seeded, synthetic particle sets for the SPH-EXA hot path (arXiv 2005.02656).

This module is the ONE piece shared by the CUDA path (bench, tests) and the
oracle tests. It holds initial conditions only -- none of the method's
arithmetic (no kernel, no density, no forces, no integrator). Every generator
returns a dict of SoA numpy fp64 arrays plus the metadata the method needs
(box, periodicity, EOS constants).

Recipes:

* Rotating square patch, §4.6 (lines 265-282): an n x n layer of a
  cell-centred lattice on [-L/2, L/2]^2, copied ``layers`` times along z with
  periodic z; rigid rotation v = (w*y, -w*x, 0) (Eq. 7)
  with w = 5 rad/s.  Units (reading R14): L = 100 cm, rho0 = 1 g/cm^3,
  depth = layers * dx, which reproduces L_tot = w rho0 L^5 / 6 = 8.33e9.
  Mass m = rho0 dx^3; the optional pressure-consistent variant (reading R16)
  modulates m by the P0 series (odd m,n, second argument y: R15).
  h = 0.5 * (3 n_target / (4 pi))^(1/3) dx so a lattice sphere of radius 2h
  holds ~n_target = 300 particles (reading R20).  Linear EOS with
  c0 = 10 w L / sqrt(2) (reading R13).
* Evrard-shaped sphere (config 3, not in the paper): cell-centred lattice in
  [-1,1]^3 clipped to r<1, radially stretched r -> r^(3/2) so rho ~ 1/(2 pi r);
  M = R = 1, v = 0, u = 0.05, ideal gas gamma = 5/3, h from the local density.
* Jittered lattice / random cloud: test-only perturbations drawn from
  numpy.random.Generator(PCG64(seed)).
"""
from __future__ import annotations

import math

import numpy as np

SEED = 20050265  # the seed every randomised test input derives from

FIELDS = ("x", "y", "z", "vx", "vy", "vz", "h", "m", "u")


def h_for_lattice(dx: float, n_target: float = 300.0) -> float:
    """h such that (4 pi / 3) (2h)^3 = n_target dx^3 (reading R20)."""
    return 0.5 * (3.0 * n_target / (4.0 * math.pi)) ** (1.0 / 3.0) * dx


def _p0_series(xp: np.ndarray, yp: np.ndarray, L: float, omega: float, rho0: float,
               n_terms: int) -> np.ndarray:
    """P0(x', y') on corner-origin coordinates, P:276-279 with readings R15.

    Sum over odd m, n <= 2*n_terms-1 of
      -32 w^2 rho / (m n pi^2 [(m pi/L)^2 + (n pi/L)^2]) sin(m pi x'/L) sin(n pi y'/L).
    Separable, so evaluated as s_x^T A s_y.
    """
    ks = np.arange(1, 2 * n_terms, 2, dtype=np.float64)
    mm, nn = np.meshgrid(ks, ks, indexing="ij")
    a = -32.0 * omega ** 2 * rho0 / (mm * nn * math.pi ** 2 *
                                      ((mm * math.pi / L) ** 2 + (nn * math.pi / L) ** 2))
    sx = np.sin(np.outer(xp, ks) * math.pi / L)  # [nx, K]
    sy = np.sin(np.outer(yp, ks) * math.pi / L)  # [ny, K]
    return sx @ a @ sy.T  # [nx, ny]


def square_patch(n: int, layers: int | None = None, *, L: float = 100.0, omega: float = 5.0,
                 rho0: float = 1.0, n_target: float = 300.0, pressure_ics: bool = False,
                 series_terms: int = 80, z_layers: tuple[int, int] | None = None,
                 u0: float = 1.0) -> dict:
    """Rotating square patch (§4.6).  ``z_layers=(k0,k1)`` returns only
    layers k0..k1-1 (a z-slab of the same global problem; ids stay global)."""
    layers = n if layers is None else layers
    dx = L / n
    Lz = layers * dx
    k0, k1 = (0, layers) if z_layers is None else z_layers
    ii = np.arange(n, dtype=np.float64)
    xs = -0.5 * L + (ii + 0.5) * dx
    kk = np.arange(k0, k1, dtype=np.float64)
    zs = -0.5 * Lz + (kk + 0.5) * dx
    nl = k1 - k0
    # id = i + n (j + n k): x fastest
    X = np.broadcast_to(xs[None, None, :], (nl, n, n)).ravel().copy()
    Y = np.broadcast_to(xs[None, :, None], (nl, n, n)).ravel().copy()
    Z = np.broadcast_to(zs[:, None, None], (nl, n, n)).ravel().copy()
    ids = (np.arange(k0 * n * n, k1 * n * n, dtype=np.int64))
    c0 = 10.0 * omega * L / math.sqrt(2.0)
    N = X.size
    if pressure_ics:
        p0 = _p0_series(xs + 0.5 * L, xs + 0.5 * L, L, omega, rho0, series_terms)  # [i(x), j(y)]
        # layer layout is [k, j(y), i(x)]
        p_layer = p0.T.ravel()
        m = np.tile(dx ** 3 * (rho0 + p_layer / c0 ** 2), nl)
    else:
        m = np.full(N, rho0 * dx ** 3)
    out = {
        "id": ids,
        "x": X, "y": Y, "z": Z,
        "vx": omega * Y, "vy": -omega * X, "vz": np.zeros(N),
        "h": np.full(N, h_for_lattice(dx, n_target)),
        "m": m,
        "u": np.full(N, u0),
        "box_lo": np.array([-0.5 * L, -0.5 * L, -0.5 * Lz]),
        "box_hi": np.array([0.5 * L, 0.5 * L, 0.5 * Lz]),
        "periodic": np.array([0, 0, 1], dtype=np.int32),
        "eos": "linear", "c0": c0, "rho0": rho0, "gamma": 5.0 / 3.0,
        "n_target": n_target, "dx": dx, "L": L, "omega": omega, "n_total": n * n * layers,
        "name": f"square_patch_{n}x{n}x{layers}",
    }
    return out


def square_patch_weak(n: int, G: int, rank: int | None = None, **kw) -> dict:
    """Config 5: z-stacked patch n x n x (n*G) with z period G*L; per-rank slab
    of n layers when ``rank`` is given (PAPER.md P:268 z replication)."""
    layers = n * G
    zl = None if rank is None else (rank * n, (rank + 1) * n)
    d = square_patch(n, layers, z_layers=zl, **kw)
    d["name"] = f"square_patch_weak_{n}x{n}x{layers}"
    return d


def evrard(n: int = 124, *, n_target: float = 300.0, u0: float = 0.05,
           gamma: float = 5.0 / 3.0) -> dict:
    """Evrard-shaped collapsing sphere (config 3; hydro only, not in the paper)."""
    dx = 2.0 / n
    c = -1.0 + (np.arange(n, dtype=np.float64) + 0.5) * dx
    Zg, Yg, Xg = np.meshgrid(c, c, c, indexing="ij")
    X, Y, Z = Xg.ravel(), Yg.ravel(), Zg.ravel()
    r = np.sqrt(X * X + Y * Y + Z * Z)
    keep = r < 1.0
    X, Y, Z, r = X[keep], Y[keep], Z[keep], r[keep]
    s = np.sqrt(r)  # r -> r^(3/2) == r * sqrt(r)
    X, Y, Z = X * s, Y * s, Z * s
    rn = r * s
    N = X.size
    m = 1.0 / N
    rho = 1.0 / (2.0 * math.pi * rn)
    h = 0.5 * (3.0 * n_target * m / (4.0 * math.pi * rho)) ** (1.0 / 3.0)
    lo = np.array([X.min(), Y.min(), Z.min()])
    hi = np.array([X.max(), Y.max(), Z.max()])
    return {
        "id": np.flatnonzero(keep).astype(np.int64),
        "x": X, "y": Y, "z": Z,
        "vx": np.zeros(N), "vy": np.zeros(N), "vz": np.zeros(N),
        "h": h, "m": np.full(N, m), "u": np.full(N, u0),
        "box_lo": lo, "box_hi": hi, "periodic": np.array([0, 0, 0], dtype=np.int32),
        "eos": "ideal", "c0": 0.0, "rho0": 0.0, "gamma": gamma,
        "n_target": n_target, "name": f"evrard_{n}", "n_total": N,
    }


def jitter(d: dict, frac: float = 0.1, seed: int = SEED) -> dict:
    """Uniform position jitter of +-frac*dx (tests only); z re-wrapped if periodic."""
    g = np.random.Generator(np.random.PCG64(seed))
    out = dict(d)
    dx = d["dx"]
    for k, ax in (("x", 0), ("y", 1), ("z", 2)):
        v = d[k] + g.uniform(-frac * dx, frac * dx, d[k].size)
        if d["periodic"][ax]:
            lo, hi = d["box_lo"][ax], d["box_hi"][ax]
            v = np.where(v >= hi, v - (hi - lo), v)
            v = np.where(v < lo, v + (hi - lo), v)
        out[k] = v
    return out


def random_cloud(N: int, *, box: float = 10.0, h0: float = 1.0, hspread: float = 0.2,
                 periodic=(0, 0, 1), seed: int = SEED, vscale: float = 1.0,
                 c0: float = 10.0) -> dict:
    """N uniform points in [0,box)^3 with h ~ U[(1-hspread) h0, (1+hspread) h0] (tests only)."""
    g = np.random.Generator(np.random.PCG64(seed))
    X = g.uniform(0.0, box, N)
    Y = g.uniform(0.0, box, N)
    Z = g.uniform(0.0, box, N)
    return {
        "id": np.arange(N, dtype=np.int64),
        "x": X, "y": Y, "z": Z,
        "vx": g.normal(0.0, vscale, N), "vy": g.normal(0.0, vscale, N),
        "vz": g.normal(0.0, vscale, N),
        "h": g.uniform((1 - hspread) * h0, (1 + hspread) * h0, N),
        "m": g.uniform(0.5, 1.5, N), "u": g.uniform(0.5, 1.5, N),
        "box_lo": np.zeros(3), "box_hi": np.full(3, box),
        "periodic": np.array(periodic, dtype=np.int32),
        "eos": "linear", "c0": c0, "rho0": 1.0, "gamma": 5.0 / 3.0,
        "n_target": 50.0, "name": f"random_cloud_{N}", "n_total": N,
    }


def subset(d: dict, idx: np.ndarray) -> dict:
    """Particles ``idx`` of ``d`` (same metadata)."""
    out = dict(d)
    for k in ("id",) + FIELDS:
        out[k] = np.ascontiguousarray(d[k][idx])
    return out


def shuffled(d: dict, seed: int = SEED) -> dict:
    """Same particles in a seeded random order (exercises the sort)."""
    g = np.random.Generator(np.random.PCG64(seed))
    return subset(d, g.permutation(d["x"].size))
