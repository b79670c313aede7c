"""Comparison helpers for GPU <-> oracle parity (tolerances: SURVEY §8(c)).

Tolerances (fp64; BASELINE north_star "<=1e-10 rel. physics", normalised per R27):
  neighbours  bit-exact as sorted global-id sets, counts equal
  rho         |d| <= 1e-10 |rho|                      (all-positive sum)
  Omega       |d| <= 1e-10 * omega_scale              (1 + h/(3 rho) sum|m dW/dh|)
  P           |d| <= 1e-10 * c0^2 max(rho, rho0)      (linear EOS) | 1e-10 |P| (ideal gas)
  c           |d| <= 1e-10 |c|
  C           ||dC||_F <= 1e-10 ||C||_F
  a, du       |d| <= 1e-10 * S_a (sum_b |summand|, exported by the oracle)
  vsig        |d| <= 1e-12 |vsig|
  dt          |d| <= 1e-12 dt
  update      |d| <= 1e-14 * (|old| + |increment|) from identical inputs
"""
import numpy as np

TOL = 1e-10
META = ("box_lo", "box_hi", "periodic", "eos", "c0", "rho0", "gamma", "n_target", "name", "dx")


def with_meta(st: dict, d: dict) -> dict:
    out = dict(st)
    for k in META:
        if k in d:
            out[k] = d[k]
    return out


def rows_by_id(off, ids):
    """canonical (row, id) ordering for set comparison"""
    n = off.size - 1
    row = np.repeat(np.arange(n), np.diff(off))
    o = np.lexsort((ids, row))
    return row[o], ids[o]


def assert_neighbors_equal(off_g, ids_g, off_o, ids_o):
    np.testing.assert_array_equal(np.diff(off_g), np.diff(off_o), err_msg="neighbour counts differ")
    rg, ig = rows_by_id(off_g, ids_g)
    ro, io = rows_by_id(off_o, ids_o)
    np.testing.assert_array_equal(rg, ro)
    bad = np.flatnonzero(ig != io)
    assert bad.size == 0, f"{bad.size} neighbour ids differ (first row {rg[bad[0]] if bad.size else -1})"


def _viol(name, d, bound):
    bad = np.flatnonzero(~(np.abs(d) <= bound))
    if bad.size:
        i = bad[0]
        raise AssertionError(f"{name}: {bad.size} violations; first i={i} diff={d[i]:.3e} "
                             f"bound={bound[i] if np.ndim(bound) else bound:.3e}")


def check_density(g: dict, o: dict, d: dict, idx=None):
    sl = slice(None) if idx is None else idx
    rho_o = o["rho"]
    _viol("rho", g["rho"][sl] - rho_o, TOL * np.abs(rho_o))
    _viol("omega", g["omega"][sl] - o["omega"], TOL * o["omega_scale"])
    if d["eos"] == "linear":
        _viol("p", g["p"][sl] - o["p"], TOL * d["c0"] ** 2 * np.maximum(rho_o, d["rho0"]))
    else:
        _viol("p", g["p"][sl] - o["p"], TOL * np.abs(o["p"]) + 1e-300)
    _viol("c", g["c"][sl] - o["c"], TOL * np.abs(o["c"]) + 1e-300)


def check_iad(g: dict, o: dict, idx=None):
    sl = slice(None) if idx is None else idx
    keys = ("c11", "c12", "c13", "c22", "c23", "c33")
    w = np.array([1, 2, 2, 1, 2, 1], dtype=np.float64)  # off-diagonals appear twice
    dF = np.sqrt(sum(wk * (g[k][sl] - o[k]) ** 2 for wk, k in zip(w, keys)))
    nF = np.sqrt(sum(wk * o[k] ** 2 for wk, k in zip(w, keys)))
    _viol("C", dF, TOL * nF)


def check_momentum(g: dict, o: dict, idx=None):
    sl = slice(None) if idx is None else idx
    for k, ax in enumerate(("ax", "ay", "az")):
        _viol(ax, g[ax][sl] - o[ax], TOL * o["scale_a"][k] + 1e-300)
    _viol("du", g["du"][sl] - o["du"], TOL * o["scale_du"] + 1e-300)
    _viol("vsig", g["vsig"][sl] - o["vsig"], 1e-12 * np.abs(o["vsig"]))


def oracle_pipeline(O, st: dict, method: int = 1, **okw):
    """Oracle on a state dict (any order); returns neighbours + all outputs.
    okw: oracle Params overrides (e.g. table_K for the table kernel mode)."""
    o = O.Oracle(O.Params.from_inputs(st, **okw))
    off, nbr = o.neighbors(st, method)
    dn = o.density(st, off, nbr)
    C = o.iad(st, dn["rho"], off, nbr)
    me = o.momentum_energy(st, dn, C, off, nbr)
    return o, off, nbr, dn, C, me
