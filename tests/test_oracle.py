"""T0: pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a closed form, a library routine
(numpy.sinc, scipy quadrature), brute force written independently in numpy, a
conservation law, or a survey value stored in tests/golden/config1_t0.json.
"""
import json
import math
import os

import numpy as np
import pytest

from paper_2005_02656_b200 import inputs as I

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config1_t0.json")))


def S_np(v, n=6.0):
    """Eq. 6 through numpy's sinc (np.sinc(t) = sin(pi t)/(pi t)): sinc(pi v/2) = np.sinc(v/2)."""
    v = np.asarray(v, dtype=np.float64)
    return np.where(v < 2.0, np.sinc(0.5 * v) ** n, 0.0)


def lattice(side, dx=1.0, m=1.0):
    c = (np.arange(side) - (side - 1) / 2.0) * dx
    Z, Y, X = np.meshgrid(c, c, c, indexing="ij")
    N = X.size
    h = I.h_for_lattice(dx)
    return {"id": np.arange(N), "x": X.ravel(), "y": Y.ravel(), "z": Z.ravel(),
            "vx": np.zeros(N), "vy": np.zeros(N), "vz": np.zeros(N), "h": np.full(N, h),
            "m": np.full(N, m), "u": np.ones(N), "box_lo": np.full(3, -1e3),
            "box_hi": np.full(3, 1e3), "periodic": np.zeros(3, dtype=np.int32), "eos": "linear",
            "c0": 1.0, "rho0": 1.0, "gamma": 5 / 3, "n_target": 300.0, "dx": dx}


def center_index(side):
    k = side // 2
    return k + side * (k + side * k)


def brute_numpy(d, symmetric=False):
    """Independent O(N^2) neighbour sets: same r^2 association, min image on periodic dims
    (symmetric: r < 2 max(h_a, h_b))."""
    X = np.stack([d["x"], d["y"], d["z"]])
    N = X.shape[1]
    lo, hi = np.asarray(d["box_lo"]), np.asarray(d["box_hi"])
    sets = []
    for a in range(N):
        D = X - X[:, a:a + 1]
        for k in range(3):
            if d["periodic"][k]:
                L = hi[k] - lo[k]
                D[k] = np.where(D[k] > 0.5 * L, D[k] - L, np.where(D[k] < -0.5 * L, D[k] + L, D[k]))
        r2 = (D[0] * D[0] + D[1] * D[1]) + D[2] * D[2]
        tha = 2.0 * (np.maximum(d["h"][a], d["h"]) if symmetric else d["h"][a])
        ok = r2 < tha * tha
        ok[a] = False
        sets.append(np.flatnonzero(ok))
    return sets


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


def mk(O, d, **kw):
    return O.Oracle(O.Params.from_inputs(d, **kw))


# ------------------------------------------------------------------ kernel (Eq. 6)

def test_norm_matches_survey_quadrature_and_scipy(O):
    from scipy.integrate import quad
    for n in (3, 4, 5, 6, 7, 8):
        B = O.norm(float(n))
        assert abs(B - GOLD["B"][str(n)]) < 1e-4 * GOLD["B"][str(n)]
        # independent quadrature of numpy's sinc: 4 pi B int S v^2 dv = 1
        I2, _ = quad(lambda v: S_np(v, n) * v * v, 0.0, 2.0, epsabs=1e-14, epsrel=1e-14, limit=200)
        assert abs(4 * math.pi * B * I2 - 1.0) < 1e-12
    assert abs(O.norm(6.0) - GOLD["B"]["6"]) < 1e-15
    Bs = [O.norm(float(n)) for n in (4, 5, 6, 7, 8)]
    assert all(b2 > b1 for b1, b2 in zip(Bs, Bs[1:]))


def test_kernel_closed_forms(O):
    o = mk(O, lattice(3))
    B = O.norm(6.0)
    assert o.W(0.0, 1.0)[0] == B
    assert abs(o.W(1.0, 1.0)[0] - GOLD["W_1_1"]) < 1e-16
    assert abs(o.W(1.0, 1.0)[0] - B * (2 / math.pi) ** 6) < 1e-15 * B
    assert o.W(2.0, 1.0)[0] == 0.0 and o.W(2.5, 1.0)[0] == 0.0
    v = np.linspace(0, 1.999, 997)
    np.testing.assert_allclose(o.S(v), S_np(v), rtol=1e-13, atol=1e-300)
    # h scaling W(v h, h) = W(v, 1) / h^3
    for h in (0.37, 2.0, 5.5):
        np.testing.assert_allclose(o.W(v * h, h), o.W(v, 1.0) / h ** 3, rtol=1e-14,
                                   atol=1e-15 * B / h ** 3)


def test_kernel_derivative_central_difference(O):
    o = mk(O, lattice(3))
    for v in (0.3, 0.7, 1.1, 1.8):
        e = 1e-6
        fd = v * (S_np(v + e) - S_np(v - e)) / (2 * e)
        assert abs(o.vdS(v)[0] - fd) < 1e-6 * max(1e-3, abs(fd))
    for r, h in ((0.5, 1.0), (1.3, 0.9), (2.9, 1.6)):
        e = 1e-6 * h
        fd = (o.W(r, h + e)[0] - o.W(r, h - e)[0]) / (2 * e)
        assert abs(o.dWdh(r, h)[0] - fd) < 1e-6 * abs(fd)
    assert o.vdS(0.0)[0] == 0.0 and o.vdS(2.0)[0] == 0.0
    assert o.dWdh(0.0, 2.0)[0] == -3 * O.norm(6.0) / 2.0 ** 4


def test_table_mode(O):
    K = 20000
    t = O.table(6.0, K)
    nodes = 2.0 * np.arange(K) / (K - 1)
    np.testing.assert_allclose(t, S_np(nodes), rtol=1e-13, atol=1e-30)
    assert t[0] == 1.0 and abs(t[-1]) < 1e-90
    assert np.all(np.diff(t) <= 0)
    o = mk(O, lattice(3), table_K=K)
    g = np.random.Generator(np.random.PCG64(I.SEED))
    v = g.uniform(0.0, 2.0, 20000)
    sT = o.S(v)
    assert np.max(np.abs(sT - S_np(v))) < 1e-4  # S:102 dense-sweep bound
    np.testing.assert_allclose(sT, np.interp(v, nodes, t), rtol=1e-12, atol=1e-18)
    np.testing.assert_allclose(o.S(nodes[:100]), t[:100], rtol=1e-15)


# ------------------------------------------------------------------ O1 neighbours

@pytest.mark.parametrize("case", ["patch", "jitter", "cloud_periodic", "cloud_open"])
def test_neighbors_brute_force(O, case):
    if case == "patch":
        d = I.square_patch(10, 10)
    elif case == "jitter":
        d = I.jitter(I.square_patch(12, 8))
    elif case == "cloud_periodic":
        d = I.random_cloud(1500, box=8.0, h0=0.9, periodic=(1, 0, 1))
    else:
        d = I.random_cloud(1500, box=8.0, h0=0.9, periodic=(0, 0, 0), seed=7)
    ref = brute_numpy(d)
    o = mk(O, d)
    for method in (0, 1):
        off, nbr = o.neighbors(d, method)
        for a in range(d["x"].size):
            np.testing.assert_array_equal(nbr[off[a]:off[a + 1]], ref[a])


def test_neighbors_config1_counts(O):
    d = I.square_patch(20)
    o = mk(O, d)
    off, nbr = o.neighbors(d, 1)
    cnt = np.diff(off)
    assert off[-1] == GOLD["directed_pairs"]
    assert cnt.min() == GOLD["nbr_min"] and cnt.max() == GOLD["nbr_max"]
    # symmetric under uniform h
    pairs = set(zip(np.repeat(np.arange(cnt.size), cnt).tolist(), nbr.tolist()))
    assert all((b, a) in pairs for a, b in list(pairs)[:20000])


def test_lattice_interior_304(O):
    d = lattice(13)
    o = mk(O, d)
    off, _ = o.neighbors(d, 1)
    assert off[center_index(13) + 1] - off[center_index(13)] == GOLD["lattice_interior_neighbors"]


# ------------------------------------------------------------------ O3-O5 density

def test_density_isolated_and_pair(O):
    d = lattice(1)
    d["h"][:] = 1.3
    d["m"][:] = 2.5
    o = mk(O, d)
    off, nbr = o.neighbors(d, 0)
    r = o.density(d, off, nbr)
    B = O.norm(6.0)
    assert abs(r["rho"][0] - 2.5 * B / 1.3 ** 3) < 1e-15 * r["rho"][0]
    assert r["omega"][0] == 0.1  # 1 + h/(3 rho) m dW/dh(0) = 0 -> clamped
    # pair at distance 1.7 with h = 1.3: rho = m (W(0) + W(1.7))
    pd = lattice(1)
    for k in ("id", "x", "y", "z", "vx", "vy", "vz", "h", "m", "u"):
        pd[k] = np.concatenate([pd[k], pd[k]])
    pd["x"][1] = 1.7
    pd["h"][:] = 1.3
    off, nbr = o.neighbors(pd, 0)
    r = o.density(pd, off, nbr)
    ref = (B / 1.3 ** 3) * (S_np(0.0) + S_np(1.7 / 1.3))
    np.testing.assert_allclose(r["rho"], [ref, ref], rtol=1e-14)


def test_density_lattice_interior_and_brute(O):
    d = lattice(13)
    o = mk(O, d)
    off, nbr = o.neighbors(d, 1)
    r = o.density(d, off, nbr)
    a = center_index(13)
    assert abs(r["rho"][a] - GOLD["lattice_interior_rho"]) < 1e-14
    assert abs(r["omega"][a] - GOLD["lattice_interior_omega"]) < 1e-13
    # random cloud vs an independent numpy all-pairs sum through numpy.sinc
    c = I.random_cloud(800, box=6.0, h0=0.8, periodic=(0, 0, 1))
    o = mk(O, c)
    off, nbr = o.neighbors(c, 1)
    r = o.density(c, off, nbr)
    B = O.norm(6.0)
    X = np.stack([c["x"], c["y"], c["z"]])
    for a in range(0, 800, 37):
        D = X - X[:, a:a + 1]
        L = c["box_hi"][2] - c["box_lo"][2]
        D[2] = np.where(D[2] > L / 2, D[2] - L, np.where(D[2] < -L / 2, D[2] + L, D[2]))
        rr = np.sqrt((D * D).sum(0))
        ref = np.sum(c["m"] * B * S_np(rr / c["h"][a]) / c["h"][a] ** 3)
        assert abs(r["rho"][a] - ref) < 1e-13 * ref


def test_omega_is_density_h_derivative(O):
    """Omega_a = 1 + h/(3 rho) d rho_a / d h_a (grad-h closure, R8): check by finite differences."""
    c = I.jitter(I.square_patch(12, 12))
    o = mk(O, c)
    off, nbr = o.neighbors(c, 1)
    r = o.density(c, off, nbr)
    for a in (0, 77, 500, 1000):
        e = 1e-5 * c["h"][a]
        rs = []
        for s in (+1, -1):
            cc = dict(c)
            cc["h"] = c["h"].copy()
            cc["h"][a] += s * e
            o2, n2 = o.neighbors(cc, 1)
            rs.append(o.density(cc, o2, n2)["rho"][a])
        fd = (rs[0] - rs[1]) / (2 * e)
        om = 1 + c["h"][a] / (3 * r["rho"][a]) * fd
        assert abs(om - r["omega"][a]) < 1e-7
    # mass scaling leaves Omega unchanged
    c2 = dict(c)
    c2["m"] = 2.0 * c["m"]
    r2 = o.density(c2, off, nbr)
    np.testing.assert_allclose(r2["omega"], r["omega"], rtol=1e-14)
    np.testing.assert_allclose(r2["rho"], 2 * r["rho"], rtol=1e-15)


def test_eos(O):
    d = lattice(5)
    o = mk(O, d, c0=3.0, rho0=1.0)
    off, nbr = o.neighbors(d, 1)
    r = o.density(d, off, nbr)
    np.testing.assert_allclose(r["p"], 9.0 * (r["rho"] - 1.0), rtol=1e-15, atol=1e-300)
    assert np.all(r["c"] == 3.0)
    o = mk(O, d, c0=3.0, rho0=float(r["rho"][0]))
    assert o.density(d, off, nbr)["p"][0] == 0.0
    oi = mk(O, d, eos="ideal", gamma=5 / 3)
    ri = oi.density(d, off, nbr)
    np.testing.assert_allclose(ri["p"], (2 / 3) * ri["rho"] * d["u"], rtol=1e-15)
    np.testing.assert_allclose(ri["c"], np.sqrt(5 / 3 * ri["p"] / ri["rho"]), rtol=1e-15)


# ------------------------------------------------------------------ O6 IAD

def test_iad_inverse_linear_field_and_lattice(O):
    d = lattice(13)
    o = mk(O, d)
    off, nbr = o.neighbors(d, 1)
    a = center_index(13)
    # survey value uses m_b / rho_b with rho_b = the lattice-interior density for every b
    C = o.iad(d, np.full(d["x"].size, GOLD["lattice_interior_rho"]), off, nbr)
    assert abs(C["c11"][a] - GOLD["lattice_interior_C"]) < 1e-13
    assert abs(C["c22"][a] - GOLD["lattice_interior_C"]) < 1e-13
    assert abs(C["c12"][a]) < 1e-15 and abs(C["c23"][a]) < 1e-15
    # jittered patch: C tau = I with tau built here in numpy through numpy.sinc
    c = I.jitter(I.square_patch(12, 12))
    o = mk(O, c)
    off, nbr = o.neighbors(c, 1)
    rho = o.density(c, off, nbr)["rho"]
    C = o.iad(c, rho, off, nbr)
    B = O.norm(6.0)
    L = c["box_hi"][2] - c["box_lo"][2]
    k = np.array([0.3, -1.7, 2.2])
    for a in range(0, c["x"].size, 97):
        nb = nbr[off[a]:off[a + 1]]
        D = np.stack([c["x"][nb] - c["x"][a], c["y"][nb] - c["y"][a], c["z"][nb] - c["z"][a]])
        D[2] = np.where(D[2] > L / 2, D[2] - L, np.where(D[2] < -L / 2, D[2] + L, D[2]))
        W = B * S_np(np.sqrt((D * D).sum(0)) / c["h"][a]) / c["h"][a] ** 3
        wt = c["m"][nb] / rho[nb] * W
        tau = (wt * D) @ D.T
        Cm = np.array([[C["c11"][a], C["c12"][a], C["c13"][a]],
                       [C["c12"][a], C["c22"][a], C["c23"][a]],
                       [C["c13"][a], C["c23"][a], C["c33"][a]]])
        np.testing.assert_allclose(Cm @ tau, np.eye(3), atol=1e-12)
        # linear field f = k.x reproduced exactly: sum_b V_b (f_b - f_a) A_ab = k
        A = (Cm @ D) * W
        grad = (wt / W * (k @ D)) @ A.T
        np.testing.assert_allclose(grad, k, rtol=1e-12, atol=1e-12)
    assert o.counters.iad_singular == 0


def test_iad_singular_fallback(O):
    # collinear neighbours: rank-1 tau -> isotropic fallback, counted (R29)
    d = lattice(1)
    for k in ("id", "x", "y", "z", "vx", "vy", "vz", "h", "m", "u"):
        d[k] = np.concatenate([d[k]] * 3)
    d["x"][:] = [0.0, 1.0, 2.0]
    d["h"][:] = 1.2
    o = mk(O, d)
    off, nbr = o.neighbors(d, 0)
    C = o.iad(d, np.ones(3), off, nbr)
    assert o.counters.iad_singular == 3
    assert C["c12"][0] == 0.0 and C["c11"][0] == C["c22"][0] == C["c33"][0] > 0


# ------------------------------------------------------------------ symmetric relation (8(f) NEXT-4)

@pytest.mark.parametrize("periodic", [(1, 0, 1), (0, 0, 0)])
def test_symmetric_neighbors_brute_force(O, periodic):
    """r < 2 max(h_a, h_b): brute force, both search methods, a true symmetric relation
    and a superset of the gather lists."""
    d = I.random_cloud(1200, box=8.0, h0=0.9, hspread=0.3, periodic=periodic, seed=11)
    ref = brute_numpy(d, symmetric=True)
    gat = brute_numpy(d)
    o = mk(O, d, symmetric=1)
    for method in (0, 1):
        off, nbr = o.neighbors(d, method)
        for a in range(d["x"].size):
            np.testing.assert_array_equal(nbr[off[a]:off[a + 1]], ref[a])
    pairs = {(a, b) for a in range(len(ref)) for b in ref[a]}
    assert all((b, a) in pairs for a, b in pairs)
    assert sum(len(s) for s in ref) > sum(len(s) for s in gat)  # variable h adds pairs
    assert all(set(g) <= set(s) for g, s in zip(gat, ref))


def test_symmetric_density_iad_unchanged(O):
    """Extra pairs (r >= 2 h_a) carry W(r, h_a) = 0 (compact support, Eq. 6): rho, Omega
    and C are the gather values."""
    d = I.random_cloud(1200, box=8.0, h0=0.9, hspread=0.3, periodic=(1, 0, 1), seed=12)
    out = []
    for sym in (0, 1):
        o = mk(O, d, symmetric=sym)
        off, nbr = o.neighbors(d, 1)
        dn = o.density(d, off, nbr)
        C = o.iad(d, dn["rho"], off, nbr)
        out.append((dn, C))
    for k in ("rho", "omega", "p"):
        np.testing.assert_allclose(out[1][0][k], out[0][0][k], rtol=1e-14, atol=0)
    for k in ("c11", "c12", "c13", "c22", "c23", "c33"):
        sc = np.abs(out[0][1]["c11"]) + np.abs(out[0][1]["c22"]) + np.abs(out[0][1]["c33"])
        assert np.max(np.abs(out[1][1][k] - out[0][1][k]) / sc) < 1e-13


def test_symmetric_conservation_variable_h(O):
    """Closes R24: with r < 2 max(h_a, h_b) every pair interacts both ways, so sum m a = 0
    and sum m (du + v.a) = 0 to round-off for variable h.  The gather relation on the
    same input does not conserve (the test is sensitive to the relation)."""
    d = I.random_cloud(1500, box=8.0, h0=0.9, hspread=0.3, periodic=(0, 0, 1), seed=13)
    d["vx"] = 0.3 * np.sin(d["y"])
    d["vy"] = -0.2 * d["x"]
    m = d["m"]
    res = {}
    for sym in (0, 1):
        r = _rates(O, d, symmetric=sym)[-1]
        mom = max(abs(np.sum(m * r[ax])) / np.sum(m * r["scale_a"][k])
                  for k, ax in enumerate(("ax", "ay", "az")))
        e = np.sum(m * (r["du"] + d["vx"] * r["ax"] + d["vy"] * r["ay"] + d["vz"] * r["az"]))
        sc = np.sum(m * (r["scale_du"] + np.abs(d["vx"]) * r["scale_a"][0] +
                         np.abs(d["vy"]) * r["scale_a"][1] + np.abs(d["vz"]) * r["scale_a"][2]))
        res[sym] = (mom, abs(e) / sc)
    assert res[1][0] < 1e-13 and res[1][1] < 1e-13
    assert res[0][0] > 1e-6 or res[0][1] > 1e-6


# ------------------------------------------------------------------ O7 momentum / energy

def _rates(O, d, **kw):
    o = mk(O, d, **kw)
    off, nbr = o.neighbors(d, 1)
    dn = o.density(d, off, nbr)
    C = o.iad(d, dn["rho"], off, nbr)
    return o, off, nbr, dn, C, o.momentum_energy(d, dn, C, off, nbr)


@pytest.mark.parametrize("case", ["cloud", "patch_rot", "patch_compress"])
def test_conservation_uniform_h(O, case):
    """Uniform h: sum m a = 0 and sum m (du + v.a) = 0 to round-off (Eqs. 2-4 with R1-R4).
    A dropped term, a wrong sign (R2) or rho instead of rho^2 (R1) fails this."""
    if case == "cloud":
        d = I.random_cloud(1200, box=7.0, h0=0.9, hspread=0.0, periodic=(0, 0, 1))
    else:
        d = I.jitter(I.square_patch(14, 10))
        if case == "patch_compress":
            d["vx"] = -0.5 * d["x"] * 5.0 + d["vx"]
            d["vy"] = -0.5 * d["y"] * 5.0 + d["vy"]
    o, off, nbr, dn, C, r = _rates(O, d)
    m = d["m"]
    for k, ax in enumerate(("ax", "ay", "az")):
        tot = np.sum(m * r[ax])
        assert abs(tot) < 1e-13 * np.sum(m * r["scale_a"][k])
    e = np.sum(m * (r["du"] + d["vx"] * r["ax"] + d["vy"] * r["ay"] + d["vz"] * r["az"]))
    sc = np.sum(m * (r["scale_du"] + np.abs(d["vx"]) * r["scale_a"][0] +
                     np.abs(d["vy"]) * r["scale_a"][1] + np.abs(d["vz"]) * r["scale_a"][2]))
    assert abs(e) < 1e-13 * sc
    # AV heating >= 0: rates with alpha=1 minus alpha=0
    r0 = _rates(O, d, alpha=0.0)[-1]
    assert np.sum(m * (r["du"] - r0["du"])) >= -1e-13 * sc
    if case == "patch_compress":
        assert np.sum(m * (r["du"] - r0["du"])) > 0


def test_head_on_pair_av_closed_form(O):
    """Isolated approaching pair, P = 0: v_sig = 2c + 3s, Pi' = (alpha/2)(2c+3s)s, decelerating
    (Eq. 5).  With the R29 isotropic C for a rank-1 tau, a_a,x = -3 Pi'/d."""
    d = lattice(1)
    for k in ("id", "x", "y", "z", "vx", "vy", "vz", "h", "m", "u"):
        d[k] = np.concatenate([d[k], d[k]])
    dd, s, c0 = 1.5, 0.8, 2.0
    d["x"][:] = [0.0, dd]
    d["vx"][:] = [0.5 * s, -0.5 * s]
    d["h"][:] = 1.0
    o = mk(O, d, c0=c0)
    off, nbr = o.neighbors(d, 0)
    dn = o.density(d, off, nbr)
    o = mk(O, d, c0=c0, rho0=float(dn["rho"][0]))  # P = 0 exactly
    dn = o.density(d, off, nbr)
    assert np.all(dn["p"] == 0.0)
    C = o.iad(d, dn["rho"], off, nbr)
    r = o.momentum_energy(d, dn, C, off, nbr)
    Pi = 0.5 * 1.0 * (2 * c0 + 3 * s) * s
    np.testing.assert_allclose(r["vsig"], [2 * c0 + 3 * s] * 2, rtol=1e-15)
    np.testing.assert_allclose(r["ax"], [-3 * Pi / dd, 3 * Pi / dd], rtol=1e-13)
    np.testing.assert_allclose(r["du"], [1.5 * s * Pi / dd] * 2, rtol=1e-13)
    # receding pair: no AV, no force, v_sig = 2c
    d["vx"][:] = [-0.5 * s, 0.5 * s]
    r = o.momentum_energy(d, dn, C, off, nbr)
    assert np.all(r["ax"] == 0.0) and np.all(r["du"] == 0.0)
    np.testing.assert_allclose(r["vsig"], [2 * c0] * 2)


def test_static_lattice_uniform_pressure_interior_force_free(O):
    d = lattice(13)
    o, off, nbr, dn, C, r = _rates(O, d, c0=10.0, rho0=0.5)
    a = center_index(13)
    for k, ax in enumerate(("ax", "ay", "az")):
        assert abs(r[ax][a]) < 1e-12 * r["scale_a"][k][a]
    assert r["du"][a] == 0.0


def test_pressure_is_repulsive(O):
    # compressed pair inside a uniform-P background: higher P pushes outward (R2/R5 sign)
    d = lattice(9)
    o, off, nbr, dn, C, r = _rates(O, d, c0=10.0, rho0=0.0)
    # boundary particles feel an outward push from the interior pressure
    a = 0  # corner (-4,-4,-4)
    assert r["ax"][a] < 0 and r["ay"][a] < 0 and r["az"][a] < 0


# ------------------------------------------------------------------ O8-O10

def test_timestep(O):
    d = lattice(7)
    o, off, nbr, dn, C, r = _rates(O, d, c0=4.0)
    dt = o.timestep(d["h"], r["vsig"], 0.0, True)
    assert dt == 0.3 * d["h"][0] / (2 * 4.0)
    assert o.timestep(0.5 * d["h"], r["vsig"], 0.0, True) == 0.5 * dt
    assert o.timestep(d["h"], r["vsig"], 0.5 * dt, False) == 1.1 * 0.5 * dt
    assert o.timestep(d["h"], r["vsig"], 10 * dt, False) == dt


def _traj(O, dts, a=np.array([1.3, -0.7, 0.25]), du=lambda t: 2.0, first_dt_prev=0.0):
    d = lattice(1)
    d["box_lo"][:] = -1e9
    d["box_hi"][:] = 1e9
    o = mk(O, d)
    st = {k: np.array([v], dtype=np.float64) for k, v in
          dict(x=0.1, y=0.2, z=0.3, vx=1.0, vy=-2.0, vz=0.5, u=1.0, vhx=0, vhy=0, vhz=0,
               du_prev=0).items()}
    t = 0.0
    dt_prev = first_dt_prev
    for i, dt in enumerate(dts):
        acc = {"ax": np.array([a[0]]), "ay": np.array([a[1]]), "az": np.array([a[2]]),
               "du": np.array([du(t)])}
        o.update(st, acc, dt, dt_prev, i == 0)
        dt_prev = dt
        t += dt
    return st, t


def test_update_constant_acceleration_exact(O):
    g = np.random.Generator(np.random.PCG64(I.SEED))
    dts = g.uniform(0.01, 0.1, 50)
    st, t = _traj(O, dts)
    a = np.array([1.3, -0.7, 0.25])
    x0 = np.array([0.1, 0.2, 0.3])
    v0 = np.array([1.0, -2.0, 0.5])
    np.testing.assert_allclose([st["x"][0], st["y"][0], st["z"][0]], x0 + v0 * t + 0.5 * a * t * t,
                               rtol=1e-13)
    np.testing.assert_allclose([st["vx"][0], st["vy"][0], st["vz"][0]], v0 + a * t, rtol=1e-13)
    assert abs(st["u"][0] - (1.0 + 2.0 * t)) < 1e-13  # AB2 exact on constant du


def test_update_ab2_linear_rate_and_order(O):
    # du = k t: after the Euler bootstrap every AB2 step is exact, so the total
    # error equals the first-step error k dt0^2 / 2
    k = 3.0
    g = np.random.Generator(np.random.PCG64(I.SEED + 1))
    dts = g.uniform(0.01, 0.05, 40)
    st, t = _traj(O, dts, du=lambda tt: k * tt)
    exact = 1.0 + 0.5 * k * t * t
    assert abs((exact - st["u"][0]) - 0.5 * k * dts[0] ** 2) < 1e-12
    # convergence order of positions on a smooth non-constant force: ratio ~ 4
    def run(n):
        # harmonic oscillator x'' = -x via repeated updates with a = -x
        d = lattice(1)
        o = mk(O, d, periodic=(0, 0, 0))
        st = {kk: np.array([v], dtype=np.float64) for kk, v in
              dict(x=1.0, y=0.0, z=0.0, vx=0.0, vy=0.0, vz=0.0, u=0.0, vhx=0, vhy=0, vhz=0,
                   du_prev=0).items()}
        dt = 1.0 / n
        for i in range(n):
            acc = {"ax": -st["x"].copy(), "ay": np.zeros(1), "az": np.zeros(1), "du": np.zeros(1)}
            o.update(st, acc, dt, dt, i == 0)
        return abs(st["x"][0] - math.cos(1.0))
    ratio = run(40) / run(80)
    assert 3.5 < ratio < 4.5


def test_update_h_rule(O):
    d = lattice(1)
    o = mk(O, d, n_target=300.0)
    h = np.array([1.0, 1.0, 1.0])
    off = np.array([0, 300, 300 + 2400, 300 + 2400 + 0], dtype=np.int64)
    o.update_h(h, off)
    assert h[0] == 1.0
    assert abs(h[1] - 0.75) < 1e-15
    assert abs(h[2] - 0.5 * (1 + 300 ** (1 / 3))) < 1e-14


def test_periodic_wrap_in_update(O):
    d = I.square_patch(4, 4)
    o = mk(O, d)
    st = {k: np.array([v], dtype=np.float64) for k, v in
          dict(x=0.0, y=0.0, z=49.9, vx=0.0, vy=0.0, vz=10.0, u=1.0, vhx=0, vhy=0, vhz=0,
               du_prev=0).items()}
    acc = {"ax": np.zeros(1), "ay": np.zeros(1), "az": np.zeros(1), "du": np.zeros(1)}
    o.update(st, acc, 0.1, 0.1, True)
    assert abs(st["z"][0] - (49.9 + 1.0 - 100.0)) < 1e-12
    # reading R30: a wrap that rounds onto the open end stays inside [lo, hi): z = -1e-15
    # in [0, 100) wraps to 100 - 1e-15, which rounds to 100.0 -> the largest double below 100
    d2 = dict(d, box_lo=np.array([-50.0, -50.0, 0.0]), box_hi=np.array([50.0, 50.0, 100.0]))
    o = mk(O, d2)
    st["z"][0], st["vz"][0] = 0.0, -1e-15
    o.update(st, acc, 1.0, 1.0, True)
    assert st["z"][0] == np.nextafter(100.0, 0.0)
    # a wrap from above that would round below lo is kept at lo
    st["z"][0], st["vz"][0] = np.nextafter(100.0, 0.0), 1e-14
    o.update(st, acc, 1.0, 1.0, True)
    assert 0.0 <= st["z"][0] < 100.0


# ------------------------------------------------------------------ O11 + ICs + config 1

def test_diagnostics_and_initial_angular_momentum(O):
    from math import fsum
    for n in (20,):
        d = I.square_patch(n)
        diag = O.Oracle.diagnostics(d)
        assert abs(diag[0]) < 1e-9 and abs(diag[1]) < 1e-9
        Lz = -5.0 * 1.0 * 100.0 ** 5 * (n * n - 1) / (6 * n * n)  # closed form (SURVEY §8c ICs)
        assert abs(diag[5] - Lz) < 1e-12 * abs(Lz)
        assert abs(abs(diag[5]) - GOLD["Lz_abs"][str(n)]) < 1e-12 * GOLD["Lz_abs"][str(n)]
        E = fsum(d["m"] * (d["u"] + 0.5 * (d["vx"] ** 2 + d["vy"] ** 2)))
        assert abs(diag[6] - E) < 1e-14 * E


def test_config1_regression(O):
    d = I.square_patch(20)
    o = mk(O, d)
    r = o.step(d)
    dn = r["dens"]
    assert dn["rho"].min() == pytest.approx(GOLD["rho_over_rho0_min"], abs=1e-4)
    assert dn["rho"].max() == pytest.approx(GOLD["rho_over_rho0_max"], abs=1e-6)
    assert dn["p"].min() == pytest.approx(GOLD["p_min"], rel=1e-3)
    assert dn["p"].max() == pytest.approx(GOLD["p_max"], rel=1e-3)
    assert dn["omega"].min() == pytest.approx(GOLD["omega_min"], abs=1e-3)
    assert r["dt"] == pytest.approx(GOLD["dt"], rel=1e-6)
    assert r["dt"] == 0.3 * d["h"][0] / (2 * d["c0"])
    assert o.counters.omega_clamped == 0 and o.counters.iad_singular == 0


def test_inputs_pins():
    d = I.square_patch(20)
    assert d["x"].size == 8000
    assert I.h_for_lattice(1.0) == pytest.approx(GOLD["h_over_dx"], rel=1e-15)
    e = I.evrard(124)
    assert e["x"].size == 998592
    p = I.square_patch(20, pressure_ics=True, series_terms=80)
    assert p["m"].min() > 0
    # P0 at patch edge = 0, symmetric in x <-> y
    from paper_2005_02656_b200.inputs import _p0_series
    xs = np.array([0.0, 50.0, 100.0])
    P = _p0_series(xs, xs, 100.0, 5.0, 1.0, 80)
    assert abs(P[0, 1]) < 1e-9 and abs(P[1, 2]) < 1e-6
    assert P[1, 1] == pytest.approx(-36835.66, rel=2e-5)
    np.testing.assert_allclose(P, P.T, rtol=1e-12, atol=1e-9)


def test_rotation_and_galilean_covariance(O):
    """Rotating the whole (open-boundary) cloud rotates a and C (a' = R a, C' = R C R^T) and
    leaves rho, du unchanged; a uniform velocity boost changes nothing.  A transposed or
    misplaced C entry in A_ab = C Delta W, or v_a used for v_ab, fails here even when
    conservation still holds."""
    d = I.random_cloud(900, box=6.0, h0=0.85, hspread=0.15, periodic=(0, 0, 0), seed=11)
    o, off, nbr, dn, C, r = _rates(O, d)
    g = np.random.Generator(np.random.PCG64(I.SEED + 5))
    Q, _ = np.linalg.qr(g.normal(size=(3, 3)))
    X = Q @ np.stack([d["x"], d["y"], d["z"]])
    V = Q @ np.stack([d["vx"], d["vy"], d["vz"]])
    d2 = dict(d, x=X[0].copy(), y=X[1].copy(), z=X[2].copy(), vx=V[0].copy(), vy=V[1].copy(),
              vz=V[2].copy(), box_lo=np.full(3, -50.0), box_hi=np.full(3, 50.0))
    o2, off2, nbr2, dn2, C2, r2 = _rates(O, d2)
    np.testing.assert_array_equal(off2, off)
    np.testing.assert_array_equal(nbr2, nbr)
    np.testing.assert_allclose(dn2["rho"], dn["rho"], rtol=1e-12)
    A = np.stack([r["ax"], r["ay"], r["az"]])
    A2 = np.stack([r2["ax"], r2["ay"], r2["az"]])
    scale = np.linalg.norm(r["scale_a"], axis=0)
    assert np.max(np.abs(A2 - Q @ A) / scale) < 1e-11
    assert np.max(np.abs(r2["du"] - r["du"]) / r["scale_du"]) < 1e-11
    Cm = np.array([[C["c11"], C["c12"], C["c13"]], [C["c12"], C["c22"], C["c23"]],
                   [C["c13"], C["c23"], C["c33"]]]).transpose(2, 0, 1)
    Cm2 = np.array([[C2["c11"], C2["c12"], C2["c13"]], [C2["c12"], C2["c22"], C2["c23"]],
                    [C2["c13"], C2["c23"], C2["c33"]]]).transpose(2, 0, 1)
    np.testing.assert_allclose(Cm2, Q @ Cm @ Q.T, rtol=1e-9, atol=1e-9 * np.abs(Cm).max())
    # Galilean boost
    d3 = dict(d, vx=d["vx"] + 3.0, vy=d["vy"] - 1.0, vz=d["vz"] + 0.5)
    r3 = _rates(O, d3)[-1]
    A3 = np.stack([r3["ax"], r3["ay"], r3["az"]])
    assert np.max(np.abs(A3 - A) / scale) < 1e-11
    assert np.max(np.abs(r3["du"] - r["du"]) / r["scale_du"]) < 1e-11
