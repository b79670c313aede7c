"""T0 pins of the oracle's parity scales and of the R29 threshold (-m "not gpu").

The GPU parity bounds are 1e-10 x a scale the oracle exports (reading R27):
omega_scale = 1 + h/(3 rho) sum_b |m_b dW/dh| (Omega), scale_a / scale_du =
sum_b |summand| (a, du).  A slip in one of them would silently loosen every
parity test that uses it, so each is pinned here against a closed form that
does not call the oracle's own expression:

* isolated particle: omega_scale = 1 + (h/(3 m B/h^3)) * 3 m B/h^4 = 2 exactly;
* close pair (every dW/dh term negative): omega_scale = 2 - Omega_unclamped, with
  Omega from Eq. 6's closed-form derivative v S'(v) = n sinc^(n-1) (cos x - sinc x);
* single-pair configurations whose pair terms carry no internal cancellation:
  scale_a = |a| and scale_du = |du| exactly (head-on pair with AV, P = 0; receding
  pair with P > 0, no AV);
* every configuration: scale >= |value| (a sum of magnitudes bounds the sum).

R29 (singular / ill-conditioned tau -> isotropic C) is pinned on both sides of its
1e12 Frobenius-condition threshold with a near-planar neighbourhood whose tau is
built independently in numpy: cond ~1e6 must keep C = tau^-1, cond ~1e14 must fall
back.
"""
import math

import numpy as np
import pytest

from paper_2005_02656_b200 import inputs as I
from tests.test_oracle import S_np, lattice, mk


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


def _pair(dd, h=1.0, m=1.0):
    d = lattice(1)
    for k in ("id", "x", "y", "z", "vx", "vy", "vz", "h", "m", "u"):
        d[k] = np.concatenate([d[k], d[k]])
    d["id"] = np.arange(2)
    d["x"][:] = [0.0, dd]
    d["h"][:] = h
    d["m"][:] = m
    return d


def vdS_closed(v, n=6.0):
    """v dS/dv of S = sinc(x)^n, x = pi v / 2:  n sinc^(n-1) (cos x - sinc x)."""
    x = 0.5 * math.pi * v
    s = math.sin(x) / x
    return n * s ** (n - 1) * (math.cos(x) - s)


def test_omega_scale_isolated_particle(O):
    d = lattice(1)
    o = mk(O, d)
    off, nbr = o.neighbors(d, 0)
    dn = o.density(d, off, nbr)
    # Omega = 1 + h/(3 rho) m dW/dh(0) = 1 - 1 = 0 -> clamped 0.1; scale = 2
    assert dn["omega"][0] == 0.1
    assert abs(dn["omega_scale"][0] - 2.0) < 1e-15


@pytest.mark.parametrize("v", [0.15, 0.3, 0.55])
def test_omega_scale_close_pair(O, v):
    n = 6.0
    d = _pair(v)  # h = 1: r/h = v
    o = mk(O, d, omega_mode=0)
    off, nbr = o.neighbors(d, 0)
    dn = o.density(d, off, nbr)
    S = float(S_np(v, n))
    vdS = vdS_closed(v, n)
    assert 3 * S + vdS > 0  # every m dW/dh term negative: no cancellation inside the sum
    # rho = m B (1 + S) / h^3; sum m dW/dh = -m B (3 + 3 S + v S') / h^4
    om_unclamped = 1.0 - (3.0 + 3.0 * S + vdS) / (3.0 * (1.0 + S))
    scale = 1.0 + (3.0 + 3.0 * S + vdS) / (3.0 * (1.0 + S))
    np.testing.assert_allclose(dn["omega_scale"], [scale, scale], rtol=1e-13)
    assert abs(scale - (2.0 - om_unclamped)) < 1e-15
    assert np.all(dn["omega_scale"] >= np.abs(om_unclamped))


def test_scales_equal_magnitudes_head_on_pair(O):
    """P = 0, approaching: every summand is the AV term, one pair -> scale = |value|."""
    dd, s, c0 = 1.5, 0.8, 2.0
    d = _pair(dd)
    d["vx"][:] = [0.5 * s, -0.5 * s]
    o = mk(O, d, c0=c0)
    off, nbr = o.neighbors(d, 0)
    dn = o.density(d, off, nbr)
    o = mk(O, d, c0=c0, rho0=float(dn["rho"][0]))  # P = 0 exactly
    dn = o.density(d, off, nbr)
    C = o.iad(d, dn["rho"], off, nbr)
    r = o.momentum_energy(d, dn, C, off, nbr)
    assert np.all(r["ax"] != 0.0) and np.all(r["du"] > 0.0)
    np.testing.assert_allclose(r["scale_a"][0], np.abs(r["ax"]), rtol=1e-15)
    assert np.all(r["scale_a"][1:] == 0.0)
    np.testing.assert_allclose(r["scale_du"], np.abs(r["du"]), rtol=1e-15)


def test_scales_equal_magnitudes_receding_pressure_pair(O):
    """P > 0 (rho0 = 0), alpha = 0 (the scale's AV bound covers receding pairs too, R28):
    a = -m (X_a A_a + X_b A_b) with equal signs, du = m X_a v_ab.A_a -> scale = |value|."""
    dd, s = 1.2, 0.6
    d = _pair(dd)
    d["vx"][:] = [-0.5 * s, 0.5 * s]
    o = mk(O, d, c0=3.0, rho0=0.0, alpha=0.0)
    off, nbr = o.neighbors(d, 0)
    dn = o.density(d, off, nbr)
    assert np.all(dn["p"] > 0)
    C = o.iad(d, dn["rho"], off, nbr)
    r = o.momentum_energy(d, dn, C, off, nbr)
    assert np.all(r["ax"] != 0.0) and np.all(r["du"] != 0.0)
    np.testing.assert_allclose(r["scale_a"][0], np.abs(r["ax"]), rtol=1e-15)
    np.testing.assert_allclose(r["scale_du"], np.abs(r["du"]), rtol=1e-15)


@pytest.mark.parametrize("case", ["patch_rot", "cloud"])
def test_scales_bound_values(O, case):
    if case == "patch_rot":
        d = I.square_patch(12, 8)
    else:
        d = I.random_cloud(900, box=6.0, h0=0.9, hspread=0.2, periodic=(1, 0, 1))
    o = mk(O, d)
    off, nbr = o.neighbors(d, 1)
    dn = o.density(d, off, nbr)
    C = o.iad(d, dn["rho"], off, nbr)
    r = o.momentum_energy(d, dn, C, off, nbr)
    for k, ax in enumerate(("ax", "ay", "az")):
        assert np.all(r["scale_a"][k] >= np.abs(r[ax]) * (1 - 1e-14))
    assert np.all(r["scale_du"] >= np.abs(r["du"]) * (1 - 1e-14))
    assert np.all(dn["omega_scale"] >= 1.0)
    # rotation at t = 0 makes du pure round-off (R27): the scale must not be that small
    if case == "patch_rot":
        assert np.median(r["scale_du"]) > 1e6 * np.median(np.abs(r["du"]))


def _planar(delta):
    """Target 0 at the origin; neighbours: a 5x5 planar grid (z = 0, spacing 0.5) and two
    particles at z = +-delta.  Every other particle has a tiny h (no neighbours)."""
    g = (np.arange(5) - 2) * 0.5
    X, Y = np.meshgrid(g, g, indexing="ij")
    pts = [(0.0, 0.0, 0.0)] + [(a, b, 0.0) for a, b in zip(X.ravel(), Y.ravel()) if a or b]
    pts += [(0.0, 0.0, delta), (0.0, 0.0, -delta)]
    P = np.array(pts)
    N = P.shape[0]
    d = lattice(1)
    for k in ("vx", "vy", "vz", "m", "u"):
        d[k] = np.full(N, d[k][0])
    d["id"] = np.arange(N)
    d["x"], d["y"], d["z"] = P[:, 0].copy(), P[:, 1].copy(), P[:, 2].copy()
    d["h"] = np.full(N, 1e-3)
    d["h"][0] = 1.0  # 2h = 2 > max distance sqrt(2)
    return d


def _tau_numpy(d):
    """tau_0 = sum_b (m_b/rho_b) W(r, h_0) Delta Delta^T with rho = 1, W via numpy's sinc."""
    D = np.stack([d["x"][1:], d["y"][1:], d["z"][1:]])
    r = np.sqrt((D * D).sum(0))
    W = S_np(r / d["h"][0])  # B / h^3 factor common -> scaled below
    return D, W


@pytest.mark.parametrize("cond_target,fallback", [(1e6, False), (1e14, True)])
def test_r29_threshold_near_planar(O, cond_target, fallback):
    B = O.norm(6.0)
    # calibrate delta: tau_zz ~ 2 W delta^2 while the in-plane block is fixed
    d0 = _planar(0.1)
    D, W = _tau_numpy(d0)
    tau0 = B * (W * D) @ D.T
    c0 = np.linalg.norm(tau0) * np.linalg.norm(np.linalg.inv(tau0))
    delta = 0.1 * math.sqrt(c0 / cond_target)
    d = _planar(delta)
    D, W = _tau_numpy(d)
    tau = B * (W * D) @ D.T  # h_0 = 1, m = rho = 1
    cond = np.linalg.norm(tau) * np.linalg.norm(np.linalg.inv(tau))
    assert cond_target / 10 < cond < cond_target * 10
    o = mk(O, d)
    off, nbr = o.neighbors(d, 0)
    assert off[1] - off[0] == d["x"].size - 1
    C = o.iad(d, np.ones(d["x"].size), off, nbr)
    Cm = np.array([[C["c11"][0], C["c12"][0], C["c13"][0]],
                   [C["c12"][0], C["c22"][0], C["c23"][0]],
                   [C["c13"][0], C["c23"][0], C["c33"][0]]])
    iso = 3.0 / np.trace(tau)
    if fallback:
        np.testing.assert_allclose(np.diag(Cm), [iso] * 3, rtol=1e-12)
        assert C["c12"][0] == C["c13"][0] == C["c23"][0] == 0.0
    else:
        inv = np.linalg.inv(tau)
        np.testing.assert_allclose(Cm, inv, rtol=1e-7, atol=1e-7 * np.abs(inv).max())
        assert abs(Cm[2, 2] - iso) > 1e3 * iso  # far from the fallback value
