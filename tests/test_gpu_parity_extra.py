"""More GPU <-> oracle parity through the C ABI (-m gpu): the configurations the
default cases leave out.

* a15 conserved sums: sph_diagnostics against the oracle's O11;
* kernel exponents n = 4, 8 (the generic N = 0 template of every pair kernel; R9);
* Omega == 1 mode and alpha != 1 (R7, R8);
* the h / u clamps of the update, counters equal;
* ragged tiny sets (n = 1, 2, 33, 257) through the whole pipeline against the
  brute-force oracle (method 0);
* config 2 (1M particles, BASELINE configs[1]): every particle of one step, and the
  20-step shadowed run (the oracle re-synced from the GPU state each step).
"""
import numpy as np
import pytest

from paper_2005_02656_b200 import inputs as I
from tests import parity_util as U
from tests.test_gpu_parity import per_call_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2005_02656_b200 import _build, sph
    _build.build()
    return sph


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


@pytest.mark.parametrize("case", ["patch", "cloud"])
def test_diagnostics_parity(S, O, case):
    """sum m v, sum m x cross v, sum m (u + v^2/2) after two steps (a15): same state,
    GPU block sums vs the oracle's fixed-order pairwise sums, |d| <= 1e-12 sum |terms|."""
    d = (I.square_patch(20) if case == "patch" else
         I.random_cloud(3000, box=9.0, h0=0.8, hspread=0.2, periodic=(1, 0, 1)))
    sim = S.Simulation(d)
    sim.step()
    sim.step()
    g = sim.diagnostics()
    st = sim.state()
    ref = O.Oracle.diagnostics(st)
    m, x, y, z = st["m"], st["x"], st["y"], st["z"]
    vx, vy, vz, u = st["vx"], st["vy"], st["vz"], st["u"]
    mag = [np.sum(np.abs(m * vx)), np.sum(np.abs(m * vy)), np.sum(np.abs(m * vz)),
           np.sum(np.abs(m * y * vz)) + np.sum(np.abs(m * z * vy)),
           np.sum(np.abs(m * z * vx)) + np.sum(np.abs(m * x * vz)),
           np.sum(np.abs(m * x * vy)) + np.sum(np.abs(m * y * vx)),
           np.sum(np.abs(m * (u + 0.5 * (vx * vx + vy * vy + vz * vz))))]
    got = list(g["momentum"]) + list(g["ang_momentum"]) + [g["energy"]]
    for k in range(7):
        assert abs(got[k] - ref[k]) <= 1e-12 * mag[k] + 1e-300, (k, got[k], ref[k])
    assert g["steps"] == 2 and g["n_owned"] == d["x"].size
    assert g["nbr_total"] > 0


@pytest.mark.parametrize("n", [4.0, 8.0])
@pytest.mark.parametrize("case", ["jitter", "cloud"])
def test_kernel_exponent(S, O, n, case):
    d = (I.shuffled(I.jitter(I.square_patch(14, 10))) if case == "jitter" else
         I.random_cloud(3000, box=9.0, h0=0.8, hspread=0.2, periodic=(1, 0, 1)))
    per_call_parity(S, O, d, oracle_kw={"n": n}, n=n)


def test_omega_one_and_alpha(S, O):
    d = I.random_cloud(3000, box=9.0, h0=0.8, hspread=0.2, periodic=(1, 0, 1), seed=7)
    per_call_parity(S, O, d, oracle_kw={"omega_mode": 1, "alpha": 0.37}, omega_mode=1, alpha=0.37)
    d = I.jitter(I.square_patch(14, 10))
    per_call_parity(S, O, d, oracle_kw={"alpha": 2.5}, alpha=2.5)


def test_update_clamps_counted(S, O):
    """Ideal-gas random cloud (du != 0): u floor and h range clamps, applied and counted like
    the oracle."""
    d = I.random_cloud(3000, box=9.0, h0=0.8, hspread=0.2, periodic=(1, 0, 1), seed=9)
    d["eos"] = "ideal"
    kw = {"u_floor": 1.0, "h_min": 0.7, "h_max": 0.9}
    sim, o = per_call_parity(S, O, d, oracle_kw=kw, **kw)
    g = sim.diagnostics()
    assert g["u_floored"] == o.counters.u_floored > 0
    assert g["h_clamped"] == o.counters.h_clamped > 0
    assert g["omega_clamped"] == o.counters.omega_clamped


@pytest.mark.parametrize("n", [1, 2, 33, 257])
def test_ragged_small_full_pipeline_brute_force(S, O, n):
    """Every output of the pipeline for tiny ragged sets (not warp or tile multiples) against
    the brute-force oracle (O1 method 0)."""
    d = I.random_cloud(n, box=3.0, h0=0.9, periodic=(0, 0, 1), seed=n)
    per_call_parity(S, O, d, method=0)


def test_config2_every_particle(S, O):
    """BASELINE configs[1] (1M square patch) at full size: every particle, every output."""
    per_call_parity(S, O, I.square_patch(100))


def shadowed(S, O, d, steps):
    """`steps` timesteps; before each, the oracle is re-synced from the GPU state and
    runs the same step on its own: rates, dt and the new state are compared per particle."""
    sim = S.Simulation(d)
    dt_prev, first = 0.0, True
    for step in range(steps):
        st = U.with_meta(sim.state(), d)
        st["dt_prev"], st["first"] = dt_prev, first
        o = O.Oracle(O.Params.from_inputs(st))
        r = o.step(st)
        dt = sim.step(want_dt=True)
        after = sim.state()
        pos = np.argsort(after["id"])
        ref = np.argsort(st["id"])
        g = {k: after[k][pos] for k in after}
        U.check_density(g, {k: v[ref] for k, v in r["dens"].items()}, d)
        acc = {k: (v[:, ref] if k == "scale_a" else v[ref]) for k, v in r["acc"].items()}
        U.check_momentum(g, acc)
        assert abs(dt - r["dt"]) <= 1e-12 * r["dt"], (step, dt, r["dt"])
        rs = {k: r["state"][k][ref] for k in ("x", "y", "z", "vx", "vy", "vz", "u", "h")}
        L = float(np.max(np.asarray(d["box_hi"]) - np.asarray(d["box_lo"])))
        for k in ("x", "y", "z"):
            assert np.max(np.abs(g[k] - rs[k])) <= 1e-12 * L, (step, k)
        for k in ("vx", "vy", "vz"):
            vs = np.abs(rs["vx"]) + np.abs(rs["vy"]) + np.abs(rs["vz"]) + 1.0
            assert np.all(np.abs(g[k] - rs[k]) <= 1e-9 * vs), (step, k)
        assert np.max(np.abs(g["h"] - rs["h"]) / rs["h"]) <= 1e-14
        dt_prev, first = dt, False
    return sim


def test_shadowed_20_steps_config2(S, O):
    """BASELINE configs[1]: square patch 100^3 = 1M particles, 20 timesteps."""
    sim = shadowed(S, O, I.square_patch(100), 20)
    diag = sim.diagnostics()
    assert diag["steps"] == 20 and diag["iad_singular"] == 0


def test_config3_every_particle(S, O):
    """BASELINE configs[2] (Evrard-shaped sphere, 1M, variable h, ideal gas): every particle."""
    per_call_parity(S, O, I.evrard(124))


def test_nonfinite_input_and_dt_reported(S, O):
    """S:90 / S:274: a NaN h is reported with its particle id; an invalid dt (ideal gas at
    u = 0: c = 0, v_sig = 0, dt = inf) leaves the state untouched even without a host read
    of dt, and the next call fails with SPH_ERR_NUMERIC."""
    d = I.random_cloud(500, box=4.0, h0=0.9, seed=4)
    d["h"][123] = np.nan
    sim = S.Simulation(d)
    with pytest.raises(S.SphError) as e:
        sim.find_neighbors()
    assert e.value.status == 1
    g = sim.diagnostics(check=False)
    assert g["status"] == 1 and g["first_bad_id"] == int(d["id"][123])
    d = I.random_cloud(500, box=4.0, h0=0.9, seed=4, vscale=0.0)
    d["eos"] = "ideal"
    d["u"][:] = 0.0
    sim = S.Simulation(d)
    before = sim.state()
    sim.step()  # dt_out == NULL: no host check inside the call
    after = sim.state()
    o = np.argsort(before["id"])
    a = np.argsort(after["id"])
    for k in ("x", "y", "z", "vx", "u"):
        assert np.array_equal(before[k][o], after[k][a]), k
    with pytest.raises(S.SphError) as e:
        sim.step()
    assert e.value.status == 1


def test_wide_rows_unit_stencil_over_65535(S, O, monkeypatch, capfd):
    """A unit stencil above 65,535 particles cannot be addressed by 16-bit flat indices:
    the search reports it, the library reallocates 32-bit rows and reruns (R23: rows
    are never truncated), and every output -- lists, rho, C, a, du, the update -- still
    matches the oracle.  cell_factor 20 puts a 68,000-particle cloud (~60 neighbours
    each) in one unit, so the 32-bit instantiations of the search, the row expansion
    and the three pair passes all run."""
    monkeypatch.setenv("SPH_DEBUG_ROWS", "1")
    d = I.random_cloud(68000, box=10.0, h0=0.3, hspread=0.1, periodic=(0, 0, 0), seed=11)
    per_call_parity(S, O, d, cell_factor=20.0)
    err = capfd.readouterr().err
    assert "wide 1" in err, err[-500:]


def test_rows_grow_past_initial_stride(S, O, monkeypatch, capfd):
    """~700 neighbours per particle: longer than the initial 384-entry row stride, so the
    search reports the overflow, the rows are reallocated at the larger stride and the
    search reruns (R23: never truncated); every output matches the oracle."""
    monkeypatch.setenv("SPH_DEBUG_ROWS", "1")
    d = I.random_cloud(6000, box=10.0, h0=1.5, hspread=0.1, periodic=(1, 1, 1), seed=5)
    per_call_parity(S, O, d)
    err = capfd.readouterr().err
    assert "rows grow (max count" in err, err[-500:]
