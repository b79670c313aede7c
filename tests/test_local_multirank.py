"""The multi-rank path (a4 halo #1, a7 halo #2, a9 halo #3, a14 migration, the bbox /
histogram / dt / diagnostics reductions) on ONE GPU (-m gpu).

G ranks run as G host threads of this process, each with its own sph_ctx and stream,
joined by the library's in-process transport (sph_local_comm_id, comm.cuh) instead of
NCCL; everything else -- splitters, migration, halo plan, pack / unpack, the exchanges
-- is the code the NCCL runs execute.  Each rank attaches a scrambled subset (ids
round-robin over ranks) so the first step migrates almost every particle.

Checks:
* per call, against the ORACLE on the gathered global state: every rank's neighbour
  rows (bit-exact global-id sets, halo neighbours included), rho/Omega/P/c, C, a, du,
  v_sig, dt (tolerances of tests/parity_util.py);
* over several steps, bit-identity of the gathered state with a 1-rank run (the
  rank-independence property), and the all-reduced diagnostics.
"""
import threading

import numpy as np
import pytest

from paper_2005_02656_b200 import inputs as I
from tests import parity_util as U

pytestmark = pytest.mark.gpu

FIELDS = ("x", "y", "z", "vx", "vy", "vz", "h", "u", "m", "rho", "omega", "p", "c", "c11", "c12",
          "c13", "c22", "c23", "c33", "ax", "ay", "az", "du", "vsig")


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


def run_ranks(sims, fn):
    """fn(rank, sim) on every rank concurrently (the collectives are rendezvous)."""
    out, err = [None] * len(sims), []

    def body(r):
        try:
            out[r] = fn(r, sims[r])
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(len(sims))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out


def make_ranks(S, d, G, **kw):
    import torch
    uid = S.local_comm_id(G)
    cap = int(d["x"].size * 1.2) + 1024
    sims, streams = [], []
    for r in range(G):
        st = torch.cuda.Stream()
        streams.append(st)
        mine = I.subset(d, np.arange(r, d["x"].size, G))
        sims.append(S.Simulation(mine, capacity=cap, rank=r, nranks=G, unique_id=uid,
                                 stream=st.cuda_stream, **kw))
    return sims, streams


def gather(sims, fields=FIELDS):
    parts = [s.state() for s in sims]
    out = {k: np.concatenate([p[k] for p in parts]) for k in ("id",) + tuple(fields)}
    o = np.argsort(out["id"], kind="stable")
    return {k: v[o] for k, v in out.items()}


CASES = {
    "patch_p0": lambda: I.square_patch(24, 24, pressure_ics=True),
    "jitter": lambda: I.jitter(I.square_patch(20, 16)),
    "evrard": lambda: I.evrard(30),
    "cloud_sym": lambda: I.random_cloud(6000, box=12.0, h0=0.8, hspread=0.3, periodic=(1, 0, 1), seed=3),
}


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("case", list(CASES))
def test_multirank_per_call_vs_oracle(S, O, case, G):
    import torch
    d = CASES[case]()
    kw = {"symmetric": 1} if case == "cloud_sym" else {}
    sims, streams = make_ranks(S, d, G, **kw)
    run_ranks(sims, lambda r, s: s.find_neighbors())
    nown = [s.n for s in sims]
    assert sum(nown) == d["x"].size and all(n > 0 for n in nown)
    halos = [s.n_halo for s in sims]
    assert all(h > 0 for h in halos), halos  # every rank has a halo (a4 ran)
    # the global state after migration + sort (positions unchanged by find_neighbors)
    st = U.with_meta(gather(sims, ("x", "y", "z", "vx", "vy", "vz", "h", "m", "u")), d)
    assert np.array_equal(st["id"], np.sort(d["id"]))
    o, off, nbr, dn, C, me = U.oracle_pipeline(O, st, symmetric=kw.get("symmetric", 0))
    pos = {int(i): k for k, i in enumerate(st["id"])}
    # every rank's rows (its owned targets, global ids incl. halo neighbours), bit-exact
    for s in sims:
        off_g, ids_g = s.get_neighbors()
        own = s.state()["id"]
        idx = np.array([pos[int(i)] for i in own])
        ref_off = np.concatenate([[0], np.cumsum(off[idx + 1] - off[idx])])
        ref_ids = np.concatenate([st["id"][nbr[off[a]:off[a + 1]]] for a in idx]) if idx.size else []
        U.assert_neighbors_equal(off_g, ids_g, ref_off, np.asarray(ref_ids, dtype=np.int64))
    run_ranks(sims, lambda r, s: s.density())
    run_ranks(sims, lambda r, s: s.iad())
    dts = run_ranks(sims, lambda r, s: s.momentum_energy(want_dt=True))
    for st_ in streams:
        st_.synchronize()
    g = gather(sims)
    U.check_density(g, dn, d)
    U.check_iad(g, C)
    U.check_momentum(g, me)
    dt_o = o.timestep(st["h"], me["vsig"], 0.0, True)
    assert len(set(dts)) == 1 and abs(dts[0] - dt_o) <= 1e-12 * dt_o  # a11: NCCL-MIN twin
    run_ranks(sims, lambda r, s: s.advance())
    torch.cuda.synchronize()


@pytest.mark.parametrize("G,case,redecomp", [(2, "patch_p0", 1), (4, "jitter", 1), (3, "evrard", 1),
                                             (4, "cloud_sym", 1), (4, "jitter", 3)])
def test_multirank_steps_bit_identical(S, O, G, case, redecomp):
    """4 full steps on G ranks == 1 rank bit for bit (every field, every dt), and the
    all-reduced diagnostics (a15) equal the oracle's O11 on the gathered state."""
    d = CASES[case]()
    kw = {"symmetric": 1} if case == "cloud_sym" else {}
    sims, streams = make_ranks(S, d, G, redecomp_every=redecomp, **kw)
    cap = int(d["x"].size * 1.2) + 1024
    ref = S.Simulation(d, capacity=cap, **kw)
    for step in range(4):
        dts = run_ranks(sims, lambda r, s: s.step(want_dt=True))
        rdt = ref.step(want_dt=True)
        assert len(set(dts)) == 1 and dts[0] == rdt, (step, dts, rdt)
    diags = run_ranks(sims, lambda r, s: s.diagnostics())
    got = gather(sims)
    rst = ref.state()
    o = np.argsort(rst["id"])
    for k in ("id",) + FIELDS:
        assert np.array_equal(got[k], rst[k][o]), k
    rd = ref.diagnostics()
    for dg in diags:
        assert dg["n_owned"] == d["x"].size and dg["nbr_total"] == rd["nbr_total"]
        assert dg["steps"] == 4
    ref_o11 = O.Oracle.diagnostics(got)
    m = got["m"]
    vmag = np.abs(got["vx"]) + np.abs(got["vy"]) + np.abs(got["vz"])
    rmag = np.abs(got["x"]) + np.abs(got["y"]) + np.abs(got["z"])
    scale_p = np.sum(m * vmag) + 1e-300
    scale_l = np.sum(m * rmag * vmag) + 1e-300
    scale_e = np.sum(m * (np.abs(got["u"]) + vmag ** 2)) + 1e-300
    dg = diags[0]
    for k in range(3):
        assert abs(dg["momentum"][k] - ref_o11[k]) <= 1e-12 * scale_p
        assert abs(dg["ang_momentum"][k] - ref_o11[3 + k]) <= 1e-12 * scale_l
    assert abs(dg["energy"] - ref_o11[6]) <= 1e-12 * scale_e
