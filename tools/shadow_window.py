"""Shadow a window of a long GPU run with the CPU oracle (test aid, uses oracle/):
integrate the 100^3 rotating patch on the GPU to step S0, then for K more steps re-run
each GPU step on the oracle from the GPU's own state and compare rates, dt and the new
state (the parity bars of tests/parity_util.py, reported instead of asserted).

    python tools/shadow_window.py --n 100 --s0 3950 --k 12 --out gpurun_out/shadow.json

Used to attribute the late energy growth of the 100^3 validation run:
if every GPU step in the growth window matches the oracle's step of the same state,
the growth is what the method (as read from the paper) does, not a kernel defect."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import oracle as O
    from paper_2005_02656_b200 import inputs, sph
    from tests import parity_util as U
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--s0", type=int, default=3950)
    ap.add_argument("--k", type=int, default=12)
    ap.add_argument("--symmetric", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "shadow.json"))
    a = ap.parse_args()
    O.build()
    d = inputs.square_patch(a.n, pressure_ics=True)
    sim = sph.Simulation(d, symmetric=a.symmetric)
    dt_prev = 0.0
    for _ in range(a.s0):
        dt_prev = sim.step(want_dt=True)
    rows = []
    for k in range(a.k):
        st = U.with_meta(sim.state(), d)
        st["dt_prev"], st["first"] = dt_prev, False
        # the GPU's integrator history (v-bar, du_prev) is part of the state
        o = O.Oracle(O.Params.from_inputs(st, symmetric=a.symmetric))
        r = o.step(st)
        dt = sim.step(want_dt=True)
        after = sim.state()
        pos, ref = np.argsort(after["id"]), np.argsort(st["id"])
        g = {kk: v[pos] for kk, v in after.items()}
        dn = {kk: v[ref] for kk, v in r["dens"].items()}
        acc = {kk: (v[:, ref] if kk == "scale_a" else v[ref]) for kk, v in r["acc"].items()}
        err = {
            "rho": float(np.max(np.abs(g["rho"] - dn["rho"]) / np.abs(dn["rho"]))),
            "a": float(max(np.max(np.abs(g[ax] - acc[ax]) / (acc["scale_a"][i] + 1e-300))
                           for i, ax in enumerate(("ax", "ay", "az")))),
            "du": float(np.max(np.abs(g["du"] - acc["du"]) / (acc["scale_du"] + 1e-300))),
            "dt": abs(dt - r["dt"]) / r["dt"],
            "x": float(np.max(np.abs(g["x"] - r["state"]["x"][ref]))),
        }
        diag = sim.diagnostics()
        rows.append({"step": a.s0 + k + 1, "dt": dt, "E": diag["energy"], "p": list(diag["momentum"]),
                     "max_rel_err": err, "parity_ok": err["rho"] <= 1e-10 and err["a"] <= 1e-10 and
                     err["du"] <= 1e-10 and err["dt"] <= 1e-12})
        print(json.dumps(rows[-1]), flush=True)
        dt_prev = dt
    json.dump({"n": a.n, "s0": a.s0, "k": a.k, "symmetric": a.symmetric, "steps": rows,
               "all_parity_ok": all(r_["parity_ok"] for r_ in rows)}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
