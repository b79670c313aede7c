"""Physics validation: rotating square patch, 100x100x100 =
10^6 particles (§4.6), integrated with the CUDA path to
t = 0.5 s, reporting |L_z| against the paper's L_tot = 8.33e9 g cm^2/s (P:285,
"~0.2% from the parent codes") and the drift of linear momentum and energy.

    python tools/validate_square_patch.py [--n 100] [--t-end 0.5] [--out profiles/r1_validation.json]

Pressure-consistent initial masses (reading R16) are used, as the paper derives P0
from the incompressible Poisson equation.  This is a physics check of
the built path, not part of the timed benchmark.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2005_02656_b200 import inputs, sph
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--t-end", type=float, default=0.5)
    ap.add_argument("--pressure-ics", type=int, default=1)
    ap.add_argument("--max-steps", type=int, default=20000)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "validation.json"))
    a = ap.parse_args()
    torch.cuda.set_device(0)
    d = inputs.square_patch(a.n, pressure_ics=bool(a.pressure_ics))
    sim = sph.Simulation(d)
    d0 = sim.diagnostics()
    hist = []
    t, steps = 0.0, 0
    t0 = time.time()
    while t < a.t_end and steps < a.max_steps:
        dt = sim.step(want_dt=True)
        t += dt
        steps += 1
        if steps % 250 == 0 or t >= a.t_end:
            g = sim.diagnostics()
            s = sim.state()
            ke = 0.5 * float((s["m"] * (s["vx"] ** 2 + s["vy"] ** 2 + s["vz"] ** 2)).sum())
            hist.append({"step": steps, "t": t, "Lz": g["ang_momentum"][2], "E": g["energy"],
                         "KE": ke, "IE": g["energy"] - ke, "rho_min": float(s["rho"].min()),
                         "rho_max": float(s["rho"].max()), "p": g["momentum"], "dt": dt})
            print(json.dumps(hist[-1]), flush=True)
    g = sim.diagnostics()
    Lz0, Lz = d0["ang_momentum"][2], g["ang_momentum"][2]
    m_scale = sum(abs(v) for v in d["m"] * (abs(d["vx"]) + abs(d["vy"])))
    res = {
        "config": f"square patch {a.n}^3, pressure-consistent ICs={bool(a.pressure_ics)}",
        "steps": steps, "t": t, "wall_s": time.time() - t0,
        "Lz_t0": Lz0, "Lz_end": Lz, "abs_Lz_end": abs(Lz),
        "paper_Ltot_t0.5": 8.33e9, "rel_to_paper": abs(Lz) / 8.33e9 - 1.0,
        "Lz_drift_rel": (Lz - Lz0) / abs(Lz0),
        "momentum_end": g["momentum"], "momentum_rel_to_sum_m_abs_v": [p / m_scale for p in g["momentum"]],
        "E_t0": d0["energy"], "E_end": g["energy"], "E_drift_rel": (g["energy"] - d0["energy"]) / d0["energy"],
        "counters": {k: g[k] for k in ("omega_clamped", "iad_singular", "coincident_pairs", "u_floored",
                                        "h_clamped")},
        "history": hist,
    }
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "history"}), flush=True)


if __name__ == "__main__":
    main()
