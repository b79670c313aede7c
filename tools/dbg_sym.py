"""Debug aid: the symmetric-relation square patch stepped until it fails."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2005_02656_b200 import inputs as I, sph
d = I.square_patch(30, pressure_ics=True)
sim = sph.Simulation(d, symmetric=1)
for step in range(300):
    try:
        sim.step(want_dt=True)
    except Exception as e:
        g = sim.diagnostics(check=False)
        print("step", step, "FAILED", e, "nbr_max", g.get("nbr_max"), flush=True)
        raise SystemExit(1)
    if step % 20 == 0:
        g = sim.diagnostics()
        print(step, "nbr_max", g["nbr_max"], "mean", g["nbr_total"] / g["n_owned"], flush=True)
print("DONE")
