"""Multi-GPU parity driver (run under torchrun with >= 2 GPUs; see tests/test_multigpu.py).

Every rank attaches a deliberately scrambled subset of a square patch (ids
round-robin over ranks, so the first step migrates almost every particle), then
runs STEPS timesteps through SFC decomposition, halo exchanges and the dt
allreduce.  Rank 0 gathers the state by id and compares it with a 1-GPU run of
the same input: every field must be bit-identical (per-target stencil slots and
within-cell order do not depend on the rank count), dt identical each step.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2005_02656_b200 import dist, inputs, sph  # noqa: E402

STEPS = int(os.environ.get("MGPU_STEPS", "4"))
CASE = os.environ.get("MGPU_CASE", "patch")
FIELDS = ("x", "y", "z", "vx", "vy", "vz", "h", "u", "rho", "omega", "p", "ax", "ay", "az", "du",
          "vsig", "c11", "c23")


def make_input():
    if CASE == "patch":
        return inputs.square_patch(24, 24, pressure_ics=True)
    if CASE == "weak":
        return inputs.square_patch_weak(20, int(os.environ["WORLD_SIZE"]))
    if CASE == "evrard":  # variable h (8x), open box, ideal gas
        return inputs.evrard(30)
    if CASE == "cloud_sym":  # variable h, periodic x and z, symmetric neighbour relation
        return inputs.random_cloud(6000, box=12.0, h0=0.8, hspread=0.3, periodic=(1, 0, 1), seed=3)
    return inputs.jitter(inputs.square_patch(20, 16))


KW = {"symmetric": 1} if CASE == "cloud_sym" else {}
# lazy re-decomposition (splitters kept for k steps): the 1-GPU
# reference ignores it, so bit-identity also checks that kept splitters stay correct
KW_MG = dict(KW, redecomp_every=int(os.environ.get("MGPU_REDECOMP", "1")))


def main():
    import torch
    world, rank, local = dist.init("nccl")
    uid = dist.share_unique_id(rank, world)
    d = make_input()
    mine = inputs.subset(d, np.arange(rank, d["x"].size, world))
    cap = int(d["x"].size * 1.2) + 1024  # any rank may end up owning a big share + halos
    sim = sph.Simulation(mine, capacity=cap, rank=rank, nranks=world, unique_id=uid, **KW_MG)
    dts = []
    for _ in range(STEPS):
        dts.append(sim.step(want_dt=True))
    diag = sim.diagnostics()
    got = dist.gather_by_id(sim.state(), world, FIELDS)
    ok, msg = True, ""
    if rank == 0:
        ref = sph.Simulation(d, capacity=cap, **KW)
        rdts = [ref.step(want_dt=True) for _ in range(STEPS)]
        rst = ref.state()
        o = np.argsort(rst["id"])
        rst = {k: v[o] for k, v in rst.items()}
        rdiag = ref.diagnostics()
        if not np.array_equal(got["id"], rst["id"]):
            ok, msg = False, "particle ids differ"
        if ok and dts != rdts:
            ok, msg = False, f"dt differs {dts} {rdts}"
        for k in FIELDS:
            if ok and not np.array_equal(got[k], rst[k]):
                bad = np.flatnonzero(got[k] != rst[k])
                ok, msg = False, f"{k}: {bad.size} particles differ, e.g. id {got['id'][bad[0]]}: {got[k][bad[0]]!r} vs {rst[k][bad[0]]!r}"
        if ok and diag["nbr_total"] != rdiag["nbr_total"]:
            ok, msg = False, f"pair count {diag['nbr_total']} vs {rdiag['nbr_total']}"
        print(json.dumps({"world": world, "case": CASE, "steps": STEPS, "ok": ok, "msg": msg,
                          "n": int(d["x"].size), "halo_rank0": int(sim.n_halo),
                          "pairs": int(diag["nbr_total"])}), flush=True)
    dist.barrier(world)
    torch.cuda.synchronize()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
