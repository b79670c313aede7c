"""bench.py -- fp64 particle-updates/s of the B200 SPH-EXA timestep (arXiv 2005.02656).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload weak|patch1m|patch27m|evrard]
                    [--impl ours|reference]

One "step" is one full pass of the hot path (bbox, Morton
sort, permutation, cells, neighbour lists, density+Omega+EOS, IAD,
momentum+energy+AV, min-dt, update, h) over all particles.  Inputs are seeded
synthetic particle sets resident in HBM before the timed region; every field
array (>=200 MB at the default workload) exceeds the 126 MB L2, so no flush is
needed.  Timing: CUDA events on the library's stream, W untimed warm-up steps,
barrier + synchronize on both sides, max over ranks.

--impl reference times the CPU oracle (oracle/, plain C + OpenMP) on the host
cores on a bounded sample of the same workload (the only other place bench.py
runs oracle/).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 particle-updates/sec per timestep at 1/2/4/8 B200; % of HBM/FP64 roofline"
UNIT = "particle-updates/s"

# Algorithmic FP64 flops per neighbour pair (FMA = 2), counted from the pair
# bodies as written: density+Omega, IAD, momentum+energy+AV;
# per candidate for the search (3 sub + r^2 + compare).
FLOPS_PER_PAIR = {"density": 70, "iad": 52, "momentum": 169}
FLOPS_PER_CANDIDATE = 9
# Whole-step roofline model: per phase max(bytes / HBM,
# flops / FP64 peak) with algorithmic bytes / flops; the search at the survey's 6.4
# candidates per neighbour x 8 flops.  Bytes per particle of the streaming phases from
# the survey table (bbox+keys 36, sort 200, permute 240, cells 10, update+h 204); the
# pair passes read 2-byte row entries per pair plus their staged fields per particle.
MODEL_STREAM_BYTES = {"bbox_keys": 36, "sort": 200, "permute": 240, "cells": 10, "update": 204}
MODEL_PAIR_BYTES = {"search": 2.0, "density": 2.0, "iad": 2.0, "momentum": 2.0}
MODEL_PARTICLE_BYTES = {"search": 32 + 8, "density": 32 + 80, "iad": 32 + 56, "momentum": 136 + 40}
SEARCH_FLOPS_PER_PAIR = 6.4 * 8


def workload(name: str, G: int, rank: int):
    from paper_2005_02656_b200 import inputs as I
    if name == "weak":  # 300 x 300 x (300 G), slab per rank: config 4 (27M) at N=1, config 5 weak scaling
        d = I.square_patch_weak(300, G, rank if G > 1 else None)
        desc = (f"square patch 300x300x{300 * G}, {300 ** 3} particles/GPU (N=1: config 4, the "
                f"north_star's 27M patch; N>1: config 5 weak scaling, z-stacked per GPU)")
    elif name == "weak292":  # config 5 as in BASELINE: 292 x 292 x (292 G)
        d = I.square_patch_weak(292, G, rank if G > 1 else None)
        desc = f"config5 weak-scaling square patch 292x292x{292 * G}, {292 ** 3} particles/GPU"
    elif name == "patch27m":  # config 4 (strong scaling): z-slab of the 300^3 patch per rank
        zl = (rank * 300 // G, (rank + 1) * 300 // G) if G > 1 else None
        d = I.square_patch(300, z_layers=zl)
        desc = f"config4 square patch 300^3 = 27M particles over {G} GPU(s)"
    elif name == "patch1m":  # config 2
        d = I.square_patch(100)
        desc = "config2 square patch 100^3 = 1M particles"
    elif name == "evrard":  # config 3
        d = I.evrard(124)
        desc = "config3 Evrard-shaped sphere, 998,592 particles, variable h"
    else:
        raise SystemExit(f"unknown workload {name}")
    return d, desc


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [q.strip() for q in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_baseline(target_seconds: float = 12.0) -> dict:
    """The oracle as it stands, one full step, on a bounded square-patch sample."""
    import oracle as O
    from paper_2005_02656_b200 import inputs as I
    O.build()
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    d = I.square_patch(20)
    o = O.Oracle(O.Params.from_inputs(d))
    t = time.perf_counter()
    o.step(d)
    rate = d["x"].size / (time.perf_counter() - t)
    n = int(round((rate * target_seconds) ** (1.0 / 3.0)))
    n = max(20, min(n, 120))
    d = I.square_patch(n)
    o = O.Oracle(O.Params.from_inputs(d))
    t = time.perf_counter()
    o.step(d)
    el = time.perf_counter() - t
    return {"value": d["x"].size / el, "unit": UNIT, "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"square patch {n}^3 = {d['x'].size} particles, 1 full step "
                      f"(grid neighbours, density, IAD, momentum, dt, update), {el:.1f} s",
            "seconds": el}


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    from paper_2005_02656_b200 import inputs as I
    O.build()
    cores = len(os.sched_getaffinity(0))
    # bounded sample per step, sized so W + K steps stay within a few minutes
    probe = cpu_baseline(target_seconds=2.0)
    per_step_s = 120.0 / max(1, args.steps + args.warmup)
    n = int(round((probe["value"] * per_step_s) ** (1.0 / 3.0)))
    n = max(20, min(n, 120))
    d = I.square_patch(n)
    o = O.Oracle(O.Params.from_inputs(d))
    st = d
    for _ in range(args.warmup):
        st = dict(d, **o.step(st)["state"])
    t = time.perf_counter()
    for _ in range(args.steps):
        st = dict(d, **o.step(st)["state"])
    el = time.perf_counter() - t
    v = d["x"].size * args.steps / el
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_label(args)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"square patch {n}^3 = {d['x'].size} particles per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_label(args):
    return {"weak": "square_patch_300^3_per_gpu (config4 at N=1, config5 weak)",
            "weak292": "config5_weak_square_patch_292^3_per_gpu", "patch27m": "config4_square_patch_300^3",
            "patch1m": "config2_square_patch_100^3", "evrard": "config3_evrard_124"}[args.workload]


def run_ours(args):
    import numpy as np
    import torch

    from paper_2005_02656_b200 import dist as D
    from paper_2005_02656_b200 import sph
    world, rank, local = D.init("nccl")
    uid = D.share_unique_id(rank, world)
    d, desc = workload(args.workload, max(world, 1), rank)
    n_local = d["x"].size
    # room for halos + migrants (multi-GPU); a single GPU needs exactly n
    cap = n_local if world == 1 else int(n_local * 1.6) + 4096
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        sim = sph.Simulation(d, capacity=cap, stream=stream.cuda_stream, rank=rank, nranks=world,
                             unique_id=uid, kernel_mode=sph.KERNEL_MODES[args.kernel_mode],
                             symmetric=int(args.symmetric), redecomp_every=args.redecomp_every,
                             cell_factor=args.cell_factor)
        for _ in range(args.warmup):
            sim.step()
        torch.cuda.synchronize()
        sim.set_profiling(True)
        sim.phase_times(reset=True)
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(stream)
            for _ in range(args.steps):
                sim.step()
            e1.record(stream)
            torch.cuda.synchronize()
        barrier(world)
        ms = e0.elapsed_time(e1)
        phase_ms, phase_launch = sim.phase_times(reset=True)
        sim.set_profiling(False)
        diag = sim.diagnostics()
        # end-to-end through the public API with host buffers: H2D state, step, D2H state
        host = sph.HostParticles(sim.state())
        nbytes = host.nbytes()
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ee0.record(stream)
        e2e_steps = max(1, min(args.steps, 3))
        for _ in range(e2e_steps):
            sim.upload(host)
            sim.step()
            sim.download(host)
        ee1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = max(ee0.elapsed_time(ee1), 1e3 * (time.perf_counter() - t0))
        peak64 = sph.measure_fp64_peak(stream.cuda_stream)
    ms_rank = ms
    mem_per_particle = (torch.cuda.max_memory_allocated() + sim.library_bytes()) / max(1, n_local)
    ms = max_over_ranks(ms, world)
    e2e_ms = max_over_ranks(e2e_ms, world)
    per_rank = None
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([n_local], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        n_total = int(t.item())
        # per-rank view of the step (load balance, halo sizes): rank 0 reports it
        sim._sync_n()
        mine = {"ms_per_step": round(ms_rank / args.steps, 3), "n_owned": int(sim.n),
                "n_halo": int(getattr(sim, "n_halo", 0)),
                "phases": {k: round(v / args.steps, 3) for k, v in phase_ms.items() if v}}
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    else:
        n_total = n_local
    if rank != 0:
        return
    ms_step = ms / args.steps
    value = n_total * args.steps / (ms * 1e-3)
    pairs = diag["nbr_total"] / max(world, 1)  # diagnostics sum over ranks; per-rank average
    mom_ms = phase_ms["momentum"] / args.steps
    mom_flops = FLOPS_PER_PAIR["momentum"] * pairs
    achieved = mom_flops / (mom_ms * 1e-3) / 1e12
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    phases = {k: round(v / args.steps, 4) for k, v in phase_ms.items() if v}
    # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    # (profiles/r2_ncu_traffic.json; only for the workload and GPU count it was captured on)
    traffic, traffic_src = None, "profiles/r2_ncu_traffic.json (dram__bytes_read+write, 1 launch)"
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "r2_ncu_traffic.json")))
        if (args.workload == tr.get("workload") and world == 1 and not args.symmetric
                and args.kernel_mode == "poly"):
            k = tr["kernels"]["k_momentum_c"]
            traffic = k["dram_read_bytes"] + k["dram_write_bytes"]
    except Exception:
        pass
    # every FP64-bound pair pass against the same measured peak (algorithmic flops / event time)
    pair_kernels = {}
    for ph_name in ("density", "iad", "momentum"):
        t = phase_ms.get(ph_name, 0.0) / args.steps
        if t > 0:
            a = FLOPS_PER_PAIR[ph_name] * pairs / (t * 1e-3) / 1e12
            pair_kernels[ph_name] = {"ms": round(t, 3), "tflops": round(a, 3),
                                     "frac": round(a / peak64, 4) if peak64 else None}
    # whole-step roofline model (SURVEY §8(d) "headline fraction = sum roofline time / measured")
    bw = (peaks.get("hbm_gbs") or 6549.1) * 1e9
    p64 = peak64 * 1e12
    model = {
        "bbox+keys": MODEL_STREAM_BYTES["bbox_keys"] * n_local / bw,
        "sort": MODEL_STREAM_BYTES["sort"] * n_local / bw,
        "permute": MODEL_STREAM_BYTES["permute"] * n_local / bw,
        "cells": MODEL_STREAM_BYTES["cells"] * n_local / bw,
        "update": MODEL_STREAM_BYTES["update"] * n_local / bw,
    }
    for ph_name in ("search", "density", "iad", "momentum"):
        fl = (SEARCH_FLOPS_PER_PAIR if ph_name == "search" else FLOPS_PER_PAIR[ph_name]) * pairs
        by = MODEL_PAIR_BYTES[ph_name] * pairs + MODEL_PARTICLE_BYTES[ph_name] * n_local
        model[ph_name] = max(fl / p64, by / bw)
    model_ms = {k: round(v * 1e3, 3) for k, v in model.items()}
    step_model_ms = sum(model.values()) * 1e3
    search_ms = phase_ms.get("neighbors", 0.0) / args.steps
    roofline_step = {"model_ms_per_step": round(step_model_ms, 3), "measured_ms_per_step": ms_step,
                     "frac": step_model_ms / ms_step, "model_phases_ms": model_ms,
                     "search_frac": (model["search"] * 1e3 / search_ms) if search_ms else None,
                     "peaks": {"fp64_tflops": peak64, "hbm_gbs": bw / 1e9},
                     "note": "per phase max(algorithmic bytes / HBM, algorithmic flops / FP64 peak); "
                             "search at 6.4 candidates x 8 flops per neighbour (SURVEY 8(d))"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": max(world, 1),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong" if args.workload == "patch27m" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_label(args), "description": desc,
                   "particles_per_gpu": n_local, "particles_total": n_total,
                   "kernel_mode": args.kernel_mode, "symmetric": bool(args.symmetric),
                   "cell_factor": args.cell_factor or 1.0,
                   "redecomp_every": args.redecomp_every,
                   "neighbors_mean": diag["nbr_total"] / max(1, diag["n_owned"]),
                   "l2": "no flush: every SoA field array >= 200 MB > 126 MB L2",
                   "parallelism": f"sfc{max(world, 1)}" if world > 1 else "1 GPU"},
        "roofline": {"kernel": "k_momentum", "bound": "alu", "achieved": achieved,
                     "peak": peak64, "unit": "TFLOP/s",
                     "peak_source": "measured live: DFMA kernel (sph_measure_fp64_peak)",
                     "frac": achieved / peak64 if peak64 else None, "traffic": traffic,
                     "traffic_source": traffic_src if traffic is not None else None,
                     "algorithmic_bytes": 4.0 * pairs + 136.0 * n_local,
                     "flops_per_pair": FLOPS_PER_PAIR["momentum"], "pairs_per_launch": pairs,
                     "avg_launch_ms": mom_ms},
        "pair_kernels_fp64": pair_kernels,
        "roofline_step": roofline_step,
        "memory_bytes_per_particle": mem_per_particle,
        "phases_ms_per_step": phases,
        "per_rank": per_rank,
        "gpu_launches": int(sum(phase_launch.values())),
        "e2e": {"value": n_total * e2e_steps / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                "steps": e2e_steps},
        "clocks": clk.summary(),
        "hbm_peak_gbs": peaks.get("hbm_gbs"),
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="weak", choices=["weak", "weak292", "patch27m", "patch1m", "evrard"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel-mode", default="poly", choices=["poly", "table", "sin"],
                    help="kernel evaluation in the pair passes (sph.h SPH_KERNEL_*; A/B of P:248)")
    ap.add_argument("--redecomp-every", type=int, default=1,
                    help="multi-GPU: recompute splitters every k-th step (sph_params.redecomp_every)")
    ap.add_argument("--cell-factor", type=float, default=0.0,
                    help="search-cell edge in units of 2 mean(h) (sph_params.cell_factor; 0: 1.0)")
    ap.add_argument("--symmetric", action="store_true",
                    help="neighbour relation r < 2 max(h_a, h_b) (sph_params.symmetric)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
