"""Copy the round's measured evidence from gpurun_out/ into profiles/ (tracked).

bench JSON lines -> profiles/r1_bench_*.json; ncu launch list -> r1_launches_weak_25M.csv;
ncu --set full capture -> r1_ncu_traffic.json (tools/ncu_traffic.py) + per-kernel stall
summaries (tools/ncu_src_stalls.py).  usage: python tools/collect_evidence.py"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def jline(log):
    for line in reversed(open(os.path.join(G, log)).read().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    return None


def dump(obj, name):
    with open(os.path.join(P, name), "w") as f:
        json.dump(obj, f)
        f.write("\n")


benches = {"ev_bench_w1.log": "r1_bench_weak_w1.json", "ev_bench_ref.log": "r1_bench_reference.json",
           "ev_bench_1m.log": "r1_bench_patch1m.json", "ev_bench_evrard.log": "r1_bench_evrard.json",
           "ev_bench_27m.log": "r1_bench_patch27m_strong1.json"}
for log, out in benches.items():
    if os.path.exists(os.path.join(G, log)):
        d = jline(log)
        if d:
            dump(d, out)
            print(out, d.get("ms_per_step"), d.get("value"))
for n in (2, 4):
    for pre, out in (("scale_w", f"r1_bench_weak_w{n}.json"), ("strong", f"r1_bench_patch27m_strong{n}.json")):
        log = f"{pre}{n}.log"
        if os.path.exists(os.path.join(G, log)) and jline(log):
            dump(jline(log), out)
            print(out, jline(log)["ms_per_step"])
if os.path.exists(os.path.join(G, "scale_w4_lazy.log")) and jline("scale_w4_lazy.log"):
    dump(jline("scale_w4_lazy.log"), "r1_bench_weak_w4_lazy10.json")
if os.path.exists(os.path.join(G, "ev_launches.csv")):
    shutil.copy(os.path.join(G, "ev_launches.csv"), os.path.join(P, "r1_launches_weak_25M.csv"))
rep = os.path.join(G, "ev_full.ncu-rep")
if os.path.exists(rep):
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_traffic.py"), rep,
                    os.path.join(P, "r1_ncu_traffic.json"),
                    "ncu --set full --clock-control none --import-source on -k regex:'k_momentum_c|k_density_c|"
                    "k_iad_c|k_search' -s 12 -c 4, bench.py --steps 1 --warmup 3 --no-cpu-baseline (config 5: "
                    "weak square patch 292^3 = 24,897,088 particles, 1 B200), one launch per kernel"], check=True,
                   stdout=subprocess.DEVNULL)
    with open(os.path.join(P, "r1_ncu_stalls.txt"), "w") as f:
        for k in ("k_momentum_c", "k_search", "k_density_c", "k_iad_c"):
            csvp = os.path.join(G, f"ev_{k}.csv")
            with open(csvp, "w") as c:
                subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{k}",
                                "--print-source", "sass"], stdout=c, check=True)
            out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_src_stalls.py"), csvp, "25"],
                                 capture_output=True, text=True).stdout
            f.write(f"== {k} (source-level warp-stall sampling, SASS)\n{out}\n")
    print("ncu summaries written")
