"""Build libsph.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsph.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills",
]


def _nccl_paths():
    try:
        import nvidia.nccl as nn  # torch-bundled NCCL (the one torch.distributed uses)
        base = os.path.dirname(nn.__file__) if nn.__file__ else list(nn.__path__)[0]
    except Exception:  # pragma: no cover
        return None, None
    inc = os.path.join(base, "include")
    lib = os.path.join(base, "lib")
    return (inc if os.path.exists(os.path.join(inc, "nccl.h")) else None,
            lib if glob.glob(os.path.join(lib, "libnccl.so*")) else None)


def sources(csrc: str = CSRC):
    return sorted(glob.glob(os.path.join(csrc, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "sph.h")]


def build(force: bool = False, verbose: bool = False, csrc: str = CSRC, out: str = LIB) -> str:
    """SPH_NVCC_EXTRA (env) adds flags, e.g. -D macros of A/B variant builds (tools/)."""
    newest = max(os.path.getmtime(p) for p in deps())
    if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    cmd = ["nvcc", *NVCC_FLAGS, *os.environ.get("SPH_NVCC_EXTRA", "").split()]
    inc, lib = _nccl_paths()
    if inc and lib:
        cmd += ["-DSPH_WITH_NCCL=1", f"-I{inc}", f"-L{lib}", "-l:libnccl.so.2",
                f"-Xlinker", f"-rpath={lib}"]
    tmp = out + f".tmp{os.getpid()}"
    cmd += [f"-I{csrc}", "-o", tmp, *sources(csrc)]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--csrc", default=CSRC, help="kernel source dir (variant builds)")
    ap.add_argument("--out", default=LIB)
    a = ap.parse_args()
    print(build(force=True, verbose=True, csrc=os.path.abspath(a.csrc), out=os.path.abspath(a.out)))
