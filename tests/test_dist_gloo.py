"""N>1 host logic on CPU (-m "not gpu"): two real processes over gloo.

Checks the pieces of the multi-GPU path that run on the host: the NCCL unique-id
bootstrap through torch.distributed, and the SFC decomposition helpers of the C
ABI (sph_decomp_splitters / sph_decomp_owner) fed with an all-reduced key-prefix
histogram exactly as sph_dist.cu does -- every rank must derive the same
splitters, the ranks' key ranges must partition the particles, and the split
must be balanced to within one histogram bin (PAPER.md P:196-197 bucket bound).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _spread(v):
    v = v.astype(np.uint64) & np.uint64(0x1FFFFF)
    for s, m in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                 (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        v = (v | (v << np.uint64(s))) & np.uint64(m)
    return v


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, ROOT)
    from paper_2005_02656_b200 import dist as D
    from paper_2005_02656_b200 import inputs, sph
    dist.init_process_group("gloo", init_method="env://")
    try:
        uid = D.share_unique_id(rank, world, device="cpu")
        allid = [None] * world
        dist.all_gather_object(allid, uid)
        d = inputs.random_cloud(20000, box=10.0, seed=123)
        mine = np.arange(rank, 20000, world)  # scrambled initial ownership
        nc, cbits = 16, 4
        c = [np.clip((d[k][mine] / 10.0 * nc).astype(np.int64), 0, nc - 1) for k in "xyz"]
        morton = _spread(c[0]) | (_spread(c[1]) << np.uint64(1)) | (_spread(c[2]) << np.uint64(2))
        shift = 3 * cbits - 9  # 512 bins
        bins = (morton >> np.uint64(shift)).astype(np.int64)
        hist = torch.from_numpy(np.bincount(bins, minlength=512).astype(np.int64))
        dist.all_reduce(hist)  # the allreduce sph_dist.cu does with NCCL
        split = sph.decomp_splitters(hist.numpy(), world)
        allsplit = [None] * world
        dist.all_gather_object(allsplit, split.tolist())
        owners = np.array([sph.decomp_owner(split, b) for b in bins])
        counts = torch.from_numpy(np.bincount(owners, minlength=world).astype(np.int64))
        dist.all_reduce(counts)
        out[rank] = {"uid_same": all(u == allid[0] for u in allid) and len(allid[0]) == 128,
                     "split_same": all(s == allsplit[0] for s in allsplit),
                     "counts": counts.tolist(), "maxbin": int(hist.max()), "split": split.tolist()}
    finally:
        dist.destroy_process_group()


def test_two_rank_bootstrap_and_splitters():
    from paper_2005_02656_b200 import _build
    _build.build()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        assert res[r]["uid_same"] and res[r]["split_same"]
    counts = res[0]["counts"]
    assert sum(counts) == 20000
    assert max(counts) - min(counts) <= 2 * res[0]["maxbin"]
    assert res[0]["split"][0] == 0 and res[0]["split"][-1] == 512


def test_splitter_edge_cases():
    from paper_2005_02656_b200 import sph
    # empty histogram, single rank, more ranks than particles
    sp = sph.decomp_splitters(np.zeros(8), 3)
    assert sp[0] == 0 and sp[-1] == 8 and np.all(np.diff(sp) >= 0)
    assert sph.decomp_splitters(np.ones(8), 1).tolist() == [0, 8]
    sp = sph.decomp_splitters(np.array([0, 0, 5, 0]), 4)
    assert sp[0] == 0 and sp[-1] == 4 and np.all(np.diff(sp) >= 0)
    h = np.random.default_rng(0).integers(0, 50, 4096)
    for G in (2, 3, 8):
        sp = sph.decomp_splitters(h, G)
        per = [h[sp[r]:sp[r + 1]].sum() for r in range(G)]
        assert sum(per) == h.sum() and max(per) - min(per) <= 2 * h.max()
        for b in (0, 100, 4095):
            r = sph.decomp_owner(sp, b)
            assert sp[r] <= b < sp[r + 1]
