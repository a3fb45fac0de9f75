"""CPU, world_size 2 over gloo: the document-sharded sweep decomposition is exact.

The multi-GPU LDA sweep (csrc/lda.cu) runs per rank: local
topic-word counts -> reduce-scatter by vocabulary slices of ceil(V / W) columns -> the
rank draws the phi cells of ITS slice only (counter RNG keyed by (k, v, iter)) ->
all-gather of the drawn cells -> the Dirichlet row normalisation over the gathered cells
(identical on every rank) -> theta + z blocks on the rank's own documents (keys use
GLOBAL document / token indices) -> all-reduce of the log-joint pieces.  Here the same
decomposition runs on the oracle restatement with torch.distributed/gloo as the
collective (reduce-scatter = all-reduce + own slice) and the C-ABI's own partition
(bnmc_gpu_partition); the gathered state must equal the unsharded reference sweep bit
for bit.  The CUDA path itself runs W ranks on one GPU in tests/test_gpu_shard.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, golden


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, sweeps, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1312_3613_b200 as g
    from oracle import Restatement

    R = Restatement()
    fx = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
    K, V, seed = int(fx["K"]), int(fx["V"]), int(fx["seed"])
    off, w = fx["offsets"], fx["w"]
    b, e = g.partition(off, world, rank)
    z, theta = fx["z0"].copy(), fx["theta0"].copy()
    ljs = []
    for it in range(sweeps):
        nkw = R.lda_count_phi(K, V, off, w, z, b, e)              # local counts
        t = torch.from_numpy(nkw)
        dist.all_reduce(t)                                        # reduce-scatter: this rank
        sl = -(-V // world)                                       # uses its slice's columns
        v0, v1 = min(V, rank * sl), min(V, rank * sl + sl)
        gam = R.lda_phi_gammas(K, V, off, w, t.numpy(), seed, it, v0, v1)
        parts = [None] * world                                    # all-gather of the slices
        dist.all_gather_object(parts, (v0, v1, gam.reshape(K, V)[:, v0:v1].copy()))
        g = np.zeros((K, V))
        for p0, p1, pg in parts:
            g[:, p0:p1] = pg
        S = np.cumsum(g, axis=1)[:, -1:]                          # left-to-right row sums and
        phi = (g / S).ravel()                                     # normalisation (batch.cpp:55-61)
        R.lda_theta_z(K, V, off, w, z, phi, theta, seed, it, b, e)
        # local pieces of the log-joint, summed over ranks
        zt = sum(np.log(theta[d * K + z[off[d]:off[d + 1]]]).sum() for d in range(b, e))
        wt = sum(np.log(phi[z[off[d]:off[d + 1]] * V + w[off[d]:off[d + 1]]]).sum() for d in range(b, e))
        pieces = torch.tensor([zt, wt], dtype=torch.float64)
        dist.all_reduce(pieces)
        # exchange the shards' z / theta so every rank holds the global state
        parts = [None] * world
        dist.all_gather_object(parts, (b, e, z[off[b]:off[e]].copy(), theta[b * K:e * K].copy()))
        for pb, pe, pz, pt in parts:
            z[off[pb]:off[pe]] = pz
            theta[pb * K:pe * K] = pt
        ljs.append(pieces.numpy().copy())
    if rank == 0:
        np.savez(os.path.join(out_dir, "sharded.npz"), z=z, theta=theta, phi=phi, pieces=np.array(ljs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["lda_desk", "lda_ragged"])
def test_document_sharded_sweep_equals_unsharded(tmp_path, name):
    fx = golden(name)
    sweeps = len(fx["lj"])
    mp.spawn(_worker, args=(2, _free_port(), name, sweeps, str(tmp_path)), nprocs=2, join=True)
    r = np.load(tmp_path / "sharded.npz")
    assert np.array_equal(r["z"], fx["z"][-1])          # integer state bit-exact
    assert np.array_equal(r["phi"], fx["phi"][-1])      # identical phi draw on every rank
    assert np.array_equal(r["theta"], fx["theta"][-1])
    K, V = int(fx["K"]), int(fx["V"])
    z, w, off = fx["z"][-1], fx["w"], fx["offsets"]
    docs = np.repeat(np.arange(len(off) - 1), np.diff(off))
    zt = np.log(fx["theta"][-1][docs * K + z]).sum()
    wt = np.log(fx["phi"][-1][z * V + w]).sum()
    assert abs(r["pieces"][-1][0] - zt) <= 1e-10 * abs(zt)
    assert abs(r["pieces"][-1][1] - wt) <= 1e-10 * abs(wt)
