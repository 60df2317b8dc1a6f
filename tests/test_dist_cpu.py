"""Multi-rank host logic on CPU (gloo, world_size 2): query sharding with a
replicated tree + all-reduce of flushed point gradients equals the
single-process adjoint. The per-rank compute is the CPU oracle standing in
for each GPU (no GPU here); the sharding / reduction code is the product's
(paper_2405_16788_b200.parallel), the same calls bench.py makes under NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_16788_b200.parallel import allreduce_point_gradients, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    rng = np.random.default_rng(5)
    n, C, q = 800, 4, 240
    pos = rng.uniform(-1, 1, (n, 3))
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    area = rng.uniform(0.5, 1, n) / n
    mu = rng.standard_normal((n, C))
    xs = rng.uniform(-1.5, 1.5, (q, 3))
    d_out = rng.standard_normal((q, C))
    return pos, nrm, area, mu, xs, d_out


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, nrm, area, mu, xs, d_out = _case()
    tree = O.OracleTree(O.Cloud(pos, nrm, area, mu))  # replicated tree
    kinds = np.array([0, 1, 1, 1], np.uint8)
    tree.set_kinds(kinds)
    lo, hi = shard_range(xs.shape[0], rank, world)
    m, n, de = tree.adjoint(O.Params(0.08), 2.0, xs[lo:hi], d_out[lo:hi], threads=1)
    mt, nt = torch.from_numpy(m), torch.from_numpy(n)
    de = allreduce_point_gradients(mt, nt, de)
    if rank == 0:
        np.savez(os.path.join(out_dir, "dist.npz"), m=mt.numpy(), n=nt.numpy(), de=de)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_covers():
    for total in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            cuts = [shard_range(total, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == total
            assert all(cuts[i][1] == cuts[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in cuts) - min(h - l for l, h in cuts) <= 1


def test_two_rank_adjoint_allreduce_matches_single(tmp_path, oracle_mod):
    O = oracle_mod
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "dist.npz")
    pos, nrm, area, mu, xs, d_out = _case()
    t = O.OracleTree(O.Cloud(pos, nrm, area, mu))
    t.set_kinds(np.array([0, 1, 1, 1], np.uint8))
    m, n, de = t.adjoint(O.Params(0.08), 2.0, xs, d_out, threads=1)
    s = np.abs(m).max()
    assert np.abs(got["m"] - m).max() <= 1e-12 * s
    assert np.abs(got["n"] - n).max() <= 1e-12 * np.abs(n).max()
    assert abs(float(got["de"]) - de) <= 1e-12 * abs(de)
