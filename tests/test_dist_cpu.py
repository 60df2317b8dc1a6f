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


# ---------------------------------------------------------------- sharded point update
class _OracleEngine:
    """sharded_point_update's device side restated on the oracle's Adam (CPU):
    fp64 parameters / state arrays, normals renormalised when changed."""

    def __init__(self, mu, nrm):
        import sys

        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
        import oracle as O

        self.O = O
        self.mu, self.nrm = mu.copy(), nrm.copy()
        self.m_mu, self.v_mu = np.zeros_like(mu), np.zeros_like(mu)
        self.m_n, self.v_n = np.zeros_like(nrm), np.zeros_like(nrm)
        self.t = 0

    def adam_range(self, g_mom, g_nrm, lo, hi):
        O = self.O
        self.t += 1
        if hi <= lo:
            return
        lib = O.port_lib()
        gm = np.ascontiguousarray(g_mom.numpy(), np.float64)
        gn = np.ascontiguousarray(g_nrm.numpy(), np.float64)
        for p, g, m, v in ((self.mu, gm, self.m_mu, self.v_mu), (self.nrm, gn, self.m_n, self.v_n)):
            ps, ms, vs = (np.ascontiguousarray(a[lo:hi]) for a in (p, m, v))
            lib.ora_adam_step(ps.ctypes.data_as(O._dp), g.ctypes.data_as(O._dp), ms.ctypes.data_as(O._dp),
                              vs.ctypes.data_as(O._dp), ps.size, 1e-2, 0.9, 0.999, 1e-8, self.t)
            if p is self.nrm:
                old = p[lo:hi]
                changed = np.any(ps != old, axis=1)
                lens = np.sqrt((ps[:, 0] ** 2 + ps[:, 1] ** 2) + ps[:, 2] ** 2)
                ok = changed & (lens > 1e-12)
                ps[ok] = ps[ok] / lens[ok, None]
                ps[~ok] = old[~ok]
            p[lo:hi], m[lo:hi], v[lo:hi] = ps, ms, vs

    def get_range(self, lo, hi, nrm_out, mom_out):
        nrm_out.copy_(torch.from_numpy(self.nrm[lo:hi]))
        mom_out.copy_(torch.from_numpy(self.mu[lo:hi]))

    def set_all(self, nrm, mom):
        self.nrm, self.mu = nrm.numpy().copy(), mom.numpy().copy()

    def refresh(self):
        pass


def _sharded_case():
    rng = np.random.default_rng(9)
    n, C = 301, 5  # uneven split: chunks of 151 / 150
    mu = rng.standard_normal((n, C))
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    g = [(rng.standard_normal((n, C)).astype(np.float32), rng.standard_normal((n, 3)).astype(np.float32))
         for _ in range(2)]  # per-rank flushed gradients
    return n, C, mu, nrm, g


def _sharded_worker(rank, world, port, out_dir):
    from paper_2405_16788_b200.parallel import sharded_point_update

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, C, mu, nrm, g = _sharded_case()
    eng = _OracleEngine(mu, nrm)
    for _ in range(2):  # two steps: the Adam state of each slice carries over
        sharded_point_update(eng, torch.from_numpy(g[rank][0]), torch.from_numpy(g[rank][1]), n, C)
    np.savez(os.path.join(out_dir, f"sharded{rank}.npz"), mu=eng.mu, nrm=eng.nrm)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_point_update_matches_single(tmp_path, oracle_mod):
    """Reduce-scatter -> Adam on each rank's slice -> all-gather (gloo, 2 ranks)
    leaves every rank with the parameters of one Adam step on the summed
    gradients."""
    mp.spawn(_sharded_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    n, C, mu, nrm, g = _sharded_case()
    ref = _OracleEngine(mu, nrm)
    gm = torch.from_numpy(g[0][0] + g[1][0])
    gn = torch.from_numpy(g[0][1] + g[1][1])
    for _ in range(2):
        ref.adam_range(gm, gn, 0, n)
    for r in range(2):
        got = np.load(tmp_path / f"sharded{r}.npz")
        assert np.array_equal(got["mu"], ref.mu)
        assert np.array_equal(got["nrm"], ref.nrm)


# ---------------------------------------------------------------- chunked flush all-reduce
class _RowsTree:
    """The flush split of DipoleTree (flush_begin / flush_rows / flush_end) over
    one rank's oracle adjoint result: rows in TREE order (the oracle's
    point_order, identical on every rank), scattered back to the original
    order at the end — the layout parallel.flush_allreduce relies on."""

    def __init__(self, m, n, de, order):
        self.m, self.n, self.de, self.order = m, n, de, order
        self.calls = []

    def point_count(self):
        return self.m.shape[0]

    def channels(self):
        return self.m.shape[1]

    def flush_begin(self, buffers):
        self.calls.append("begin")
        return self.de

    def flush_rows(self, buf, lo, hi, rows):
        self.calls.append(("rows", lo, hi))
        full = np.concatenate([self.m, self.n], 1)[self.order[lo:hi]]
        rows.copy_(torch.from_numpy(full.astype(np.float32)))

    def flush_end(self, buffers, rows, out=None):
        self.calls.append("end")
        C = self.m.shape[1]
        mom = torch.empty((self.m.shape[0], C), dtype=torch.float32)
        nrm = torch.empty((self.m.shape[0], 3), dtype=torch.float32)
        idx = torch.from_numpy(self.order.astype(np.int64))
        mom[idx] = rows[:, :C]
        nrm[idx] = rows[:, C:]
        return mom, nrm


def _flush_worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle as O
    from paper_2405_16788_b200.parallel import flush_allreduce

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pos, nrm, area, mu, xs, d_out = _case()
    tree = O.OracleTree(O.Cloud(pos, nrm, area, mu))
    tree.set_kinds(np.array([0, 1, 1, 1], np.uint8))
    lo, hi = shard_range(xs.shape[0], rank, world)
    m, n, de = tree.adjoint(O.Params(0.08), 2.0, xs[lo:hi], d_out[lo:hi], threads=1)
    rt = _RowsTree(m, n, de, tree.export()["order"])
    rows = torch.empty((m.shape[0], m.shape[1] + 3), dtype=torch.float32)
    mom, nr, de_sum = flush_allreduce(rt, [None], rows=rows, chunks=3)
    if rank == 0:
        np.savez(os.path.join(out_dir, "flush.npz"), m=mom.numpy(), n=nr.numpy(), de=de_sum,
                 calls=np.array([str(c) for c in rt.calls]))
    dist.barrier()
    dist.destroy_process_group()


def test_chunked_flush_allreduce_matches_single(tmp_path, oracle_mod):
    """parallel.flush_allreduce (the multi-GPU flush bench.py runs under NCCL):
    push-down once, rows of 3 point chunks each all-reduced asynchronously as
    soon as they exist, scatter to the original order — equal to the
    single-process flush of the whole batch (fp32 rows)."""
    O = oracle_mod
    mp.spawn(_flush_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "flush.npz")
    pos, nrm, area, mu, xs, d_out = _case()
    t = O.OracleTree(O.Cloud(pos, nrm, area, mu))
    t.set_kinds(np.array([0, 1, 1, 1], np.uint8))
    m, n, de = t.adjoint(O.Params(0.08), 2.0, xs, d_out, threads=1)
    assert np.abs(got["m"] - m).max() <= 2e-6 * np.abs(m).max()
    assert np.abs(got["n"] - n).max() <= 2e-6 * np.abs(n).max()
    assert abs(float(got["de"]) - de) <= 1e-12 * abs(de)
    calls = list(got["calls"])
    assert calls[0] == "begin" and calls[-1] == "end" and len(calls) == 5
