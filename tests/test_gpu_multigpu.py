"""GPU side of the multi-GPU path at world size 1 (one GPU per gpurun box):
the split flush (flush_begin / flush_rows / flush_end, the pieces
parallel.flush_allreduce interleaves with NCCL) gives exactly dpl_flush's
results, with and without NCCL at world size 1; the adjoint's xs=None reuse of
the primal's batch (host batches cross PCIe once) equals passing xs again.
The cross-rank orchestration itself is tested with gloo, world size 2
(tests/test_dist_cpu.py::test_chunked_flush_allreduce_matches_single)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def same(got, want):
    """Equal up to the fp64 atomic accumulation order of the adjoint (each run
    sums the same terms in a different order): <= 1 fp32 ulp, or 1e-12 of the
    largest entry where terms cancel."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    tol = 2.0 ** -23 * np.abs(want) + 1e-12 * np.abs(want).max(initial=0.0)
    bad = np.abs(got - want) > tol
    assert not bad.any(), f"{int(bad.sum())} entries differ, max {np.abs(got - want).max():.3e}"


def _setup(n=20000, q=60000, C=7, seed=3):
    import paper_2405_16788_b200 as P

    rng = np.random.default_rng(seed)
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32).astype(np.float64)
    nrm = rng.standard_normal((n, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    area = rng.uniform(0.5, 1, n) / n
    mu = rng.standard_normal((n, C))
    kinds = np.ones(C, np.uint8)
    kinds[0] = 0
    t = P.DipoleTree(0)
    t.build(P.OrientedPointCloud(pos, nrm, area, mu))
    t.set_channel_kernels(kinds)
    xs = rng.uniform(-1.3, 1.3, (q, 3)).astype(np.float32).astype(np.float64)
    d_out = rng.standard_normal((q, C)).astype(np.float32)
    return P, t, xs, d_out


@pytest.mark.parametrize("chunks", [1, 5])
def test_split_flush_equals_flush(chunks):
    import torch

    from paper_2405_16788_b200.parallel import flush_allreduce

    P, t, xs, d_out = _setup()
    p = P.KernelParams(epsilon=0.04)
    b = t.make_buffer()
    t.adjoint(xs, p, 2.0, d_out, None, b)
    g = t.flush_gradients(b)
    t.adjoint(xs, p, 2.0, d_out, None, b)
    mom, nrm, de = flush_allreduce(t, b, chunks=chunks)
    same(mom.cpu().numpy(), g.moments)
    same(nrm.cpu().numpy(), g.normals)
    assert abs(de - g.d_epsilon) <= 1e-12 * abs(g.d_epsilon)
    # the buffers were zeroed (reset(), bhtree.cpp:438)
    z = t.flush_gradients(b)
    assert not z.moments.any() and not z.normals.any() and z.d_epsilon == 0.0
    torch.cuda.synchronize()


def test_split_flush_nccl_world1():
    """The NCCL branch of flush_allreduce (async all-reduce per chunk on the
    tree's stream) at world size 1: sums over one rank are the identity."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2405_16788_b200.parallel import flush_allreduce

    P, t0, xs, d_out = _setup(seed=4)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        s = torch.cuda.Stream()
        t = P.DipoleTree(0, stream=s)
        import paper_2405_16788_b200.workloads  # noqa: F401

        rng = np.random.default_rng(4)
        n = t0.point_count()
        pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32).astype(np.float64)
        nrm = rng.standard_normal((n, 3))
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
        area = rng.uniform(0.5, 1, n) / n
        mu = rng.standard_normal((n, t0.channels()))
        kinds = np.ones(t0.channels(), np.uint8)
        kinds[0] = 0
        t.build(P.OrientedPointCloud(pos, nrm, area, mu))
        t.set_channel_kernels(kinds)
        p = P.KernelParams(epsilon=0.04)
        b = t.make_buffer()
        t.adjoint(xs, p, 2.0, d_out, None, b)
        g = t.flush_gradients(b)
        t.adjoint(xs, p, 2.0, d_out, None, b)
        # world size 1 skips the collectives; force them through a 1-rank NCCL group
        mom, nrm_, de = flush_allreduce(t, b, chunks=4)
        rows = torch.empty((n, t.channels() + 3), dtype=torch.float32, device="cuda")
        t.adjoint(xs, p, 2.0, d_out, None, b)
        de2 = t.flush_begin(b)
        with torch.cuda.stream(s):
            works = []
            for k in range(4):
                lo, hi = k * n // 4, (k + 1) * n // 4
                t.flush_rows(b, lo, hi, rows[lo:hi])
                works.append(dist.all_reduce(rows[lo:hi], async_op=True))
            for w in works:
                w.wait()
        m2, n2 = t.flush_end(b, rows)
        for got in (mom, m2):
            same(got.cpu().numpy(), g.moments)
        for got in (nrm_, n2):
            same(got.cpu().numpy(), g.normals)
        for d in (de, de2):
            assert abs(d - g.d_epsilon) <= 1e-12 * abs(g.d_epsilon)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("host_async", [False, True])
def test_adjoint_reuses_primal_batch(host_async):
    """dpl_adjoint(xs = NULL): the queries of the preceding primal (host batch
    uploaded once) — identical gradients to passing the batch again."""
    import torch

    P, t, xs, d_out = _setup(q=400_000, seed=5)  # > 2^18: the pipelined host path
    p = P.KernelParams(epsilon=0.04)
    C = t.channels()
    xs_h = torch.from_numpy(xs).pin_memory()
    do_h = torch.from_numpy(d_out).pin_memory()
    out_h = torch.empty((xs.shape[0], C), dtype=torch.float32).pin_memory()
    b = t.make_buffer()
    t.primal(xs_h, p, 2.0, out=out_h)
    t.adjoint(xs_h, p, 2.0, do_h, None, b)
    want = t.flush_gradients(b)
    want_out = out_h.numpy().copy()
    t.set_host_async(host_async)
    for _ in range(2):  # second round: lists policy on, hazards across calls
        t.primal(xs_h, p, 2.0, out=out_h)
        t.adjoint(None, p, 2.0, do_h, None, b)
        got = t.flush_gradients(b)
        t.synchronize()  # host-async: outputs complete after synchronize()
        assert np.array_equal(out_h.numpy(), want_out)
        same(got.moments, want.moments)
        same(got.normals, want.normals)
        assert abs(got.d_epsilon - want.d_epsilon) <= 1e-12 * abs(want.d_epsilon)
    t.set_host_async(False)


def test_adjoint_reuse_requires_preceding_primal():
    P, t, xs, d_out = _setup(q=1000, seed=6)
    p = P.KernelParams(epsilon=0.04)
    b = t.make_buffer()
    with pytest.raises(P.UsageError):
        t.adjoint(None, p, 2.0, d_out, None, b)
    t.primal(xs, p, 2.0)
    with pytest.raises(P.UsageError):  # different batch size
        t.adjoint(None, p, 2.0, d_out[:500], None, b)


def test_prefetch_and_async_flush_pipeline():
    """Host-async training loop as bench.py's e2e runs it: the next batch is
    prefetched while the adjoint runs and the point gradients of a flush arrive
    while the next step's kernels run — the results equal the synchronous
    loop's, batch by batch."""
    import torch

    P, t, xs, d_out = _setup(q=400_000, seed=8)
    p = P.KernelParams(epsilon=0.04)
    C, n = t.channels(), t.point_count()
    rng = np.random.default_rng(9)
    batches = [xs, rng.uniform(-1.3, 1.3, xs.shape).astype(np.float32).astype(np.float64)]
    xs_h = [torch.from_numpy(b).pin_memory() for b in batches]
    do_h = torch.from_numpy(d_out).pin_memory()
    b = t.make_buffer()
    want = []
    for k in range(2):  # synchronous reference results per batch
        out = torch.empty((xs.shape[0], C), dtype=torch.float32).pin_memory()
        t.primal(xs_h[k], p, 2.0, out=out)
        t.adjoint(None, p, 2.0, do_h, None, b)
        g = t.flush_gradients(b)
        want.append((out.numpy().copy(), g.moments.copy(), g.normals.copy(), g.d_epsilon))
    t.set_host_async(True)
    outs = [torch.empty((xs.shape[0], C), dtype=torch.float32).pin_memory() for _ in range(2)]
    moms = [torch.empty((n, C), dtype=torch.float32).pin_memory() for _ in range(2)]
    nrms = [torch.empty((n, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
    deps = []
    for step in range(4):
        k = step % 2
        t.primal(xs_h[k], p, 2.0, out=outs[k])
        t.adjoint(None, p, 2.0, do_h, None, b)
        t.prefetch(xs_h[(step + 1) % 2])
        deps.append(t.flush_gradients(b, out=(moms[k], nrms[k])).d_epsilon)
    t.synchronize()
    t.set_host_async(False)
    for k in range(2):
        assert np.array_equal(outs[k].numpy(), want[k][0])
        same(moms[k].numpy(), want[k][1])
        same(nrms[k].numpy(), want[k][2])
    for step, de in enumerate(deps):
        assert abs(de - want[step % 2][3]) <= 1e-12 * abs(want[step % 2][3])
