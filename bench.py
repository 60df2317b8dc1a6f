#!/usr/bin/env python
"""bench.py — Barnes-Hut dipole-sum queries/sec on B200 (BASELINE.json metric).

Workload (default): BASELINE config 4 — N = 8,000,000 points (64 random
spheres / tori + 3% outliers), C = 49 channels (ch 0 Dipole, 1..48 Radial),
Q = 64,000,000 Morton-unsorted uniform queries in [-2,2]^3, beta = 2, leaf 8,
eps = 1.5 x mean 8-NN spacing (the reference's value, recorded in workloads).
One STEP = forward primal of all Q queries + adjoint of the same Q queries
with N(0,1) upstream gradients + flush_gradients. With N GPUs the Q queries of
the step are sharded (STRONG scaling: every rank takes a contiguous 1/N of the
same global batch) against a replicated, bit-identical tree, and the per-point
gradients (moments, normals, d_eps) are NCCL-all-reduced in point chunks
overlapped with the gradient push-down (parallel.flush_allreduce).

value = Q / step time [queries/s; every query is evaluated forward AND
adjoint], CUDA events on the tree's stream, max over ranks, inputs resident in
HBM. e2e = the same through the public API from pinned HOST buffers (H2D of the
queries once per step and of d_out, D2H of the outputs and point gradients,
all inside the timed region). Step inputs (1.5 GB queries + 12.5 GB d_out at
N=1) exceed the 126 MB L2, so no explicit flush.

`python bench.py --gpus N` without WORLD_SIZE in the environment launches N
ranks itself (torch.distributed.run on 127.0.0.1); under torchrun it is one
rank. --config 2 selects BASELINE config 2 (N=1e6, Q=4e6) instead; at N=1 the
config-4 line also carries configs 1, 2, 3 and 5 under "extra" (every BASELINE
configuration in one driver-run line).

--impl reference: the reference's own CPU path (oracle/_ref, compiled from the
reference's sources unmodified) on the box's host cores, on a fixed 1M-query
subset of the same config-4 batch; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "dipole-sum queries/sec (forward, adjoint) at 1/2/4/8 B200; % of roofline"
UNIT = "queries/s"
BETA = 2.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[2, 4])
    ap.add_argument("--scale", type=float, default=1.0, help="shrink N and Q (development only)")
    ap.add_argument("--chunks", type=int, default=8, help="point chunks of the overlapped all-reduce")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the config-2 / config-5 extra lines")
    ap.add_argument("--ref-subset", type=int, default=1_000_000,
                    help="reference arm: queries of the fixed subset covered by the timed steps")
    ap.add_argument("--ref-workers", type=int, default=4,
                    help="reference arm: adjoint GradientBuffers (SURVEY §8(d): <= 4 at config 4)")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
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

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = max(mx, float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ cost model
def flops_model(tot, Cd, Cr):
    """SURVEY §8(d) cost model v1 (flop constants: add/mul 1, FMA 2, div/sqrt 4,
    exp 8, erf 16). tot = summed counters (V, F_near, F_far, P_near, P_far)."""
    V, Fn, Ff, Pn, Pf = [float(x) for x in tot]
    K0n, K0f, K2n = 40.0, 11.0, 12.0
    fwd = (9 * V + Fn * (K0n + 2 + 7 * Cd + 2 * Cr) + Ff * (K0f + 2 + 7 * Cd + 2 * Cr)
           + Pn * (14 + K0n + 2 * Cd + 2 * Cr) + Pf * (14 + K0f + 2 * Cd + 2 * Cr))
    adj = (9 * V + Fn * (K0n + K2n + 2 + 15 * Cd + 6 * Cr) + Ff * (K0f + 2 + 7 * Cd + 2 * Cr)
           + Pn * (14 + K0n + K2n + 15 * Cd + 6 * Cr) + Pf * (14 + K0f + 11 * Cd + 3 * Cr))
    return fwd, adj


# ------------------------------------------------------------------ workloads
class Workload:
    """One BASELINE configuration, with this rank's shard of the global query
    batches (strong scaling: the global batch is the same for every rank count)."""

    def __init__(self, config, scale, rank, world, queries=True):
        from paper_2405_16788_b200 import parallel as Pl
        from paper_2405_16788_b200 import workloads as W

        self.config = config
        if config == 4:
            w = W.config4(scale=scale, queries=False)
            self.q_total = w["q"]
            self.eps = W.EPSILON["config4"] / math.sqrt(scale)
            self.desc = ("config4: N=8e6 (64 spheres/tori + 3% outliers), C=49 (1 Dipole + 48 "
                         "Radial), Q=64e6 Morton-unsorted uniform queries in [-2,2]^3, beta=2, leaf 8, "
                         "forward+adjoint+flush per step")
            lo, hi = Pl.shard_range(self.q_total, rank, world)
            self.lo, self.hi = lo, hi
            self.batches = ([W.config4_queries(lo, hi, batch=b) for b in (0, 1)] if queries
                            else None)
        else:
            w = W.config2(scale=scale)
            self.q_total = w["xs"].shape[0]
            self.eps = W.epsilon_for("config2", scale)
            self.desc = ("config2: N=1e6 torus+outliers, C=49 (1 Dipole + 48 Radial), Q=4e6 "
                         "uniform queries in [-2,2]^3, beta=2, leaf 8, forward+adjoint+flush per step")
            lo, hi = Pl.shard_range(self.q_total, rank, world)
            self.lo, self.hi = lo, hi
            b1 = W.step_queries(w, 0, 1)
            self.batches = [w["xs"][lo:hi], b1[lo:hi]] if queries else None
            self.xs0_full = w["xs"]
        self.cloud = w["cloud"]
        self.kinds = w["kinds"]
        self.name = w["name"]


# ------------------------------------------------------------------ reference (CPU)
def cpu_info():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def ref_tree(wl):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    if not O.have_ref():
        raise RuntimeError("oracle/_ref/libdipole_ref.so missing (built by __graft_entry__.build())")
    c = wl.cloud
    t0 = time.time()
    tree = O.OracleTree(O.Cloud(c.positions, c.normals, c.areas, c.moments), backend="ref")
    tree.set_kinds(wl.kinds)
    return O, tree, time.time() - t0


def ref_workers(tree, want):
    """Adjoint GradientBuffers: <= want, and <= what half the host RAM holds
    (each is nodes x C x 4 + N x (C + 3) doubles, bhtree.cpp:336-343)."""
    bb = 8.0 * (tree.node_count() * tree.C * 4 + tree.n * (tree.C + 3))
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16e9
    return int(max(1, min(want, 0.5 * avail // bb))), bb


def reference_sample(O, tree, wl, n_fwd, n_adj, workers, threads):
    """Reference path on bounded samples: DipoleTree::primal over n_fwd queries
    (parallel_for, `threads` workers), adjoint over n_adj queries into `workers`
    caller-held GradientBuffers, one flush_gradients. Returns per-query costs and
    the per-step fixed cost (buffer setup + flush), and the extrapolated rate."""
    from paper_2405_16788_b200 import workloads as W

    p = O.Params(wl.eps)
    xs = W.config4_queries(0, max(n_fwd, n_adj)) if wl.config == 4 else wl.xs0_full[:max(n_fwd, n_adj)]
    d_out = W.upstream(n_adj, tree.C, [11, 0]).astype(np.float64)
    nw = min(2000, n_fwd, n_adj)  # untimed warm-up slice (as the --impl reference arm does)
    tree.primal(p, BETA, xs[:nw], threads=threads)
    t = time.time()
    tree.primal(p, BETA, xs[:n_fwd], threads=threads)
    tf = time.time() - t
    t = time.time()
    bufs = tree.gradient_buffers(workers)
    tsetup = time.time() - t
    bufs.adjoint(p, BETA, xs[:nw], d_out[:nw])
    t = time.time()
    bufs.adjoint(p, BETA, xs[:n_adj], d_out)
    ta = time.time() - t
    t = time.time()
    bufs.flush(want=False)
    tflush = time.time() - t
    del bufs
    Q = wl.q_total
    full = Q * tf / n_fwd + Q * ta / n_adj + tsetup + tflush
    return dict(value=Q / full, full_step_s=full, forward_qps=n_fwd / tf, adjoint_qps=n_adj / ta,
                t_forward_s=tf, t_adjoint_s=ta, t_buffer_setup_s=tsetup, t_flush_s=tflush)


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from paper_2405_16788_b200 import workloads as W

    wl = Workload(args.config, args.scale, 0, 1, queries=False)
    O, tree, build_s = ref_tree(wl)
    cores = O.ref_lib().ref_hardware_concurrency()
    workers, buf_bytes = ref_workers(tree, args.ref_workers)
    p = O.Params(wl.eps)
    C = tree.C
    Q = wl.q_total
    # fixed subset: the first `sub` queries of the step's batch (the batch is
    # i.i.d. uniform, so a prefix is a random subset); the timed steps cover it
    # in K contiguous slices; warm-up steps use small slices after it
    sub = int(min(Q, args.ref_subset))
    K, Wm = max(1, args.steps), max(0, args.warmup)
    s = -(-sub // K)
    wq = max(1, min(2000, s))
    xq = (W.config4_queries(0, sub + Wm * wq) if wl.config == 4
          else W.config2(scale=args.scale)["xs"][:sub + Wm * wq])
    d_out = W.upstream(xq.shape[0], C, [11, 1]).astype(np.float64)
    t = time.time()
    bufs = tree.gradient_buffers(workers)  # make_buffer per worker (per-step fixed cost)
    t_setup = time.time() - t
    for i in range(Wm):
        a, b = sub + i * wq, sub + (i + 1) * wq
        tree.primal(p, BETA, xq[a:b], threads=cores)
        bufs.adjoint(p, BETA, xq[a:b], d_out[a:b])
    bufs.flush(want=False)  # warm-up contributions do not reach the timed flush
    t_f = t_a = 0.0
    t0 = time.time()
    for k in range(K):
        a, b = k * s, min(sub, (k + 1) * s)
        if b <= a:
            continue
        t = time.time()
        tree.primal(p, BETA, xq[a:b], threads=cores)
        t_f += time.time() - t
        t = time.time()
        bufs.adjoint(p, BETA, xq[a:b], d_out[a:b])
        t_a += time.time() - t
    t = time.time()
    bufs.flush(want=False)  # flush_gradients(span) of the timed queries (zeroes the buffers)
    t_flush = time.time() - t
    timed = time.time() - t0
    full = Q * (t_f + t_a) / sub + t_setup + t_flush
    value = Q / full
    desc = (f"fixed {sub}-query prefix of the config-{wl.config} batch (of {Q}) covered by the "
            f"{K} timed steps ({s} queries each: forward with {cores} threads + adjoint into "
            f"{workers} GradientBuffers), one flush_gradients after them; full step "
            f"extrapolated as Q*(t_fwd+t_adj)/subset + buffer setup + flush; reference sources "
            f"compiled -O3 without -march; CPU {cpu_info()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * timed / K, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": f"synthetic (seeded config-{wl.config} generator)",
        # the same workload keys as the GPU arm's line; what was sampled is in "sample"
        "config": {"workload": wl.desc, "points": int(wl.cloud.size), "queries": int(Q),
                   "channels": int(C), "epsilon": wl.eps, "nodes": int(tree.node_count())},
        "sample": {"subset_queries": sub, "queries_per_timed_step": s, "timed_steps": K,
                   "adjoint_workers": workers, "threads": cores},
        "ms_per_step_note": "measured: the timed region (K sample steps + the flush) / K",
        "extrapolated_full_step_ms": 1e3 * full,
        "forward_qps": sub / t_f, "adjoint_qps": sub / t_a,
        "reference_timings": {"forward_s": t_f, "adjoint_s": t_a, "flush_s": t_flush,
                              "buffer_setup_s": t_setup, "tree_build_s": build_s,
                              "gradient_buffer_bytes": buf_bytes},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "adjoint_workers": workers,
                         "kind": "reference", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ------------------------------------------------------------------ our arm
def measure_device(tree, wl, params, dev, steps, warmup, dist, chunks, local):
    """The step on device-resident inputs: returns timing, phases, counters."""
    import torch

    from paper_2405_16788_b200 import bhtree as B
    from paper_2405_16788_b200 import parallel as Pl

    stream = torch.cuda.current_stream()
    N, C = wl.cloud.size, wl.cloud.channels
    xs_b = [torch.from_numpy(b).to(dev) for b in wl.batches]
    Qr = xs_b[0].shape[0]
    g = torch.Generator(device=dev).manual_seed(1000 + wl.lo)
    d_out = torch.randn((Qr, C), generator=g, device=dev, dtype=torch.float32)
    out = torch.empty((Qr, C), dtype=torch.float32, device=dev)
    mom = torch.empty((N, C), dtype=torch.float32, device=dev)
    nrm = torch.empty((N, 3), dtype=torch.float32, device=dev)
    rows = torch.empty((N, C + 3), dtype=torch.float32, device=dev) if dist is not None else None
    buf = tree.make_buffer()

    # counting pass (untimed): replays the opening decisions -> algorithmic work
    tot = 0
    for xb in xs_b:
        _, cnt = tree.primal(xb, params, BETA, out=out, visited=True)
        tot = tot + cnt.sum(dim=0).cpu().numpy() / len(xs_b)
        del cnt
    it = [0]

    def step():
        xs = xs_b[it[0] % 2]
        it[0] += 1
        tree.primal(xs, params, BETA, out=out)
        tree.adjoint(xs, params, BETA, d_out, None, buf)
        if dist is None:
            tree.flush_gradients(buf, out=(mom, nrm))
        else:
            Pl.flush_allreduce(tree, buf, rows=rows, chunks=chunks, out=(mom, nrm))

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    B.profile_read(tree)
    B.profile_enable(tree, True)
    launches0 = B.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
    launches = B.launch_count() - launches0
    ms = e0.elapsed_time(e1) / steps
    prof = B.profile_read(tree)
    B.profile_enable(tree, False)
    ms_t = torch.tensor([ms], device=dev)
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ph = {k: prof[k][0] / max(1, prof[k][1]) for k in ("forward", "adjoint")}
    ph["morton_sort_x2"] = prof["sort"][0] / steps
    ph["flush"] = prof["flush"][0] / steps
    del xs_b, d_out, out
    return dict(ms=float(ms_t.item()), ms_local=ms, phases=ph, tot=tot, launches=int(launches),
                clocks=clk.summary(), buf=buf, mom=mom, nrm=nrm, rows=rows, Qr=Qr)


def roofline_for(tot, Cd, Cr, ph, peak32, traffic):
    f_fwd, f_adj = flops_model(tot, Cd, Cr)
    dom = "adjoint" if ph["adjoint"] >= ph["forward"] else "forward"
    fl = f_adj if dom == "adjoint" else f_fwd
    achieved = fl / (ph[dom] * 1e-3) / 1e12
    return dom, {"bound": "fp32", "achieved": achieved, "peak": peak32, "unit": "TFLOP/s",
                 "frac": achieved / peak32, "flops_per_launch": fl,
                 "traffic": (traffic or {}).get(dom)}


def load_traffic(config):
    """DRAM bytes per launch of the dominant kernels from the committed ncu capture."""
    for name in (f"r02_traffic_config{config}.json", "r01_traffic.json" if config == 2 else ""):
        if not name:
            continue
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                tj = json.load(f)
            out = {"_source": tj["_source"]}
            for k in ("adjoint", "forward"):
                if k in tj:
                    out[k] = tj[k]["dram_read"] + tj[k]["dram_write"]
            return out
        except (OSError, KeyError, ValueError):
            continue
    return None


def run_ours(args):
    import torch

    import paper_2405_16788_b200 as P
    from paper_2405_16788_b200 import bhtree as B
    from paper_2405_16788_b200 import parallel as Pl

    rank, world, local = env_rank()
    dist = None
    # DPL_BENCH_DIST=1 exercises the NCCL path at world size 1 (one-GPU boxes)
    if world > 1 or os.environ.get("DPL_BENCH_DIST"):
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    t0 = time.time()
    wl = Workload(args.config, args.scale, rank, world)
    gen_s = time.time() - t0
    c = wl.cloud
    N, C = c.size, c.channels
    params = P.KernelParams(epsilon=wl.eps)
    tree = P.DipoleTree(local, stream=stream)
    t0 = time.time()
    tree.build(c)
    tree.set_channel_kernels(wl.kinds)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    nodes = tree.node_count()

    m = measure_device(tree, wl, params, dev, args.steps, args.warmup, dist, args.chunks, local)
    Qr, ph, tot = m["Qr"], m["phases"], m["tot"]
    value = wl.q_total / (m["ms"] * 1e-3)

    # ------------------------------------------------------------ e2e (host buffers)
    e2e = None
    if not args.no_e2e:
        xs_hb = [torch.from_numpy(b).pin_memory() for b in wl.batches]
        do_h = torch.empty((Qr, C), dtype=torch.float32, pin_memory=True)
        do_h.copy_(torch.randn((Qr, C), generator=torch.Generator(device=dev).manual_seed(7 + rank),
                               device=dev))
        out_h = torch.empty((Qr, C), dtype=torch.float32, pin_memory=True)
        mom_h = torch.empty((N, C), dtype=torch.float32, pin_memory=True)
        nrm_h = torch.empty((N, 3), dtype=torch.float32, pin_memory=True)
        buf = m["buf"]
        rows = m["rows"]
        # host-async mode: primal / adjoint return once queued, so the d_out H2D
        # overlaps the forward kernel and the out D2H overlaps the adjoint; the
        # adjoint reuses the primal's device copy of the queries (xs=None); the
        # flush synchronizes every stream (all host results complete)
        tree.set_host_async(True)
        it = [0]

        def step_host():
            xs_h = xs_hb[it[0] % 2]
            it[0] += 1
            tree.primal(xs_h, params, BETA, out=out_h)
            tree.adjoint(None, params, BETA, do_h, None, buf)
            # the next step's queries upload while this adjoint runs (a data
            # loader's prefetch); the flush's point gradients land while the
            # next step's kernels run (host-async; complete at synchronize)
            tree.prefetch(xs_hb[it[0] % 2])
            if dist is None:
                tree.flush_gradients(buf, out=(mom_h, nrm_h))
            else:
                Pl.flush_allreduce(tree, buf, rows=rows, chunks=args.chunks, out=(mom_h, nrm_h))

        step_host()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        tree.synchronize()
        k2 = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(k2):
            step_host()
        tree.synchronize()  # every step's outputs and point gradients are on the host
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / k2
        tree.set_host_async(False)
        t_t = torch.tensor([e2e_s], device=dev)
        if dist is not None:
            dist.all_reduce(t_t, op=dist.ReduceOp.MAX)
        e2e_s = float(t_t.item())
        h2d = Qr * 24 + Qr * C * 4
        d2h = Qr * C * 4 + N * C * 4 + N * 12 + 8
        e2e = {"value": wl.q_total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * e2e_s,
               "timing": "wall clock around public-API calls on pinned host buffers (host-async "
                         "mode: the adjoint reuses the primal's device copy of the queries, the next "
                         "batch is prefetched during the adjoint, the point gradients download while "
                         "the next step runs; synchronized at the end: every step's outputs and "
                         "gradients on the host), max over ranks",
               "bytes": "per rank"}
        del xs_hb, do_h, out_h

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    traffic = load_traffic(args.config)
    peak32 = B.peak_fp32(local)
    dom, roof = roofline_for(tot, 1, C - 1, ph, peak32, traffic)
    roof.update({"kernel": {"adjoint": "k_adjoint2 (interaction-list replay)",
                            "forward": "k_forward_tc (interaction-list replay)"}[dom],
                 "peak_source": "measured FFMA microbenchmark in this run (dpl_peak_fp32); "
                                "MEASURED_PEAKS.json has no FP32 figure",
                 "flop_model": "SURVEY §8(d) cost model v1 on replayed counters (rank 0's shard)",
                 "traffic_source": (traffic or {}).get("_source"),
                 "peak_fp64_measured": B.peak_fp64(local)})
    # per-launch duration of the dominant kernel: CUDA events around each launch
    # on the tree's stream (dpl_profile), mean over the timed steps

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            O, rtree, rbuild = ref_tree(wl)
            cores = O.ref_lib().ref_hardware_concurrency()
            workers, _ = ref_workers(rtree, 4)
            n_fwd, n_adj = (400_000, 160_000) if args.config == 4 else (400_000, 100_000)
            n_fwd, n_adj = (max(1000, int(n_fwd * args.scale)), max(500, int(n_adj * args.scale)))
            r = reference_sample(O, rtree, wl, n_fwd, n_adj, workers, cores)
            del rtree
            cpu = {"value": r["value"], "unit": UNIT, "cores": cores, "kind": "reference",
                   "adjoint_workers": workers,
                   "sample": f"{n_fwd} forward queries ({cores} threads) + {n_adj} adjoint "
                             f"queries ({workers} GradientBuffers) + one flush_gradients of the "
                             f"config-{args.config} workload; the {wl.q_total}-query step "
                             f"extrapolated as Q*t_query + buffer setup + flush; reference "
                             f"sources compiled unmodified; CPU {cpu_info()}",
                   "measured": {k: v for k, v in r.items() if k != "value"},
                   "tree_build_s": rbuild}
        except Exception as e:  # report, do not hide
            cpu = {"value": None, "error": str(e)}

    Qsh = m["Qr"]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": m["ms"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f32 (fp64 opening tests and accumulators)",
        "data": f"synthetic (seeded config-{args.config} generator; no dataset)",
        "config": {"workload": wl.desc, "points": N, "queries": wl.q_total,
                   "queries_per_gpu": Qsh, "channels": C, "nodes": nodes, "epsilon": wl.eps,
                   "l2": "inputs > L2 (queries + d_out per step >> 126 MB), no explicit flush",
                   "batches": "2 query batches alternated per step (no cross-step reuse); "
                              "the adjoint reuses its own step's interaction lists",
                   "parallelism": f"replicated tree, {world}-way query sharding"
                                  + (f", NCCL all-reduce of point gradients in {args.chunks} "
                                     "chunks overlapped with the push-down" if world > 1 else "")},
        "forward_qps": wl.q_total / ((ph["forward"] + ph["morton_sort_x2"] / 2) * 1e-3),
        "adjoint_qps": wl.q_total / ((ph["adjoint"] + ph["morton_sort_x2"] / 2 + ph["flush"]) * 1e-3),
        "phase_ms": ph,
        "interactions_per_query": float((tot[1] + tot[2] + tot[3] + tot[4]) / Qsh),
        "visited_per_query": float(tot[0] / Qsh),
        "roofline": roof,
        "gpu_launches": m["launches"],
        "clocks": m["clocks"],
        "build_s": build_s, "generate_s": gen_s,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    del m
    if world == 1 and args.config == 4 and not args.no_extra:
        try:
            line["extra"] = {"config2": extra_config2(args, dev, local, peak32)}
        except Exception as e:
            line["extra"] = {"config2": {"error": str(e)}}
        # release the config-4 tree (its staging buffers), the gradient buffer that
        # references it and torch's cached blocks before the larger extras
        import gc

        tree = wl = c = None
        buf = rows = mom_h = nrm_h = None  # noqa: F841 (set in the e2e leg)
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        for name, fn in (("config1", extra_config1), ("config3", lambda a, d, l: extra_render(a, d, l, 3)),
                         ("config5", lambda a, d, l: extra_render(a, d, l, 5))):
            try:
                line["extra"][name] = fn(args, dev, local)
            except Exception as e:
                line["extra"][name] = {"error": str(e)}
            gc.collect()
            torch.cuda.empty_cache()
    emit(line)
    if dist is not None:
        dist.destroy_process_group()


def extra_config2(args, dev, local, peak32):
    """BASELINE config 2 on the same GPU (device-resident inputs), N=1."""
    import torch

    import paper_2405_16788_b200 as P

    wl = Workload(2, args.scale, 0, 1)
    params = P.KernelParams(epsilon=wl.eps)
    tree = P.DipoleTree(local, stream=torch.cuda.current_stream())
    tree.build(wl.cloud)
    tree.set_channel_kernels(wl.kinds)
    m = measure_device(tree, wl, params, dev, max(args.steps, 10), args.warmup, None, 1, local)
    _, roof = roofline_for(m["tot"], 1, wl.cloud.channels - 1, m["phases"], peak32,
                           load_traffic(2))
    return {"workload": wl.desc, "value": wl.q_total / (m["ms"] * 1e-3), "unit": UNIT,
            "ms_per_step": m["ms"], "phase_ms": m["phases"], "roofline_frac": roof["frac"],
            "roofline_achieved_tflops": roof["achieved"], "gpu_launches": m["launches"],
            "clocks": m["clocks"]}


def extra_config1(args, dev, local):
    """BASELINE config 1 on the same GPU: forward-only, N=1e5 sphere, C=2,
    Q=1e6 uniform queries (two alternating batches: no list reuse), CUDA events
    on the tree's stream, inputs device-resident."""
    import torch

    import paper_2405_16788_b200 as P
    from paper_2405_16788_b200 import workloads as W

    w = W.config1(scale=args.scale)
    c = w["cloud"]
    tree = P.DipoleTree(local, stream=torch.cuda.current_stream())
    tree.build(c)
    tree.set_channel_kernels(w["kinds"])
    Q, C = w["xs"].shape[0], c.channels
    xs_b = [torch.from_numpy(w["xs"]).to(dev), torch.from_numpy(W.step_queries(w, 0, 1)).to(dev)]
    out = torch.empty((Q, C), device=dev)
    p = P.KernelParams(epsilon=W.epsilon_for("config1", args.scale))
    for i in range(max(3, args.warmup)):
        tree.primal(xs_b[i % 2], p, BETA, out=out)
    k = max(10, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(k):
        tree.primal(xs_b[i % 2], p, BETA, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    return {"workload": f"config1: N={c.size} sphere, C={C}, Q={Q} uniform queries in [-1.5,1.5]^3, "
                        "forward only (query sort + traversal)",
            "value": Q / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "steps": k}


def extra_render(args, dev, local, config):
    """BASELINE configs 3 and 5 on the same GPU, N=1. Config 3: render step on
    the config-1 cloud (C=4), 65,536 rays x 128 samples: render forward -> L2
    d_rgb -> render backward / adjoint -> flush. Config 5: the full
    differentiable step on N=4e6 points, C=49, 1,048,576 rays x 192 samples, also
    Adam on beta, alpha, n and update_moments. Direct-rgb head. Timed with CUDA
    events on the tree's stream; rays and targets device-resident
    (tools/bench_configs.py --config 3|5 is the same step with its roofline and
    CPU baseline)."""
    import numpy as np
    import torch

    import paper_2405_16788_b200 as P
    from paper_2405_16788_b200 import bhtree as B
    from paper_2405_16788_b200 import renderer as Rn
    from paper_2405_16788_b200 import workloads as W

    if config == 3:
        w = W.config3(scale=args.scale)
        c, rays, S, kinds = w["cloud"], w["rays"], w["S"], w["kinds"]
        what = "config-1 sphere cloud"
    else:
        n = max(64, int(4_000_000 * args.scale))
        pos, nrm_, area, rng = W.shapes_cloud(n, 5)
        mu = rng.standard_normal((n, 49))
        mu[:, 0] = 1.0  # geometry moment 1: the shapes' winding-number field (opaque surfaces)
        c = W.cloud(pos, nrm_, area, mu)
        kinds = np.ones(49, np.uint8)
        kinds[0] = 0
        rays = W.camera_rays(64, 1024, max(1, int(16384 * args.scale)), seed=2)
        S = 192
        what = "shapes cloud"
    eps = B.default_epsilon(c)
    tree = P.DipoleTree(local, stream=torch.cuda.current_stream())
    tree.build(c)
    tree.set_channel_kernels(kinds)
    R = rays.shape[0]
    rays_d = torch.from_numpy(rays).to(dev)
    target = torch.rand((R, 3), device=dev, generator=torch.Generator(device=dev).manual_seed(4))
    p = P.KernelParams(epsilon=eps)
    rs = Rn.RenderSettings(t_near=2.0, t_far=6.0, seed=3)
    buf = tree.make_buffer()
    mom = torch.empty((c.size, c.channels), device=dev)
    nrm = torch.empty((c.size, 3), device=dev)
    opt = B.PointAdam(tree, lr=1e-2) if config == 5 else None
    tape = Rn.Tape()
    scale = 2.0 / (3.0 * R)

    def step():
        rgb, _ = Rn.render_forward(tree, p, rs, rays_d, S, tape=tape)
        d_rgb = (scale * (rgb - target)).float()
        Rn.render_backward(tree, p, rs, tape, d_rgb, buf)
        g = tree.flush_gradients(buf, out=(mom, nrm))
        if opt is not None:
            opt.step(g)

    for _ in range(max(3, args.warmup)):  # the list policy settles after one step
        step()
    torch.cuda.synchronize()
    B.profile_read(tree)
    B.profile_enable(tree, True)
    l0 = B.launch_count()
    k = max(3, min(args.steps, 5)) if config == 5 else max(10, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    prof = B.profile_read(tree)
    B.profile_enable(tree, False)
    Q = R * S
    tail = (" + Adam(beta, alpha, n) + update_moments" if config == 5 else "")
    return {"workload": f"config{config}: N={c.size} {what}, C={c.channels}, {R} rays x {S} samples "
                        f"= {Q} queries per step; render forward + composite + L2 adjoint + flush"
                        f"{tail}; direct-rgb head",
            "value": Q / (ms * 1e-3), "unit": "ray samples/s", "ms_per_step": ms, "steps": k,
            "phase_ms": {key: v[0] / k for key, v in prof.items() if v[1]},
            "gpu_launches": B.launch_count() - l0,
            "channels_computed": f"0..3 of {c.channels}: the direct-rgb head reads only these "
                                 "(radiance.cpp:133-145); the reference interpolates every channel "
                                 "(renderer.cpp:125), the others never reach the output and "
                                 "receive exactly zero adjoint"}


# ------------------------------------------------------------------ launcher
_JSON_OUT = None


def emit(line):
    """The one JSON line, on the process's original stdout."""
    out = _JSON_OUT or sys.stdout
    print(json.dumps(line), file=out, flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(n, json_fd):
    """`--gpus N` outside torchrun: launch N ranks of this script (one per GPU)
    with torch.distributed.run on 127.0.0.1; rank 0's JSON line goes straight
    to our stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, stdout=json_fd, stderr=sys.stderr)


def main():
    global _JSON_OUT
    # stdout carries exactly one JSON line: anything else native code prints
    # there (e.g. NCCL's version banner at communicator creation) goes to stderr
    sys.stdout.flush()
    json_fd = os.dup(1)
    _JSON_OUT = os.fdopen(json_fd, "w")
    os.dup2(2, 1)
    args = parse()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus, json_fd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
