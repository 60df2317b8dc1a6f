"""e2e step timing breakdown on config 2: synchronous vs host-async mode, same vs alternating pinned query batches (python tools/e2e_breakdown.py on a GPU box)."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2405_16788_b200 as P
from paper_2405_16788_b200 import workloads as W
w = W.config2(); c = w['cloud']
eps = W.epsilon_for('config2')
dev = torch.device('cuda', 0)
t = P.DipoleTree(0, stream=torch.cuda.current_stream()); t.build(c); t.set_channel_kernels(w['kinds'])
Q, N, C = w['xs'].shape[0], c.size, c.channels
p = P.KernelParams(epsilon=eps)
xs_hb = [torch.from_numpy(w['xs']).pin_memory(), torch.from_numpy(W.step_queries(w, 0, 1)).pin_memory()]
do_h = torch.from_numpy(W.upstream(Q, C, w['d_out_seed'])).pin_memory()
out_h = torch.empty((Q, C), dtype=torch.float32).pin_memory()
mom_h = torch.empty((N, C), dtype=torch.float32).pin_memory(); nrm_h = torch.empty((N, 3), dtype=torch.float32).pin_memory()
buf = t.make_buffer()
it = [0]
def step(alt=True, sync_each=False):
    x = xs_hb[it[0] % 2] if alt else xs_hb[0]
    it[0] += 1
    t0 = time.perf_counter()
    t.primal(x, p, 2.0, out=out_h)
    if sync_each: t.synchronize()
    t1 = time.perf_counter()
    t.adjoint(x, p, 2.0, do_h, None, buf)
    if sync_each: t.synchronize()
    t2 = time.perf_counter()
    t.flush_gradients(buf, out=(mom_h, nrm_h))
    t3 = time.perf_counter()
    return 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2)
for mode in (False, True):
    t.set_host_async(mode)
    for alt in (False, True):
        for _ in range(3): step(alt)
        torch.cuda.synchronize()
        a = time.perf_counter(); parts = [step(alt) for _ in range(5)]; torch.cuda.synchronize()
        print(f"async={mode} alt={alt}: {1e3*(time.perf_counter()-a)/5:.1f} ms/step; host-call ms (fwd, adj, flush) = {np.mean(parts, axis=0).round(1)}")
    for _ in range(2): step(True, True)
    parts = [step(True, True) for _ in range(3)]
    print(f"async={mode} alt, synced per call (fwd, adj, flush) = {np.mean(parts, axis=0).round(1)}")
