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
xs_h = torch.from_numpy(w['xs']).pin_memory()
do_h = torch.from_numpy(W.upstream(Q, C, w['d_out_seed'])).pin_memory()
out_h = torch.empty((Q, C), dtype=torch.float32).pin_memory()
mom_h = torch.empty((N, C), dtype=torch.float32).pin_memory(); nrm_h = torch.empty((N, 3), dtype=torch.float32).pin_memory()
buf = t.make_buffer()
xs_d = xs_h.to(dev); do_d = do_h.to(dev); out_d = torch.empty((Q, C), device=dev)
def tm(f, k=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): f()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / k
print('fwd host  ', tm(lambda: t.primal(xs_h, p, 2.0, out=out_h)))
print('fwd dev   ', tm(lambda: t.primal(xs_d, p, 2.0, out=out_d)))
print('adj host  ', tm(lambda: t.adjoint(xs_h, p, 2.0, do_h, None, buf)))
print('adj dev   ', tm(lambda: t.adjoint(xs_d, p, 2.0, do_d, None, buf)))
print('flush host', tm(lambda: t.flush_gradients(buf, out=(mom_h, nrm_h))))
print('H2D 976MB ', tm(lambda: (xs_h.to(dev, non_blocking=True), do_h.to(dev, non_blocking=True))))
print('D2H 784MB ', tm(lambda: out_h.copy_(out_d, non_blocking=True)))
from paper_2405_16788_b200 import bhtree as B
B.profile_read(t); B.profile_enable(t, True)
t.primal(xs_h, p, 2.0, out=out_h); torch.cuda.synchronize()
print('host-path kernel phases', B.profile_read(t))
B.profile_enable(t, False)
t2 = P.DipoleTree(0); t2.build(c); t2.set_channel_kernels(w['kinds'])
print('fwd host own-stream', tm(lambda: t2.primal(xs_h, p, 2.0, out=out_h)))
buf2 = t2.make_buffer()
print('adj host own-stream', tm(lambda: t2.adjoint(xs_h, p, 2.0, do_h, None, buf2)))
