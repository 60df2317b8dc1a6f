import sys, time, torch
sys.path.insert(0, '.')
import paper_2405_16788_b200 as P
from paper_2405_16788_b200 import workloads as W
w = W.config4(scale=1.0)
c = w['cloud']
for i in range(2):
    t = P.DipoleTree(0, stream=torch.cuda.current_stream())
    torch.cuda.synchronize(); t0 = time.perf_counter()
    t.build(c); t.set_channel_kernels(w['kinds'])
    torch.cuda.synchronize(); print('build_s', time.perf_counter() - t0, flush=True)
    del t
